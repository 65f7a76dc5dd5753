// Green operator: setup (preconditioners.py:50-80) and the per-frequency
// block solve of its application (preconditioners.py:83-94), including the
// Parseval quadratic forms PCG needs (<r, G r>, <s, G s>) fused into the same
// pass over the half spectrum.
//
// Blocks are stored Hermitian-packed and planar (one plane of Nh doubles per
// packed entry) so that every access in the hot kernel is coalesced:
//   d = 2: G00, G11, Re G01, Im G01
//   d = 3: G00, G11, G22, Re G01, Im G01, Re G02, Im G02, Re G12, Im G12
#include <cmath>

#include "common.cuh"
#include "fft.cuh"

namespace jfftb {

int green_planes(int d) { return d == 2 ? 4 : 9; }

namespace {

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}

template <int NV>
__device__ __forceinline__ void block_sums(double (&v)[NV], double* red /*32*NV*/,
                                           double* out) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int j = 0; j < NV; ++j) v[j] = warp_sum(v[j]);
  __syncthreads();
  if (lane == 0)
#pragma unroll
    for (int j = 0; j < NV; ++j) red[j * 32 + wid] = v[j];
  __syncthreads();
  if (wid == 0) {
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      double s = lane < (int)(blockDim.x >> 5) ? red[j * 32 + lane] : 0.0;
      s = warp_sum(s);
      if (lane == 0) out[j] = s;
    }
  }
}

// Hermitian packed block, d x d
template <int D>
struct HBlock {
  double dg[D];
  double re[3], im[3];  // (0,1), (0,2), (1,2)
};

template <int D>
__device__ __forceinline__ HBlock<D> load_block(const double* __restrict__ b, int64_t Nh,
                                                int64_t f) {
  HBlock<D> B;
#pragma unroll
  for (int a = 0; a < D; ++a) B.dg[a] = __ldg(b + a * Nh + f);
  constexpr int NO = D == 2 ? 1 : 3;
#pragma unroll
  for (int k = 0; k < NO; ++k) {
    B.re[k] = __ldg(b + (D + 2 * k) * Nh + f);
    B.im[k] = __ldg(b + (D + 2 * k + 1) * Nh + f);
  }
  return B;
}

__device__ __forceinline__ int off_index(int a, int b) {  // a < b
  return a == 0 ? b - 1 : 2;
}

// z = G s ; returns s^H G s (real)
template <int D>
__device__ __forceinline__ double block_apply(const HBlock<D>& B, const double2 (&s)[D],
                                              double2 (&z)[D]) {
#pragma unroll
  for (int a = 0; a < D; ++a) {
    double zr = B.dg[a] * s[a].x, zi = B.dg[a] * s[a].y;
#pragma unroll
    for (int b = 0; b < D; ++b) {
      if (b == a) continue;
      const int k = a < b ? off_index(a, b) : off_index(b, a);
      const double gr = B.re[k];
      const double gi = a < b ? B.im[k] : -B.im[k];  // G_ba = conj(G_ab)
      zr += gr * s[b].x - gi * s[b].y;
      zi += gr * s[b].y + gi * s[b].x;
    }
    z[a] = make_double2(zr, zi);
  }
  double q = 0.0;
#pragma unroll
  for (int a = 0; a < D; ++a) q += s[a].x * z[a].x + s[a].y * z[a].y;
  return q;
}

template <int D>
__device__ __forceinline__ double block_quad(const HBlock<D>& B, const double2 (&s)[D]) {
  double2 z[D];
  return block_apply<D>(B, s, z);
}

__device__ __forceinline__ double parseval_weight(int64_t f, int nh, int nlast) {
  const int k = (int)(f % nh);
  return (k == 0 || (2 * k == nlast)) ? 1.0 : 2.0;
}

// ---------------------------------------------------------------------------
// out = G in / N for `nb` stacked vector spectra (apply_green's einsum + the
// inverse transform's 1/N); optional per-block partials of in^H G in / N.
// `in` and `out` may alias.
// ---------------------------------------------------------------------------
template <int D>
__global__ void green_apply_kernel(Geom g, const double* __restrict__ blocks,
                                   const double2* in, double2* out) {
  const double invN = 1.0 / (double)g.N;
  for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < g.Nh;
       f += (int64_t)gridDim.x * blockDim.x) {
    const HBlock<D> B = load_block<D>(blocks, g.Nh, f);
    double2 s[D], z[D];
#pragma unroll
    for (int a = 0; a < D; ++a) s[a] = in[a * g.Nh + f];
    block_apply<D>(B, s, z);
#pragma unroll
    for (int a = 0; a < D; ++a) out[a * g.Nh + f] = make_double2(z[a].x * invN, z[a].y * invN);
  }
}

// ---------------------------------------------------------------------------
// Green setup: K_ref^ from the impulse responses, Hermitise, pseudo-invert
// ---------------------------------------------------------------------------
// real symmetric cyclic Jacobi on the 2D x 2D embedding [[X,-Y],[Y,X]] of the
// Hermitian H = X + iY; pseudo-inverse with the reference's cutoff
template <int D>
__device__ void herm_pinv(const double (&Hr)[D][D], const double (&Hi)[D][D],
                          double (&Pr)[D][D], double (&Pi)[D][D]) {
  constexpr int R = 2 * D;
  double A[R][R], V[R][R];
#pragma unroll
  for (int i = 0; i < D; ++i)
#pragma unroll
    for (int j = 0; j < D; ++j) {
      A[i][j] = Hr[i][j];
      A[i + D][j + D] = Hr[i][j];
      A[i + D][j] = Hi[i][j];
      A[i][j + D] = -Hi[i][j];
    }
#pragma unroll
  for (int i = 0; i < R; ++i)
#pragma unroll
    for (int j = 0; j < R; ++j) V[i][j] = (i == j) ? 1.0 : 0.0;
  for (int sweep = 0; sweep < 30; ++sweep) {
    double off = 0.0, tot = 0.0;
#pragma unroll
    for (int i = 0; i < R; ++i)
#pragma unroll
      for (int j = 0; j < R; ++j) {
        tot += A[i][j] * A[i][j];
        if (i != j) off += A[i][j] * A[i][j];
      }
    if (off <= 1e-36 * tot || off == 0.0) break;
#pragma unroll
    for (int p = 0; p < R; ++p)
#pragma unroll
      for (int q = p + 1; q < R; ++q) {
        const double apq = A[p][q];
        if (apq == 0.0) continue;
        const double theta = (A[q][q] - A[p][p]) / (2.0 * apq);
        const double t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        const double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
#pragma unroll
        for (int k = 0; k < R; ++k) {  // A <- A J (columns p, q)
          const double akp = A[k][p], akq = A[k][q];
          A[k][p] = c * akp - s * akq;
          A[k][q] = s * akp + c * akq;
        }
#pragma unroll
        for (int k = 0; k < R; ++k) {  // A <- J^T A (rows p, q)
          const double apk = A[p][k], aqk = A[q][k];
          A[p][k] = c * apk - s * aqk;
          A[q][k] = s * apk + c * aqk;
        }
#pragma unroll
        for (int k = 0; k < R; ++k) {
          const double vkp = V[k][p], vkq = V[k][q];
          V[k][p] = c * vkp - s * vkq;
          V[k][q] = s * vkp + c * vkq;
        }
      }
  }
  double lmax = A[0][0];
#pragma unroll
  for (int i = 1; i < R; ++i) lmax = fmax(lmax, A[i][i]);
  const double cutoff = 1e-12 * fmax(lmax, 0.0);
  double inv[R];
#pragma unroll
  for (int i = 0; i < R; ++i) inv[i] = A[i][i] > cutoff ? 1.0 / A[i][i] : 0.0;
#pragma unroll
  for (int i = 0; i < D; ++i)
#pragma unroll
    for (int j = 0; j < D; ++j) {
      double pr = 0.0, pi = 0.0;
#pragma unroll
      for (int k = 0; k < R; ++k) {
        pr += V[i][k] * inv[k] * V[j][k];
        pi += V[i + D][k] * inv[k] * V[j][k];
      }
      Pr[i][j] = pr;
      Pi[i][j] = pi;
    }
}

// layout 0: numpy rfftn half spectrum (last axis halved), nfreq = Nh;
// layout 1: fused.cu half spectrum (axis 0 halved), nfreq = (n0/2+1) N / n0
template <int D>
__global__ void green_setup_kernel(Geom g, const double* __restrict__ resp, int m0, int m1,
                                   int m2, double* __restrict__ blocks, int layout,
                                   bool dif_last, int64_t nfreq, int k0_off) {
  // resp: D impulse responses (beta) of D components on the small m-grid
  const int m[3] = {m0, m1, m2};
  int64_t msz = 1;
  for (int a = 0; a < D; ++a) msz *= m[a];
  for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < nfreq;
       f += (int64_t)gridDim.x * blockDim.x) {
    int q[3];
    int64_t rem = f;
    if (layout == 0) {
      q[D - 1] = (int)(rem % g.nh);
      rem /= g.nh;
      for (int a = D - 2; a >= 0; --a) { q[a] = (int)(rem % g.n[a]); rem /= g.n[a]; }
    } else {
      for (int a = D - 1; a >= 1; --a) { q[a] = (int)(rem % g.n[a]); rem /= g.n[a]; }
      q[0] = (int)rem + k0_off;  // k0-slab of a distributed solve (dist.cu)
      // slot -> frequency of the in-place last-axis transform (fused pass C)
      if (dif_last) q[D - 1] = dif_freq(g.n[D - 1], q[D - 1]);
    }
    double Kr[D][D], Ki[D][D];
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
      for (int b = 0; b < D; ++b) Kr[a][b] = Ki[a][b] = 0.0;
    for (int64_t y = 0; y < msz; ++y) {
      int yy[3];
      int64_t r2 = y;
      for (int a = D - 1; a >= 0; --a) { yy[a] = (int)(r2 % m[a]); r2 /= m[a]; }
      // phase exp(-2 pi i sum_a q_a delta_a / n_a)
      double pr = 1.0, pim = 0.0;
      for (int a = 0; a < D; ++a) {
        int delta = yy[a];
        if (m[a] != g.n[a] && delta > 1) delta -= m[a];
        int64_t t = ((int64_t)q[a] * delta) % g.n[a];
        if (t < 0) t += g.n[a];
        double sn, cs;
        sincospi(-2.0 * (double)t / (double)g.n[a], &sn, &cs);
        const double nr = pr * cs - pim * sn, ni = pr * sn + pim * cs;
        pr = nr;
        pim = ni;
      }
#pragma unroll
      for (int b = 0; b < D; ++b)
#pragma unroll
        for (int a = 0; a < D; ++a) {
          const double v = resp[((int64_t)b * D + a) * msz + y];
          if (v != 0.0) {
            Kr[a][b] += v * pr;
            Ki[a][b] += v * pim;
          }
        }
    }
    bool dc = true;
    for (int a = 0; a < D; ++a) dc = dc && q[a] == 0;
    double Hr[D][D], Hi[D][D], Pr[D][D], Pi[D][D];
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
      for (int b = 0; b < D; ++b) {
        // 0.5 (K + K^H)
        Hr[a][b] = dc ? 0.0 : 0.5 * (Kr[a][b] + Kr[b][a]);
        Hi[a][b] = dc ? 0.0 : 0.5 * (Ki[a][b] - Ki[b][a]);
      }
    herm_pinv<D>(Hr, Hi, Pr, Pi);
    if (dc) {
#pragma unroll
      for (int a = 0; a < D; ++a)
#pragma unroll
        for (int b = 0; b < D; ++b) Pr[a][b] = Pi[a][b] = 0.0;
    }
#pragma unroll
    for (int a = 0; a < D; ++a) blocks[a * nfreq + f] = Pr[a][a];
    int k = 0;
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
      for (int b = a + 1; b < D; ++b) {
        blocks[(D + 2 * k) * nfreq + f] = 0.5 * (Pr[a][b] + Pr[b][a]);
        blocks[(D + 2 * k + 1) * nfreq + f] = 0.5 * (Pi[a][b] - Pi[b][a]);
        ++k;
      }
  }
}

int spec_blocks(int64_t n) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 16));
}

}  // namespace

void launch_green_apply(const Geom& g, cudaStream_t s, const double* blocks, const double2* in,
                        double2* out, int nbatch) {
  for (int b = 0; b < nbatch; ++b) {
    const double2* ib = in + (int64_t)b * g.d * g.Nh;
    double2* ob = out + (int64_t)b * g.d * g.Nh;
    if (g.d == 3) green_apply_kernel<3><<<spec_blocks(g.Nh), 256, 0, s>>>(g, blocks, ib, ob);
    else green_apply_kernel<2><<<spec_blocks(g.Nh), 256, 0, s>>>(g, blocks, ib, ob);
    JF_LAUNCHED();
  }
}

void launch_green_setup(const Geom& g, cudaStream_t s, const double* resp, int m3, double* blocks,
                        int layout, int64_t nfreq, bool dif_last, int k0_off) {
  // m3 packs the small-grid extents as m0 | m1 << 8 | m2 << 16
  const int m0 = m3 & 0xff, m1 = (m3 >> 8) & 0xff, m2 = (m3 >> 16) & 0xff;
  if (g.d == 3)
    green_setup_kernel<3><<<spec_blocks(nfreq), 128, 0, s>>>(g, resp, m0, m1, m2, blocks, layout, dif_last,
                                                             nfreq, k0_off);
  else
    green_setup_kernel<2><<<spec_blocks(nfreq), 128, 0, s>>>(g, resp, m0, m1, m2, blocks, layout, dif_last,
                                                             nfreq, k0_off);
  JF_LAUNCHED();
}

// ---------------------------------------------------------------------------
// PCG spectral step: per frequency, with r^ = spec[0:d] and (green-jacobi)
// s^ = spec[d:2d]:
//   MODE 0 (green)        z^ = G r^ / N  -> spec[0:d];   q0 = r^H Gt r^ / N,
//                                                        q1 = r^H G r^ / N
//   MODE 1 (green-jacobi) z^ = G s^ / N  -> spec[d:2d];  q0 = r^H Gt r^ / N,
//                                                        q1 = s^H G s^ / N
//   MODE 2 (none/jacobi)  q0 = r^H Gt r^ / N (no output)
// Gt is the termination Green operator, G the preconditioner's; the common
// case Gt == G reads one set of blocks.
// ---------------------------------------------------------------------------
template <int D, int MODE>
__global__ void __launch_bounds__(256)
    pcg_spectral_kernel(Geom g, const double* __restrict__ gpc, const double* __restrict__ gterm,
                        double2* spec, const PcgState* __restrict__ st,
                        double* __restrict__ partials) {
  __shared__ double red[64];
  if (st->done) return;
  const double invN = 1.0 / (double)g.N;
  const int nlast = g.n[D - 1];
  double q0 = 0.0, q1 = 0.0;
  for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < g.Nh;
       f += (int64_t)gridDim.x * blockDim.x) {
    const double w = parseval_weight(f, g.nh, nlast);
    double2 r[D];
#pragma unroll
    for (int a = 0; a < D; ++a) r[a] = spec[a * g.Nh + f];
    if (MODE == 0) {
      const HBlock<D> B = load_block<D>(gpc, g.Nh, f);
      double2 z[D];
      const double qp = w * block_apply<D>(B, r, z);
      q1 += qp;
      if (gterm != gpc) {
        const HBlock<D> Bt = load_block<D>(gterm, g.Nh, f);
        q0 += w * block_quad<D>(Bt, r);
      } else {
        q0 += qp;
      }
#pragma unroll
      for (int a = 0; a < D; ++a) spec[a * g.Nh + f] = make_double2(z[a].x * invN, z[a].y * invN);
    } else if (MODE == 1) {
      double2 s[D], z[D];
#pragma unroll
      for (int a = 0; a < D; ++a) s[a] = spec[(D + a) * g.Nh + f];
      const HBlock<D> B = load_block<D>(gpc, g.Nh, f);
      q1 += w * block_apply<D>(B, s, z);
      if (gterm == gpc) {
        q0 += w * block_quad<D>(B, r);
      } else {
        const HBlock<D> Bt = load_block<D>(gterm, g.Nh, f);
        q0 += w * block_quad<D>(Bt, r);
      }
#pragma unroll
      for (int a = 0; a < D; ++a)
        spec[(D + a) * g.Nh + f] = make_double2(z[a].x * invN, z[a].y * invN);
    } else {
      const HBlock<D> Bt = load_block<D>(gterm, g.Nh, f);
      q0 += w * block_quad<D>(Bt, r);
    }
  }
  double v[2] = {q0 * invN, q1 * invN};
  double out[2];
  block_sums<2>(v, red, out);
  if (threadIdx.x == 0) {
    partials[blockIdx.x * 2 + 0] = out[0];
    partials[blockIdx.x * 2 + 1] = out[1];
  }
}

void launch_pcg_spectral(const Geom& g, cudaStream_t s, int mode, const double* gpc,
                         const double* gterm, double2* spec, const PcgState* st,
                         double* partials) {
#define JF_SPEC(D, M) \
  pcg_spectral_kernel<D, M><<<kRedBlocks, 256, 0, s>>>(g, gpc, gterm, spec, st, partials)
  if (g.d == 3) {
    if (mode == 0) JF_SPEC(3, 0);
    else if (mode == 1) JF_SPEC(3, 1);
    else JF_SPEC(3, 2);
  } else {
    if (mode == 0) JF_SPEC(2, 0);
    else if (mode == 1) JF_SPEC(2, 1);
    else JF_SPEC(2, 2);
  }
#undef JF_SPEC
  JF_LAUNCHED();
}

}  // namespace jfftb
