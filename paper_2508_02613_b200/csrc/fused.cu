// Fused spectral passes: the Green / Green-Jacobi preconditioner and the PCG
// vector updates with hand-written fp64 FFTs (replaces preconditioners.py:
// 83-94, 122-136 and the axpys of solver.py:119-136 on power-of-two grids).
//
// Internal spectrum layout ("axis-0 half spectrum"): spec[c][k0][i1][i2],
// k0 = 0..n0/2 (the real-to-complex axis is the slowest one), full extent on
// the other axes, so the last transform before the Green block solve runs
// along contiguous rows.  Per PCG iteration (d = 3, green-jacobi):
//
//   A   axis-0 R2C of r and s = D^-1/2 r, fused with r -= alpha Kp   (18 U)
//   B   axis-1 complex FFT of the 6 half spectra, in place            (12 U)
//   C   axis-2 FFT + Green block solve + <r,Gr>, <s,Gs> + axis-2 iFFT (13.5 U)
//   B'  axis-1 inverse FFT of the 3 z^ spectra                        ( 6 U)
//   I   axis-0 C2R fused with x += alpha p, p = D^-1/2 z + beta p     (18 U)
//
// (U = 8 N bytes.)  Every pass is one read and one write of its data; the
// forward and inverse transforms along the last axis share one pass with the
// block solve between them.  All passes are predicated on the device PCG
// state, so iterations can be queued / graph-captured without host syncs.
#include "common.cuh"
#include "fft.cuh"

#include <cstdlib>

namespace jfftb {

namespace {

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}

__global__ void twiddle_kernel(double2* tw) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < kTwN) {
    double s, c;
    sincospi(-2.0 * (double)j / (double)kTwN, &s, &c);
    tw[j] = make_double2(c, s);
  }
}
// per-stage tables (fft.cuh tw_stage_off), copied from the 4096 table
__global__ void twiddle_stage_kernel(double2* tw) {
  const int lgP = blockIdx.y, ri = blockIdx.z;
  const int P = 1 << lgP, R = ri == 0 ? 8 : (ri == 1 ? 4 : 2);
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (P < R || P > kTwN) return;
  const int NS = P / R;
  if (e >= (R - 1) * NS) return;
  const int t = e / NS + 1, j = e % NS;
  tw[tw_stage_off(P, R) + e] = tw[(j * (kTwN / P) * t) & (kTwN - 1)];
}

enum FMode { FM_APPLY = FUSED_APPLY, FM_INIT = FUSED_INIT, FM_ITER = FUSED_ITER, FM_QUAD = 3 };

struct FGeom {
  int d, n0, nlast;
  int M0, K0;      // n0 / 2, n0 / 2 + 1 (spectral passes B, C: the k0 rows held here)
  int64_t PS;      // elements per axis-0 plane (= N / n0)
  int64_t CS;      // complex elements per spectral component (= K0 * PS)
  int64_t N;
  int n1;          // d = 3: axis-1 extent
  // spectral-pass addressing (B, C).  Frequency row (k, k1) of field f sits
  // at f FS + (k1 >> sh) SS + k KS + (k1 & (2^sh - 1)) nlast: one segment per
  // source rank of a distributed solve (dist.cu), a single segment (SS = 0,
  // KS = PS, FS = CS) on one GPU.  k0lo: global index of the first k0 row.
  int64_t FS, KS, SS;
  int sh, rsh;     // segment shift; log2(rows per k0 row = PS / nlast)
  int k0lo;
  // pass I: the direction p may live in a halo-extended slab (dist.cu)
  int64_t pN, pPS, poff;
  // batched right-hand sides (pcg_batch): L solves side by side, one PCG
  // state each; vector fields vs doubles and spectra bss complex apart
  int L;
  int64_t vs, bss;
  // passes A and I: components [c0, c0 + nc) of this launch (dist.cu runs them
  // component by component to overlap the all-to-all with the next one)
  int c0, nc;
  __device__ __forceinline__ int64_t row_off(int64_t row) const {
    const int64_t k = row >> rsh;
    const int k1 = (int)(row & ((1 << rsh) - 1));
    return (int64_t)(k1 >> sh) * SS + k * KS + (int64_t)(k1 & ((1 << sh) - 1)) * nlast;
  }
};

constexpr int tw_a(int M) { return M >= 1024 ? 4 : (M >= 512 ? 8 : 16); }
#ifndef JF_TWB_1024
#define JF_TWB_1024 4
#endif
constexpr int tw_b(int L) { return L >= 2048 ? 4 : (L >= 1024 ? JF_TWB_1024 : 8); }
// one radix-8 butterfly per thread where possible (<= 512 threads)
constexpr int nt_for(int butterflies) {
  return butterflies >= 512 ? 512 : (butterflies <= 64 ? 64 : (butterflies + 31) / 32 * 32);
}

// ---------------------------------------------------------------------------
// pass A: axis-0 real-to-complex of r (and s = D^-1/2 r), fused with the
// residual update r -= alpha Kp (FM_ITER).  F = 1 (green) or 2 (green-jacobi).
// FM_APPLY: src = the vector to precondition (not written), F = 1, s-only when
// `dinv` is given (green-jacobi) else r-only.
// ---------------------------------------------------------------------------
// Tiles are TW = 16 real columns (128-byte row segments: at 2 MB strides
// 64-byte segments reach only ~52% of HBM bandwidth, 128-byte ones ~93%,
// measured).  Each thread owns PE consecutive (row, column) elements; the
// inputs stream straight from global in batches, r' goes straight back, and
// the (up to two) fields are transformed one after the other through one
// packed smem tile, the s field waiting in registers.
// F = 2 holds both packed fields side by side ([k][field][col], 2 TW
// sequences) and transforms them in one pass: 1024 threads, one CTA per SM.
constexpr int passA_nt(int M, int F, int TW) {
  return F == 2 ? (2 * TW * M / 8 >= 1024 ? 1024 : nt_for(2 * TW * M / 8)) : nt_for(TW * M / 8);
}

template <int M, int F, int MODE, int TW>
__global__ void __launch_bounds__(passA_nt(M, F, TW),
                                  passA_nt(M, F, TW) <= 512 && 16 * F * TW * M <= 110 * 1024 ? 2 : 1)
    passA(FGeom g, const PcgState* __restrict__ st, double* __restrict__ r,
          const double* __restrict__ kp, const double* __restrict__ dinv,
          double2* __restrict__ spec, const double2* __restrict__ tw) {
  constexpr int NT = passA_nt(M, F, TW);
  constexpr int FTW = F * TW;       // sequences of the packed tile
  constexpr int RAWN = 2 * M * TW;  // real elements of one field's tile
  constexpr int PE = RAWN / NT, CH = PE < 8 ? PE : 8;
  static_assert(PE * NT == RAWN && PE % CH == 0, "pass A tiling");
  static_assert(F == 1 || MODE != FM_APPLY, "APPLY transforms one field");
  extern __shared__ double2 sbuf[];  // packed tile [k][field][col], k < M
  // component; right-hand side (fastest block index: the L solves' CTAs of a
  // tile run together and share its D^-1/2 reads through L2)
  const int c = g.c0 + blockIdx.y, bl = blockIdx.x % g.L;
  const int64_t tile = blockIdx.x / g.L;
  if (st) st += bl;
  r += bl * g.vs;
  if (kp) kp += bl * g.vs;
  spec += bl * g.bss;
  if (MODE != FM_APPLY && st->done) return;
  const int64_t col0 = tile * TW;
  const double alpha = MODE == FM_ITER ? st->alpha : 0.0;
  double* rc = r + c * g.N + col0;
  const double* kc = kp ? kp + c * g.N + col0 : nullptr;
  const double* dc = dinv ? dinv + c * g.N + col0 : nullptr;
  double* pk = reinterpret_cast<double*>(sbuf);
  const bool use_k = MODE == FM_ITER;
  const bool use_d = MODE == FM_APPLY ? dc != nullptr : F == 2;
#pragma unroll
  for (int j0 = 0; j0 < PE; j0 += CH) {
    double a[CH], kv[CH], dv[CH];
#pragma unroll
    for (int j = 0; j < CH; ++j) {
      const int e = threadIdx.x + (j0 + j) * NT;
      const int64_t gi = (int64_t)(e / TW) * g.PS + (e % TW);
      a[j] = rc[gi];
      if (use_k) kv[j] = kc[gi];
      if (use_d) dv[j] = __ldg(dc + gi);
    }
#pragma unroll
    for (int j = 0; j < CH; ++j) {
      const int e = threadIdx.x + (j0 + j) * NT;
      const int i0 = e / TW, col = e % TW;
      double xv = a[j];
      if (use_k) {
        xv = xv - alpha * kv[j];
        rc[(int64_t)i0 * g.PS + col] = xv;
      }
      // packed complex tile: row i0 = 2m + h is Re (h = 0) / Im (h = 1) of z[m]
      double* row = pk + (size_t)(i0 >> 1) * FTW * 2 + (i0 & 1);
      if (F == 2) {
        row[col * 2] = xv;
        row[(TW + col) * 2] = dv[j] * xv;  // s = D^-1/2 r'
      } else {
        row[col * 2] = (MODE == FM_APPLY && use_d) ? dv[j] * xv : xv;
      }
    }
  }
  __syncthreads();
  cta_fft<M, FTW, NT, false>(sbuf, FTW, 1, tw);
  // unpack the packed half-length transforms into X[k], k = 0..M, pairwise:
  // X[k] and X[M-k] come from the same two entries z[k], z[M-k] (k = 0
  // pairs with the Nyquist row M), so each entry is read once
  constexpr int TWS = kTwN / (2 * M);
  auto unpack = [&](double2 zk, double2 zc, int k) {
    const double2 fe = cscale(cadd(zk, zc), 0.5);
    const double2 fo = cscale(csub(zk, zc), 0.5);                   // = i Fo
    const double2 w = __ldg(tw + ((k * TWS) & (kTwN - 1)));         // e^{-2 pi i k / n0}
    return cadd(fe, cmul(w, mul_mi<false>(fo)));                    // Fe + w Fo
  };
  for (int e = threadIdx.x; e < (M / 2 + 1) * FTW; e += NT) {
    const int k = e / FTW, q = e % FTW;
    const int f = q / TW, col = q % TW;
    const int kc = M - k;
    const double2 za = sbuf[k * FTW + q];
    const double2 zb = sbuf[(kc % M) * FTW + q];
    double2* out = spec + (f * g.d + c) * g.CS + col0 + col;
    out[(int64_t)k * g.PS] = unpack(za, cconj(zb), k);
    if (kc != k) out[(int64_t)kc * g.PS] = unpack(zb, cconj(za), kc);
  }
}

// ---------------------------------------------------------------------------
// pass A, green-jacobi (F = 2) INIT / ITER with the first transform stage in
// registers: thread (col, j) loads exactly the 2 R0 real rows its stage-0
// radix-R0 butterfly needs (packed entries j + Q0 t) for both fields, so the
// tile is never staged through shared memory before the transform and the
// remaining stages run in place (DIF, one barrier each).  The unpack reads
// the digit-reversed slots (fft.cuh dif_pos).  Same tile, same traffic.
// ---------------------------------------------------------------------------
template <int M>
constexpr int passA3_nt() { return tw_a(M) * (M / fft_radix(M, 0)); }
template <int M>
constexpr bool passA3_ok() { return passA3_nt<M>() >= 64 && passA3_nt<M>() <= 1024; }

template <int M, int MODE, bool FL>
__global__ void __launch_bounds__(passA3_nt<M>(), 1)
    passA3(FGeom g, const PcgState* __restrict__ st, double* __restrict__ r,
           const double* __restrict__ kp, const double* __restrict__ dinv,
           double2* __restrict__ spec, const double2* __restrict__ tw) {
  constexpr int TW = tw_a(M);
  constexpr int FTW = 2 * TW;         // sequences: [field][col]
  constexpr int NT = passA3_nt<M>();
  constexpr int R0 = fft_radix(M, 0);
  constexpr int Q0 = M / R0;
  static_assert(MODE == FM_ITER || MODE == FM_INIT, "pass A3 runs the PCG modes");
  extern __shared__ double2 sbuf[];   // [m][field][col]
  // component; right-hand side (fastest block index: the L solves' CTAs of a
  // tile run together and share its D^-1/2 reads through L2)
  const int c = g.c0 + blockIdx.y, bl = blockIdx.x % g.L;
  const int64_t tile = blockIdx.x / g.L;
  st += bl;
  r += bl * g.vs;
  kp += bl * g.vs;
  spec += bl * g.bss;
  if (st->done) return;
  const int64_t col0 = tile * TW;
  const double alpha = MODE == FM_ITER ? st->alpha : 0.0;
  const int col = threadIdx.x % TW, j = threadIdx.x / TW;
  double* rc = r + c * g.N + col0 + col;
  const double* kc = kp + c * g.N + col0 + col;
  const double* dc = dinv + c * g.N + col0 + col;
  double a[R0][2], kv[R0][2], dv[R0][2];
#pragma unroll
  for (int t = 0; t < R0; ++t)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t gi = (int64_t)(2 * (j + Q0 * t) + h) * g.PS;
      a[t][h] = rc[gi];
      if (MODE == FM_ITER) kv[t][h] = kc[gi];
      dv[t][h] = __ldg(dc + gi);
    }
  double2 v0[8], v1[8];
#pragma unroll
  for (int t = 0; t < R0; ++t) {
    double x[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      x[h] = a[t][h];
      if (MODE == FM_ITER) {
        x[h] = x[h] - alpha * kv[t][h];
        rc[(int64_t)(2 * (j + Q0 * t) + h) * g.PS] = x[h];
      }
    }
    v0[t] = make_double2(x[0], x[1]);
    v1[t] = make_double2(dv[t][0] * x[0], dv[t][1] * x[1]);  // s = D^-1/2 r'
  }
  dftR<R0, false>(v0);
  dftR<R0, false>(v1);
  if constexpr (Q0 > 1) {
    const double2* __restrict__ tws = tw + tw_stage_off(M, R0);
#pragma unroll
    for (int t = 1; t < R0; ++t) {
      const double2 w = __ldg(tws + (t - 1) * Q0 + j);
      v0[t] = cmul(v0[t], w);
      v1[t] = cmul(v1[t], w);
    }
  }
#pragma unroll
  for (int t = 0; t < R0; ++t) {
    sbuf[(j + Q0 * t) * FTW + col] = v0[t];
    sbuf[(j + Q0 * t) * FTW + TW + col] = v1[t];
  }
  __syncthreads();
  constexpr int TWS = kTwN / (2 * M);
  auto unpack = [&](double2 zk, double2 zc, int k) {
    const double2 fe = cscale(cadd(zk, zc), 0.5);
    const double2 fo = cscale(csub(zk, zc), 0.5);                   // = i Fo
    const double2 w = __ldg(tw + ((k * TWS) & (kTwN - 1)));         // e^{-2 pi i k / n0}
    return cadd(fe, cmul(w, mul_mi<false>(fo)));                    // Fe + w Fo
  };
  if constexpr (FL) {
    // last DIF stage (unit stride: butterfly b owns slots RL b .. RL b + RL-1)
    // fused with the unpack.  The mirror frequencies (M - k) mod M of one
    // butterfly all sit in one partner butterfly bp, so a thread transforms
    // the pair (b, bp) in registers and emits every X[k], X[M - k] they
    // hold: two shared-memory passes (last-stage write, unpack read) fewer.
    constexpr int NS = fft_nstages(M);
    constexpr int RL = fft_radix(M, NS - 1);
    static_assert(fft_span(M, NS - 1) == RL, "last DIF stage has unit stride");
    cta_fft_dif_qf_until<M, FTW, NT, 1, NS - 1>(sbuf, FTW, tw);
    constexpr int NB = M / RL;
    for (int e = threadIdx.x; e < NB * FTW; e += NT) {
      const int b = e / FTW, q = e % FTW;  // warp-uniform b
      const int bp = dif_pos(M, (M - dif_freq(M, RL * b)) % M) / RL;
      if (bp < b) continue;
      double2 u[8], w[8];  // dftR works on 8-slot arrays
#pragma unroll
      for (int t = 0; t < RL; ++t) {
        u[t] = sbuf[(RL * b + t) * FTW + q];
        w[t] = sbuf[(RL * bp + t) * FTW + q];
      }
      dftR<RL, false>(u);
      dftR<RL, false>(w);
      const int f = q / TW, cl = q % TW;
      double2* out = spec + (f * g.d + c) * g.CS + col0 + cl;
      auto emit = [&](const double2 (&x)[8], const double2 (&y)[8], int bx, int by) {
#pragma unroll
        for (int t = 0; t < RL; ++t) {
          const int k = dif_freq(M, RL * bx + t);
          if (2 * k > M) continue;
          const int kc = M - k;
          const int tp = dif_pos(M, kc % M) - RL * by;
          double2 zb = y[0];
#pragma unroll
          for (int s = 1; s < RL; ++s)
            if (s == tp) zb = y[s];
          out[(int64_t)k * g.PS] = unpack(x[t], cconj(zb), k);
          if (kc != k) out[(int64_t)kc * g.PS] = unpack(zb, cconj(x[t]), kc);
        }
      };
      emit(u, w, b, bp);
      if (bp != b) emit(w, u, bp, b);
    }
    return;
  }
  cta_fft_dif_qf<M, FTW, NT, 1>(sbuf, FTW, tw);
  // unpack X[k], k = 0..M, pairwise (k, M - k) from the digit-reversed slots
  for (int e = threadIdx.x; e < (M / 2 + 1) * FTW; e += NT) {
    const int k = e / FTW, q = e % FTW;
    const int f = q / TW, cl = q % TW;
    const int kc = M - k;
    const double2 za = sbuf[dif_pos(M, k) * FTW + q];
    const double2 zb = sbuf[dif_pos(M, kc % M) * FTW + q];
    double2* out = spec + (f * g.d + c) * g.CS + col0 + cl;
    out[(int64_t)k * g.PS] = unpack(za, cconj(zb), k);
    if (kc != k) out[(int64_t)kc * g.PS] = unpack(zb, cconj(za), kc);
  }
}

// ---------------------------------------------------------------------------
// pass B: complex FFT along axis 1 (d = 3), in place, components
// [comp0, comp0 + gridDim.z)
// ---------------------------------------------------------------------------
template <int L, bool INV, bool PRED, bool SEG>
__global__ void __launch_bounds__(nt_for(tw_b(L) * L / 8))
    passB(FGeom g, const PcgState* __restrict__ st, double2* __restrict__ spec, int comp0,
          int ncomp, const double2* __restrict__ tw) {
  constexpr int TW = tw_b(L);
  constexpr int NT = nt_for(TW * L / 8);
  extern __shared__ double2 sbuf[];  // [i1][col]
  const int nlast = g.nlast;
  const int c = comp0 + (int)blockIdx.z, bl = (int)(blockIdx.x % g.L);
  if (st) st += bl;
  spec += bl * g.bss;
  if (PRED && st->done) return;
  const int k0 = blockIdx.y;
  const int64_t col0 = (int64_t)(blockIdx.x / g.L) * TW;
  double2* base = spec + c * g.FS + (int64_t)k0 * g.KS + col0;
  // column col of the tile is sequence col: element i at base + i nlast + col
  // (TW columns = 128-byte row segments), read by the first stage and written
  // by the last straight from/to global memory; SEG: element i at
  // base + (i >> sh) SS + (i & (2^sh - 1)) nlast (per-rank segments)
  cta_fft_io<L, TW, NT, INV, true, 0, true, true, SEG>(sbuf, TW, 1, tw, base, base, 1, nlast,
                                                       g.sh, g.SS);
}

// ---------------------------------------------------------------------------
// pass C: last-axis FFT of every row of the listed spectra, Green block solve
// (z^ = G s^ / N) with the Parseval quadratic forms, inverse last-axis FFT of
// z^, written over the solved spectrum.
//   F = 2 (green-jacobi): rows r^ (comps 0..d-1) and s^ (d..2d-1); q0 = r^H Gt r^,
//                         q1 = s^H G s^; z^ replaces s^.
//   F = 1 (green):        rows r^; q0 = r^H Gt r^, q1 = r^H G r^; z^ replaces r^.
//   APPLY (F = 1):        rows of the input spectrum; z^ replaces it.
// ---------------------------------------------------------------------------
template <int D>
struct HB {
  double dg[D];
  double re[3], im[3];
};
template <int D>
__device__ __forceinline__ HB<D> ld_block(const double* __restrict__ b, int64_t Nh, int64_t f) {
  HB<D> B;
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
template <int D>
__device__ __forceinline__ double hb_apply(const HB<D>& B, const double2 (&s)[D], double2 (&z)[D]) {
#pragma unroll
  for (int a = 0; a < D; ++a) {
    double zr = B.dg[a] * s[a].x, zi = B.dg[a] * s[a].y;
#pragma unroll
    for (int b = 0; b < D; ++b) {
      if (b == a) continue;
      const int lo = a < b ? a : b, hi = a < b ? b : a;
      const int k = lo == 0 ? hi - 1 : 2;
      const double gr = B.re[k];
      const double gi = a < b ? B.im[k] : -B.im[k];
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

// ---------------------------------------------------------------------------
// Analytic Green blocks (3-D).  For the P1 Kuhn split the reference
// operator's symbol is, with E_a = e^{i q_a}, D_a = E_a - 1, h_a = 1/dx_a,
// w = prod(dx)/6 and P_ab = sum_t e^{i q.(o_tb - o_ta)} over the 6 simplices
// (o_ta: low node of simplex t's edge along axis a, common.cuh edge_base),
//   K_aa = 6 w ((lam + mu) h_a^2 |D_a|^2 + mu sum_c h_c^2 |D_c|^2)
//   K_ab = w h_a h_b (lam conj(D_a) D_b P_ab + mu D_a conj(D_b) conj(P_ab))
// (checked against the impulse-response transform of assemble_green,
// preconditioners.py:50-80, to 4e-16 of its scale).  Every block but the DC
// one is nonsingular (a nonzero q leaves some edge difference nonzero), so
// the pseudo-inverse with the 1e-12 eigenvalue cutoff is the inverse, taken
// here by cofactors; DC stays 0.  Pass C evaluates this per frequency instead
// of streaming 4.5 U of stored Green planes: per row-set the q0 / q1 parts
// are folded into a few constants, per frequency it costs ~150 flops.
// ---------------------------------------------------------------------------
struct GreenAna {
  double lam, mu, w, h[3];
};
__device__ __forceinline__ double2 cpow1(double2 e, int v) {
  return v > 0 ? e : (v < 0 ? cconj(e) : make_double2(1.0, 0.0));
}
constexpr int edge_bit(int t, int a, int c) { return (edge_base(3, t, a) >> c) & 1; }
struct GRow {
  double2 c01, d01, c02, d02, c12, d12;
  double2 A[3][3];  // pair (01, 02, 12) x v2 + 1
  double r0, r1;
};
__device__ __forceinline__ GRow green_row(const GreenAna& ga, double2 E0, double2 E1) {
  GRow R;
  const double2 D0 = make_double2(E0.x - 1.0, E0.y), D1 = make_double2(E1.x - 1.0, E1.y);
  R.r0 = ga.h[0] * ga.h[0] * (D0.x * D0.x + D0.y * D0.y);
  R.r1 = ga.h[1] * ga.h[1] * (D1.x * D1.x + D1.y * D1.y);
  const double l01 = ga.w * ga.h[0] * ga.h[1], l02 = ga.w * ga.h[0] * ga.h[2],
               l12 = ga.w * ga.h[1] * ga.h[2];
  R.c01 = cscale(cmul(cconj(D0), D1), ga.lam * l01);
  R.d01 = cscale(cmul(D0, cconj(D1)), ga.mu * l01);
  R.c02 = cscale(cconj(D0), ga.lam * l02);
  R.d02 = cscale(D0, ga.mu * l02);
  R.c12 = cscale(cconj(D1), ga.lam * l12);
  R.d12 = cscale(D1, ga.mu * l12);
#pragma unroll
  for (int pr = 0; pr < 3; ++pr)
#pragma unroll
    for (int v = 0; v < 3; ++v) R.A[pr][v] = make_double2(0.0, 0.0);
#pragma unroll
  for (int pr = 0; pr < 3; ++pr) {
    const int a = pr == 2 ? 1 : 0, b = pr == 0 ? 1 : 2;
#pragma unroll
    for (int t = 0; t < 6; ++t) {
      const int v0 = edge_bit(t, b, 0) - edge_bit(t, a, 0);
      const int v1 = edge_bit(t, b, 1) - edge_bit(t, a, 1);
      const int v2 = edge_bit(t, b, 2) - edge_bit(t, a, 2);
      R.A[pr][v2 + 1] = cadd(R.A[pr][v2 + 1], cmul(cpow1(E0, v0), cpow1(E1, v1)));
    }
  }
  return R;
}
__device__ __forceinline__ HB<3> green_block(const GreenAna& ga, const GRow& R, double2 E2,
                                             bool dc) {
  HB<3> B;
  if (dc) {
#pragma unroll
    for (int k = 0; k < 3; ++k) B.dg[k] = B.re[k] = B.im[k] = 0.0;
    return B;
  }
  const double2 D2 = make_double2(E2.x - 1.0, E2.y);
  const double r2 = ga.h[2] * ga.h[2] * (D2.x * D2.x + D2.y * D2.y);
  const double S = R.r0 + R.r1 + r2, lm = ga.lam + ga.mu, w6 = 6.0 * ga.w;
  const double ka = w6 * (lm * R.r0 + ga.mu * S);
  const double kd = w6 * (lm * R.r1 + ga.mu * S);
  const double kf = w6 * (lm * r2 + ga.mu * S);
  const double2 E2c = cconj(E2);
  auto P = [&](int pr) {
    return cadd(cadd(cmul(R.A[pr][0], E2c), R.A[pr][1]), cmul(R.A[pr][2], E2));
  };
  const double2 P01 = P(0), T02 = cmul(D2, P(1)), T12 = cmul(D2, P(2));
  const double2 kb = cadd(cmul(R.c01, P01), cmul(R.d01, cconj(P01)));
  const double2 kc = cadd(cmul(R.c02, T02), cmul(R.d02, cconj(T02)));
  const double2 ke = cadd(cmul(R.c12, T12), cmul(R.d12, cconj(T12)));
  const double nb = kb.x * kb.x + kb.y * kb.y, nc = kc.x * kc.x + kc.y * kc.y,
               ne = ke.x * ke.x + ke.y * ke.y;
  const double A0 = kd * kf - ne, A1 = ka * kf - nc, A2 = ka * kd - nb;
  const double2 bec = cmul(cmul(kb, ke), cconj(kc));
  const double det = ka * A0 - kd * nc - kf * nb + 2.0 * bec.x;
  const double id = 1.0 / det;
  B.dg[0] = A0 * id;
  B.dg[1] = A1 * id;
  B.dg[2] = A2 * id;
  const double2 g01 = cscale(csub(cmul(kc, cconj(ke)), cscale(kb, kf)), id);
  const double2 g02 = cscale(csub(cmul(kb, ke), cscale(kc, kd)), id);
  const double2 g12 = cscale(csub(cmul(kc, cconj(kb)), cscale(ke, ka)), id);
  B.re[0] = g01.x; B.im[0] = g01.y;
  B.re[1] = g02.x; B.im[1] = g02.y;
  B.re[2] = g12.x; B.im[2] = g12.y;
  return B;
}

// Two CTAs per SM, two radix-8 butterflies per thread per stage.  The rows
// never take a staging trip through shared memory: the first forward stage
// reads its butterfly inputs straight from global memory (coalesced: thread j
// of a sequence takes elements j + t L/8) and the last inverse stage writes
// straight back, so a row-set costs two shared-memory round trips per
// transform instead of four.  The Green planes of the next row-set are copied
// to shared memory with cp.async while the current inverse transform runs.
constexpr int CPAD = 8;  // one padding slot every 8 elements of a row
// Green planes staged in smem (GS) or read straight from global in the solve
// (measured at 512^3: staged 3.69 ms, direct 4.19 ms)
constexpr bool kGStage = true;
// GS: 0 Green planes read from global in the solve, 1 bulk-staged in shared
// memory, 2 evaluated analytically (3-D, green_block)
constexpr int passC_gp(int D, int GS) { return GS == 1 ? (D == 2 ? 4 : 9) : 0; }
#ifndef JF_PC_NTDIV
#define JF_PC_NTDIV 16
#endif
constexpr int passC_nt(int D, int L, int F) { return nt_for(F * D * L / JF_PC_NTDIV); }
constexpr int passC_bufd(int D, int L, int F, int GS = 1) {
  return F * D * padded_len<CPAD>(L) * 2 + passC_gp(D, GS) * L;
}
// resident CTAs per SM the launch bounds aim for (capped by shared memory).
// Double buffering the rows (next row-set in flight during this one's
// transforms) was measured slower at 512^3 (6.6 ms vs 5.7 ms): it halves the
// resident CTAs.
#ifndef JF_CA_MINB
#define JF_CA_MINB 2
#endif
constexpr int passC_minb(int D, int L, int F, int GS = 1) {
  return GS == 2 ? JF_CA_MINB
                 : passC_bufd(D, L, F, GS) * 8 <= 72 * 1024 ? 3
                                                   : (passC_bufd(D, L, F, GS) * 8 <= 110 * 1024 ? 2 : 1);
}

template <int D, int L, int F, int MODE, int GS, bool IP>
__global__ void __launch_bounds__(passC_nt(D, L, F), passC_minb(D, L, F, GS))
    passC(FGeom g, const PcgState* __restrict__ st, const double* __restrict__ gpc,
          const double* __restrict__ gterm, double2* __restrict__ spec,
          double* __restrict__ partials, const double2* __restrict__ tw, GreenAna ga) {
  static_assert(GS != 2 || D == 3, "analytic Green blocks are 3-D");
  constexpr int NQ = F * D;  // rows held per frequency row
  constexpr int NT = passC_nt(D, L, F);
  constexpr int RL = padded_len<CPAD>(L);
  constexpr int GP = passC_gp(D, GS);            // Green planes staged with the rows
  constexpr int BUFD = passC_bufd(D, L, F, GS);  // doubles of shared memory
  static_assert(BUFD == NQ * RL * 2 + GP * L, "buffer layout");
  // [ rows: NQ x RL double2 | Green planes: GP x L double ]
  extern __shared__ double2 sbuf[];
  __shared__ double red[64];
  // right-hand side = fastest block index: the L CTAs working on a row-set
  // run together and share its Green planes through L2
  const int bl = blockIdx.x % g.L, bx = blockIdx.x / g.L, nbx = gridDim.x / g.L;
  if (st) st += bl;
  spec += bl * g.bss;
  if (partials) partials += 2 * (int64_t)nbx * bl;
  if (MODE != FM_APPLY && st->done) return;
  static_assert(MODE != FM_QUAD || F == 1, "quad-only pass holds one spectrum");
  const double invN = 1.0 / (double)g.N;
  const int64_t rows = g.CS / L;
  const int64_t Nh = g.CS;
  double q0 = 0.0, q1 = 0.0;
  constexpr int ZQ = F == 2 ? D : 0;  // first row of the solved spectrum
  double* gsm = reinterpret_cast<double*>(sbuf + NQ * RL);
  // the Green planes of a row-set (GP contiguous L-double runs) arrive by
  // bulk copies issued by one thread and complete on gbar
  __shared__ uint64_t gbar;
  unsigned gphase = 0;
  if (GS == 1 && threadIdx.x == 0) mbar_init(&gbar, 1);
  __syncthreads();
  auto prefetch_green = [&](int64_t row) {
    if (GS != 1 || threadIdx.x != 0) return;
    const int64_t rbase = row * L;
    fence_proxy_async();  // the previous row-set's reads of gsm come first
    mbar_expect_tx(&gbar, GP * L * sizeof(double));
#pragma unroll 1
    for (int p = 0; p < GP; ++p)
      bulk_g2s(gsm + p * L, gpc + p * Nh + rbase, L * sizeof(double), &gbar);
  };
  int64_t row = bx;
  if (row < rows) prefetch_green(row);
  for (; row < rows; row += nbx) {
    const int64_t rbase = row * L;        // Green planes: rows back to back
    const int64_t sbase = g.row_off(row);  // spectra: (segmented) row address
    const int k0 = g.k0lo + (int)(row >> g.rsh);
    const double w = (k0 == 0 || 2 * k0 == g.n0) ? 1.0 : 2.0;
    // forward: global rows -> (stage 1) -> shared; barrier-separated from the
    // previous row-set's last shared-memory reads by the loop-end barrier
    if constexpr (IP)
      cta_fft_dif<L, NQ, NT, CPAD, true>(sbuf, RL, tw, spec + sbase, g.FS);
    else
      cta_fft_io<L, NQ, NT, false, false, CPAD, true, false>(sbuf, 1, RL, tw, spec + sbase,
                                                             nullptr, g.FS, 1);
#ifndef JF_NO_PREFETCH
    // the next row-set's rows into L2 while this one is solved and inverted
    if (threadIdx.x < NQ && row + nbx < rows)
      bulk_prefetch_l2(spec + threadIdx.x * g.FS + g.row_off(row + nbx),
                       L * sizeof(double2));
#endif
    if (GS == 1) mbar_wait(&gbar, gphase);  // this row-set's Green planes
    gphase ^= 1;
    __syncthreads();
    GRow grow;
    bool dcrow = false;  // the row holding the zero frequency
    if constexpr (GS == 2) {
      const int k1 = (int)(row & ((1 << g.rsh) - 1));
      grow = green_row(ga, cconj(__ldg(tw + ((k0 * (kTwN / g.n0)) & (kTwN - 1)))),
                       cconj(__ldg(tw + ((k1 * (kTwN / g.n1)) & (kTwN - 1)))));
      dcrow = k0 == 0 && k1 == 0;
    }
#pragma unroll 1
    for (int k = threadIdx.x; k < L; k += NT) {
      const int64_t f = rbase + k;
      HB<D> B;
      if constexpr (GS == 2) {
        const int k2 = IP ? dif_freq(L, k) : k;
        B = green_block(ga, grow, cconj(__ldg(tw + ((k2 * (kTwN / L)) & (kTwN - 1)))),
                        dcrow && k2 == 0);
      } else if constexpr (GS == 1) {
#pragma unroll
        for (int a = 0; a < D; ++a) B.dg[a] = gsm[a * L + k];
#pragma unroll
        for (int o = 0; o < (D == 2 ? 1 : 3); ++o) {
          B.re[o] = gsm[(D + 2 * o) * L + k];
          B.im[o] = gsm[(D + 2 * o + 1) * L + k];
        }
      } else {
        B = ld_block<D>(gpc, Nh, f);
      }
      double2 s[D], z[D];
#pragma unroll
      for (int a = 0; a < D; ++a) s[a] = sbuf[(ZQ + a) * RL + pidx<CPAD>(k)];
      const double qs = hb_apply<D>(B, s, z);
      if (MODE == FM_QUAD) {
        q0 += w * qs;  // gpc is the termination operator here
      } else if (MODE != FM_APPLY) {
        if (F == 2) {
          double2 rr[D], tmp[D];
#pragma unroll
          for (int a = 0; a < D; ++a) rr[a] = sbuf[a * RL + pidx<CPAD>(k)];
          const double qr = (gterm == gpc) ? hb_apply<D>(B, rr, tmp)
                                           : hb_apply<D>(ld_block<D>(gterm, Nh, f), rr, tmp);
          q0 += w * qr;
          q1 += w * qs;
        } else {
          q1 += w * qs;
          if (gterm == gpc) {
            q0 += w * qs;
          } else {
            double2 tmp[D];
            q0 += w * hb_apply<D>(ld_block<D>(gterm, Nh, f), s, tmp);
          }
        }
      }
      if (MODE != FM_QUAD)
#pragma unroll
        for (int a = 0; a < D; ++a) sbuf[(ZQ + a) * RL + pidx<CPAD>(k)] = cscale(z[a], invN);
    }
    __syncthreads();  // block solve done: Green planes and r^ rows are free
    if (row + nbx < rows) prefetch_green(row + nbx);
    if (MODE != FM_QUAD) {
      if constexpr (IP)
        cta_fft_dit_inv<L, D, NT, CPAD, true>(sbuf + ZQ * RL, RL, tw, spec + ZQ * g.FS + sbase,
                                              g.FS);
      else
        cta_fft_io<L, D, NT, true, false, CPAD, false, true>(sbuf + ZQ * RL, 1, RL, tw, nullptr,
                                                             spec + ZQ * g.FS + sbase, g.FS, 1);
    }
    __syncthreads();
  }
  if (MODE != FM_APPLY) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    q0 = warp_sum(q0 * invN);
    q1 = warp_sum(q1 * invN);
    if (lane == 0) { red[wid] = q0; red[32 + wid] = q1; }
    __syncthreads();
    if (wid == 0) {
      double a = lane < NT / 32 ? red[lane] : 0.0, b = lane < NT / 32 ? red[32 + lane] : 0.0;
      a = warp_sum(a);
      b = warp_sum(b);
      if (lane == 0) {
        partials[2 * bx] = a;
        partials[2 * bx + 1] = b;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// passes B, C and B' merged into one persistent kernel (3-D, one solve,
// n1 == n2): the axis-1 transform of a k0-plane, the axis-2 transform / Green
// block solve / inverse of its rows and the inverse axis-1 transform of its
// z^ fields run back to back while the plane is still in L2 (one plane of
// six fields is 24 MiB at 512^2; the 126 MB L2 holds the planes in flight),
// so the spectra cross HBM once on the way in and z^ once on the way out
// instead of three round trips: 16.5 U of DRAM traffic instead of 31.5 U for
// the three passes (green-jacobi, incl. 4.5 U of Green planes and 3 U of
// write-back of the transformed r^ rows).
//
// Work items, claimed in order from a global ticket counter by the resident
// CTAs; stage s = 0 .. K0 holds, in this order,
//   Cr(s-1)  one r^ row-set (3 rows) of plane s-1: axis-2 transform and the
//            termination form r^H Gt r^            (green-jacobi only)
//   Cs(s-1)  one s^ row-set: axis-2 transform, z^ = G s^ / N, s^H G s^,
//            inverse axis-2 transform, z^ written over s^
//   B(s)     one (field, 8-column tile) axis-1 transform of plane s,
//            r^ fields first
//   B'(s-1)  one (z^ component, tile) inverse axis-1 transform of plane s-1
// so a plane's rows are re-read after a few tens of MiB of other traffic.
// Every item is at most 64.5 KB of shared memory and 192 threads: three fit
// an SM.  The axis-1 transforms run in place (DIF forward, DIT inverse), so
// between B and B' the rows of a plane sit in digit-reversed k1 order; a row
// item looks its Green planes up at the true k1 = dif_freq(position).
// Cr(k) / Cs(k) wait until the r^ / s^ tiles of B(k) have signalled
// (per-plane counters, release reduction / acquire load at gpu scope), B'(k)
// until all Cs(k) have.  A waiting CTA only ever waits on items with smaller
// tickets, which running CTAs hold, so the schedule cannot deadlock whatever
// the residency; by the time a dependent item is claimed its producers were
// claimed a few hundred tickets earlier.  Rows written during the launch are
// read with L2 loads (ld.cg).  Every row item writes its own Parseval
// partial: the sums stay in a fixed order (bitwise deterministic) although
// the item -> CTA map is not.
// ---------------------------------------------------------------------------
#ifndef JF_BCB_NT
#define JF_BCB_NT 192
#endif
constexpr int BCB_NT = JF_BCB_NT;
constexpr int bcb_bufd(int L) {  // doubles: 3 padded rows + 9 Green planes, or one tile
  return 3 * padded_len<CPAD>(L) * 2 + 9 * L > 2 * tw_b(L) * L ? 3 * padded_len<CPAD>(L) * 2 + 9 * L
                                                                : 2 * tw_b(L) * L;
}
constexpr int bcb_minb(int L) {
  return bcb_bufd(L) * 8 <= 72 * 1024 ? 3 : (bcb_bufd(L) * 8 <= 110 * 1024 ? 2 : 1);
}
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// one in-place stage of the axis-1 transform of a [L][TW] tile (element e of
// column q at buf[e * TW + q], in global memory at base + e * gks + q;
// consecutive threads take consecutive columns: 128-byte row segments).
// Forward DIF: stage 0 reads global, the last stage writes global; inverse
// DIT: stage nstages-1 reads global, stage 0 writes global.
template <int L, int TW, int NT, bool INV, int S>
__device__ __forceinline__ void tile_ip_stage(double2* buf, const double2* __restrict__ tw,
                                              double2* base, int64_t gks) {
  constexpr int NS = fft_nstages(L);
  constexpr int R = fft_radix(L, S);
  constexpr int P = fft_span(L, S);
  constexpr int Q = P / R;
  constexpr int B = TW * (L / R);
  constexpr bool FIRST = INV ? S == NS - 1 : S == 0;  // reads global
  constexpr bool LAST = INV ? S == 0 : S == NS - 1;   // writes global
  const double2* __restrict__ tws = tw + tw_stage_off(P, R);
#pragma unroll 1
  for (int b = threadIdx.x; b < B; b += NT) {
    const int q = b % TW, bb = b / TW;
    const int j = bb % Q;
    const int e0 = (bb / Q) * P + j;
    double2 v[8];
    if constexpr (FIRST) {
#pragma unroll
      for (int t = 0; t < R; ++t) v[t] = __ldcg(base + (int64_t)(e0 + Q * t) * gks + q);
    } else {
#pragma unroll
      for (int t = 0; t < R; ++t) v[t] = buf[(e0 + Q * t) * TW + q];
    }
    if (INV && Q > 1) {
#pragma unroll
      for (int t = 1; t < R; ++t) v[t] = cmulc(v[t], __ldg(tws + (t - 1) * Q + j));
    }
    dftR<R, INV>(v);
    if (!INV && Q > 1) {
#pragma unroll
      for (int t = 1; t < R; ++t) v[t] = cmul(v[t], __ldg(tws + (t - 1) * Q + j));
    }
    if constexpr (LAST) {
#pragma unroll
      for (int t = 0; t < R; ++t) base[(int64_t)(e0 + Q * t) * gks + q] = v[t];
    } else {
#pragma unroll
      for (int t = 0; t < R; ++t) buf[(e0 + Q * t) * TW + q] = v[t];
    }
  }
  if constexpr (!LAST) __syncthreads();
}
template <int L, int TW, int NT, int S = 0>
__device__ __forceinline__ void tile_fft_dif(double2* buf, const double2* __restrict__ tw,
                                             double2* base, int64_t gks) {
  if constexpr (S < fft_nstages(L)) {
    tile_ip_stage<L, TW, NT, false, S>(buf, tw, base, gks);
    tile_fft_dif<L, TW, NT, S + 1>(buf, tw, base, gks);
  }
}
template <int L, int TW, int NT, int S = fft_nstages(L) - 1>
__device__ __forceinline__ void tile_fft_dit_inv(double2* buf, const double2* __restrict__ tw,
                                                 double2* base, int64_t gks) {
  if constexpr (S >= 0) {
    tile_ip_stage<L, TW, NT, true, S>(buf, tw, base, gks);
    tile_fft_dit_inv<L, TW, NT, S - 1>(buf, tw, base, gks);
  }
}

template <int L, int F>
__global__ void __launch_bounds__(BCB_NT, bcb_minb(L))
    passBCB(FGeom g, const PcgState* __restrict__ st, const double* __restrict__ gpc,
            const double* __restrict__ gterm, double2* __restrict__ spec,
            double* __restrict__ partials, const double2* __restrict__ tw,
            unsigned* __restrict__ q) {
  constexpr int D = 3, NT = BCB_NT;
  constexpr int TW = tw_b(L), NTILE = L / TW;
  constexpr int RL = padded_len<CPAD>(L);
  constexpr int GP = 9;
  constexpr int ZQ = F == 2 ? D : 0;  // first field of the solved spectrum
  static_assert(fft_nstages(L) >= 2, "axis-1 tiles need two stages");
  extern __shared__ double2 sbuf[];
  __shared__ double red[32];
  __shared__ uint64_t gbar;
  __shared__ unsigned s_ticket;
  if (st->done) return;
  const int K = g.K0;
  const unsigned nR = (unsigned)(g.PS / L);          // rows of a plane
  const unsigned nCr = F == 2 ? nR : 0, nCs = nR;
  const unsigned nB = F * D * NTILE, nBi = D * NTILE;
  const unsigned per = nCr + nCs + nB + nBi, total = (unsigned)(K + 1) * per;
  unsigned* cntBr = q + 2;      // r^ tiles of plane k transformed (F = 2)
  unsigned* cntBs = cntBr + K;  // tiles of the solved fields transformed
  unsigned* cntC = cntBs + K;   // solved row-sets of plane k written
  const double invN = 1.0 / (double)g.N;
  const int64_t Nh = g.CS;
  double* gsm = reinterpret_cast<double*>(sbuf + D * RL);
  unsigned gphase = 0;
  if (threadIdx.x == 0) mbar_init(&gbar, 1);
  // all of a producer item's stores, then (thread 0) a release reduction:
  // nobody waits for its round trip
  auto signal = [&](unsigned* cnt) {
    __syncthreads();
    if (threadIdx.x == 0)
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;\n" ::"l"(cnt) : "memory");
  };
  // (the spin bound is a bug guard, not a path: q[1] reports it)
  auto wait_for = [&](const unsigned* cnt, unsigned need) {
    if (threadIdx.x == 0) {
      unsigned spins = 0;
      while (ld_acquire_u32(cnt) < need) {
        __nanosleep(32);
        if (++spins > (1u << 24)) {
          atomicExch(q + 1, 1u);
          break;
        }
      }
    }
    __syncthreads();
  };
  // the Green planes of frequency row (k, k1) -> shared memory (bulk copies)
  auto fetch_green = [&](const double* gp, int64_t grow) {
    if (threadIdx.x == 0) {
      fence_proxy_async();  // earlier generic accesses of the buffer come first
      mbar_expect_tx(&gbar, GP * L * sizeof(double));
#pragma unroll 1
      for (int p = 0; p < GP; ++p)
        bulk_g2s(gsm + p * L, gp + p * Nh + grow * L, L * sizeof(double), &gbar);
    }
  };
  auto load_block = [&](int kk) {
    HB<D> B;
#pragma unroll
    for (int a = 0; a < D; ++a) B.dg[a] = gsm[a * L + kk];
#pragma unroll
    for (int oo = 0; oo < 3; ++oo) {
      B.re[oo] = gsm[(D + 2 * oo) * L + kk];
      B.im[oo] = gsm[(D + 2 * oo + 1) * L + kk];
    }
    return B;
  };
  // fixed-order block sum (warp tree, then warps in order) -> *out by thread 0
  auto block_partial = [&](double v, double* out) {
    v = warp_sum(v * invN);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
      double a = 0.0;
#pragma unroll
      for (int i = 0; i < NT / 32; ++i) a += red[i];
      *out = a;
    }
  };
  // the next ticket is drawn while the current item runs
  unsigned next = 0;
  if (threadIdx.x == 0) next = atomicAdd(q, 1u);
  for (;;) {
    __syncthreads();  // the previous item is done with s_ticket and the buffer
    if (threadIdx.x == 0) s_ticket = next;
    __syncthreads();
    const unsigned t = s_ticket;
    if (t >= total) break;
    if (threadIdx.x == 0) next = atomicAdd(q, 1u);
    const int s = (int)(t / per);
    unsigned o = t % per;
    if (o < nCr + nCs) {
      // ---- a row-set of plane s - 1 (position pr along axis 1 holds k1)
      const int k = s - 1;
      if (k < 0) continue;
      const bool solve = o >= nCr;  // Cs; else Cr (termination form only)
      const unsigned pr = solve ? o - nCr : o;
      const int k1 = dif_freq(L, (int)pr);
      const int64_t row = (int64_t)k * nR + pr;
      const int k0 = g.k0lo + k;
      const double w = (k0 == 0 || 2 * k0 == g.n0) ? 1.0 : 2.0;
      const int fq = solve ? ZQ : 0;  // first field of the row-set
      fetch_green(solve ? gpc : gterm, (int64_t)k * nR + k1);
      wait_for((solve || F == 1) ? cntBs + k : cntBr + k, D * NTILE);
      cta_fft_dif<L, D, NT, CPAD, true>(sbuf, RL, tw, spec + fq * g.FS + row * L, g.FS);
      mbar_wait(&gbar, gphase);
      gphase ^= 1;
      double q0 = 0.0, q1 = 0.0;
#pragma unroll 1
      for (int kk = threadIdx.x; kk < L; kk += NT) {
        const HB<D> B = load_block(kk);
        double2 sv[D], z[D];
#pragma unroll
        for (int a = 0; a < D; ++a) sv[a] = sbuf[a * RL + pidx<CPAD>(kk)];
        const double qs = hb_apply<D>(B, sv, z);
        if (!solve) {
          q0 += w * qs;
        } else {
          q1 += w * qs;
          if (F == 1) {
            if (gterm == gpc) {
              q0 += w * qs;
            } else {
              double2 tmp[D];
              q0 += w * hb_apply<D>(ld_block<D>(gterm, Nh, ((int64_t)k * nR + k1) * L + kk), sv,
                                    tmp);
            }
          }
#pragma unroll
          for (int a = 0; a < D; ++a) sbuf[a * RL + pidx<CPAD>(kk)] = cscale(z[a], invN);
        }
      }
      if (!solve) {
        block_partial(q0, partials + 2 * row);
      } else {
        if (F == 1) {
          block_partial(q0, partials + 2 * row);
          __syncthreads();  // red is reused
        }
        block_partial(q1, partials + 2 * row + 1);  // (its barrier: z^ rows complete)
        cta_fft_dit_inv<L, D, NT, CPAD, true>(sbuf, RL, tw, spec + ZQ * g.FS + row * L, g.FS);
        signal(cntC + k);
      }
    } else if (o < nCr + nCs + nB) {
      // ---- B(s): axis-1 transform of (field c, column tile) of plane s
      const int k = s;
      if (k >= K) continue;
      o -= nCr + nCs;
      const int c = (int)(o / NTILE), tile = (int)(o % NTILE);
      double2* base = spec + c * g.FS + (int64_t)k * g.KS + (int64_t)tile * TW;
      tile_fft_dif<L, TW, NT>(sbuf, tw, base, g.nlast);
      signal((F == 2 && c < D) ? cntBr + k : cntBs + k);
    } else {
      // ---- B'(s-1): inverse axis-1 transform of (z^ component, tile) of plane s - 1
      const int k = s - 1;
      if (k < 0) continue;
      o -= nCr + nCs + nB;
      const int c = ZQ + (int)(o / NTILE), tile = (int)(o % NTILE);
      wait_for(cntC + k, nR);
      double2* base = spec + c * g.FS + (int64_t)k * g.KS + (int64_t)tile * TW;
      tile_fft_dit_inv<L, TW, NT>(sbuf, tw, base, g.nlast);
    }
  }
}

// ---------------------------------------------------------------------------
// pass I: axis-0 complex-to-real of z^ fused with the PCG direction update.
//   FM_ITER:  if alpha is valid: x += alpha p ; unless done: p = Dz + beta p
//   FM_INIT:  p = Dz
//   FM_APPLY: out = Dz           (D = D^-1/2 for green-jacobi, identity for green)
// ---------------------------------------------------------------------------
// pass I tile width (columns): its tile holds one field, so at M = 512
// (n0 = 1024: the per-rank slabs of the 1024^3 multi-GPU configuration) it
// keeps 16 columns (128-byte row segments, one 131 KB tile per SM) where pass
// A's two-field tile only fits 8 -- measured on a (1024, 256, 512) grid: pass
// I 5.57 -> 3.86 ms, the iteration 21.07 -> 20.02 ms; at M = 1024 (2-D
// 2048^2) 8 columns measured no better than 4
#ifndef JF_TWI_512
#define JF_TWI_512 16
#endif
#ifndef JF_TWI_1024
#define JF_TWI_1024 4
#endif
constexpr int tw_i(int M) { return M >= 1024 ? JF_TWI_1024 : (M >= 512 ? JF_TWI_512 : 16); }
constexpr int passI_nt(int M) { return nt_for(tw_i(M) * M / 4); }
// two resident CTAs per SM where the tile fits twice (register cap 64)
constexpr int passI_minb(int M) {
  return 2 * (size_t)16 * tw_i(M) * (M + 1) <= 200 * 1024 && passI_nt(M) >= 512 ? 2 : 1;
}

template <int M, int MODE>
__global__ void __launch_bounds__(passI_nt(M), passI_minb(M))
    passI(FGeom g, const PcgState* __restrict__ st, const double2* __restrict__ zspec,
          const double* __restrict__ dinv, double* __restrict__ p, double* __restrict__ x,
          double* __restrict__ out, const double2* __restrict__ tw) {
  constexpr int TW = tw_i(M);
  constexpr int NT = passI_nt(M);
  extern __shared__ double2 sbuf[];  // [k][col], k <= M
  // component; right-hand side (fastest block index: the L solves' CTAs of a
  // tile run together and share its D^-1/2 reads through L2)
  const int c = g.c0 + blockIdx.y, bl = blockIdx.x % g.L;
  const int64_t tile = blockIdx.x / g.L;
  if (st) st += bl;
  zspec += bl * g.bss;
  if (p) p += bl * g.vs;
  if (x) x += bl * g.vs;
  if (MODE == FM_ITER && !st->xupd) return;
  if (MODE == FM_INIT && st->done) return;
  const int64_t col0 = tile * TW;
  const double2* zc = zspec + c * g.CS + col0;
  for (int e = threadIdx.x; e < (M + 1) * TW; e += NT) {
    const int k = e / TW, col = e % TW;
    cpa16(sbuf + e, zc + (int64_t)k * g.PS + col);
  }
  cpa_commit();
  constexpr int RAWN = 2 * M * TW;  // real elements of the tile
  const bool use_d = dinv != nullptr;
  const int64_t cbase = c * g.N + col0;
  const int64_t pbase = c * g.pN + g.poff + col0;
  cpa_wait<0>();
  __syncthreads();
  // Z'[k] = (X[k] + conj X[M-k]) + i e^{+2 pi i k / n0} (X[k] - conj X[M-k]),
  // computed pairwise (k, M-k) in place; k = 0 pairs with the Nyquist row M
  constexpr int TWS = kTwN / (2 * M);
  for (int e = threadIdx.x; e < (M / 2 + 1) * TW; e += NT) {
    const int k = e / TW, col = e % TW;
    const int kc = M - k;
    const double2 xa = sbuf[k * TW + col], xb = sbuf[kc * TW + col];
    const double2 wa = cconj(__ldg(tw + ((k * TWS) & (kTwN - 1))));
    const double2 wb = cconj(__ldg(tw + ((kc * TWS) & (kTwN - 1))));
    const double2 za = cadd(cadd(xa, cconj(xb)), mul_mi<true>(cmul(wa, csub(xa, cconj(xb)))));
    const double2 zb = cadd(cadd(xb, cconj(xa)), mul_mi<true>(cmul(wb, csub(xb, cconj(xa)))));
    sbuf[k * TW + col] = za;
    if (kc != M && kc != k) sbuf[kc * TW + col] = zb;
  }
  __syncthreads();
  cta_fft<M, TW, NT, true>(sbuf, TW, 1, tw);
  const bool done = MODE == FM_ITER ? (st->done != 0) : false;
  const double alpha = MODE == FM_ITER ? st->alpha : 0.0;
  const double beta = MODE == FM_ITER ? st->beta : 0.0;
  // consecutive threads -> consecutive (row, column): 128-byte row segments;
  // row i0 = 2m + h is the real (h = 0) / imaginary (h = 1) part of z[m].
  // D, p, x are loaded in batches of CH elements ahead of their use.
  const double* zr = reinterpret_cast<const double*>(sbuf);
  constexpr int PE = RAWN / NT, CH = PE < 4 ? PE : 4;
  static_assert(PE * NT == RAWN && PE % CH == 0, "pass I tiling");
#pragma unroll 1
  for (int j0 = 0; j0 < PE; j0 += CH) {
    double dv[CH], pv[CH], xv[CH];
#pragma unroll
    for (int j = 0; j < CH; ++j) {
      const int e = threadIdx.x + (j0 + j) * NT;
      const int64_t idx = cbase + (int64_t)(e / TW) * g.PS + (e % TW);
      const int64_t pix = pbase + (int64_t)(e / TW) * g.pPS + (e % TW);
      if (use_d) dv[j] = __ldg(dinv + idx);
      if (MODE == FM_ITER) { pv[j] = p[pix]; xv[j] = x[idx]; }
    }
#pragma unroll
    for (int j = 0; j < CH; ++j) {
      const int e = threadIdx.x + (j0 + j) * NT;
      const int i0 = e / TW, col = e % TW;
      const int64_t idx = cbase + (int64_t)i0 * g.PS + col;
      const int64_t pix = pbase + (int64_t)i0 * g.pPS + col;
      double zz = zr[((i0 >> 1) * TW + col) * 2 + (i0 & 1)];
      if (use_d) zz = dv[j] * zz;
      if (MODE == FM_APPLY) {
        out[idx] = zz;
      } else if (MODE == FM_INIT) {
        p[pix] = zz;
      } else {
        x[idx] = xv[j] + alpha * pv[j];
        if (!done) p[pix] = beta * pv[j] + zz;
      }
    }
  }
}

FGeom fgeom(const Geom& g) {
  FGeom f{};
  f.d = g.d;
  f.n0 = g.n[0];
  f.nlast = g.n[g.d - 1];
  f.M0 = g.n[0] / 2;
  f.K0 = f.M0 + 1;
  f.N = g.N;
  f.PS = g.N / g.n[0];
  f.CS = (int64_t)f.K0 * f.PS;
  f.n1 = g.d == 3 ? g.n[1] : 1;
  f.FS = f.CS;
  f.KS = f.PS;
  f.SS = 0;
  f.rsh = ilog2c((int)(f.PS / f.nlast));
  f.sh = f.rsh;
  f.k0lo = 0;
  f.pN = f.N;
  f.pPS = f.PS;
  f.poff = 0;
  f.L = 1;
  f.vs = 0;
  f.bss = 0;
  f.c0 = 0;
  f.nc = g.d;
  return f;
}

// ---- size dispatch -------------------------------------------------------
template <int M, int F, int MODE, int TW>
void launchA_MT(const FGeom& g, cudaStream_t s, const PcgState* st, double* r, const double* kp,
                const double* dinv, double2* spec, const double2* tw) {
  constexpr int NT = passA_nt(M, F, TW);
  const size_t smem = sizeof(double2) * F * TW * M;
  auto k = passA<M, F, MODE, TW>;
  static std::atomic<uint64_t> attr{0};
  set_smem_once(k, smem, attr);
  dim3 grid((unsigned)(g.PS / TW) * g.L, g.nc);
  k<<<grid, NT, smem, s>>>(g, st, r, kp, dinv, spec, tw);
  JF_LAUNCHED();
}
// JFFTB_PASSA3=0 keeps the Stockham green-jacobi tile (A/B measurements)
inline bool passA3_enabled() {
  static const bool v = [] {
    const char* e = std::getenv("JFFTB_PASSA3");
    return !(e && e[0] == '0');
  }();
  return v;
}
// JFFTB_PASSA3_FL=0: last transform stage and unpack as separate smem passes
inline bool passA3_fused_last() {
  static const bool v = [] {
    const char* e = std::getenv("JFFTB_PASSA3_FL");
    return !(e && e[0] == '0');
  }();
  return v;
}
template <int M, int F, int MODE>
void launchA_M(const FGeom& g, cudaStream_t s, const PcgState* st, double* r, const double* kp,
               const double* dinv, double2* spec, const double2* tw) {
  if constexpr (F == 2 && MODE != FM_APPLY && passA3_ok<M>()) {
    if (passA3_enabled()) {
      constexpr int TW = tw_a(M);
      constexpr int NT = passA3_nt<M>();
      const size_t smem = sizeof(double2) * 2 * TW * M;
      auto k = passA3_fused_last() ? passA3<M, MODE, true> : passA3<M, MODE, false>;
      static std::atomic<uint64_t> attr{0};
      set_smem_once(k, smem, attr);
      dim3 grid((unsigned)(g.PS / TW) * g.L, g.nc);
      k<<<grid, NT, smem, s>>>(g, st, r, kp, dinv, spec, tw);
      JF_LAUNCHED();
      return;
    }
  }
  launchA_MT<M, F, MODE, tw_a(M)>(g, s, st, r, kp, dinv, spec, tw);
}
template <int L, bool INV, bool PRED>
void launchB_L(const FGeom& g, cudaStream_t s, const PcgState* st, double2* spec, int comp0,
               int ncomp, const double2* tw) {
  constexpr int TW = tw_b(L);
  constexpr int NT = nt_for(TW * L / 8);
  const size_t smem = sizeof(double2) * TW * L;
  auto k = g.SS != 0 ? passB<L, INV, PRED, true> : passB<L, INV, PRED, false>;
  static std::atomic<uint64_t> attr{0};
  set_smem_once(k, smem, attr);
  dim3 grid((unsigned)(g.nlast / TW) * g.L, g.K0, ncomp);
  k<<<grid, NT, smem, s>>>(g, st, spec, comp0, ncomp, tw);
  JF_LAUNCHED();
}
template <int D, int L, int F, int MODE, int GS, bool IP>
int launchC_V(const FGeom& g, cudaStream_t s, const PcgState* st, const double* gpc,
              const double* gterm, double2* spec, double* partials, const double2* tw,
              const GreenAna& ga) {
  constexpr int NT = passC_nt(D, L, F);
  const size_t smem = sizeof(double) * passC_bufd(D, L, F, GS);
  auto k = passC<D, L, F, MODE, GS, IP>;
  static std::atomic<uint64_t> attr{0};
  static int per_sm_dev[64];  // per instantiation and device
  const int dev = current_device();
  if (!(attr.load() & (1ull << dev))) {
    set_smem_once(k, smem, attr);
    JF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_dev[dev], k, NT, smem));
  }
  const int per_sm = per_sm_dev[dev];
  const int64_t rows = g.CS / L;
  // batched right-hand sides share the grid's blocks (the rows of one Green
  // plane set are read by L CTAs at about the same time: L2 hits)
  const int blocks = (int)std::min<int64_t>(rows, (int64_t)std::max(per_sm, 1) * 148 * 4 / g.L);
  k<<<blocks * g.L, NT, smem, s>>>(g, st, gpc, gterm, spec, partials, tw, ga);
  JF_LAUNCHED();
  return blocks;
}
// JFFTB_GREEN_ANALYTIC=1 evaluates the 3-D Green blocks in pass C instead of
// streaming the stored planes: 4.5 U less traffic and 36 KB less shared
// memory per CTA, but measured slower at 512^3 (4.02 vs 3.34 ms: pass C is
// bound by its shared-memory pipe and the ~150 extra flops per frequency
// cost more than the Green reads) -- off by default; kept for grids where
// the stored planes do not fit
inline bool green_analytic_enabled() {
  static const bool v = [] {
    const char* e = std::getenv("JFFTB_GREEN_ANALYTIC");
    return e && e[0] == '1';
  }();
  return v;
}
template <int D, int L, int F, int MODE>
int launchC_L(const FGeom& g, cudaStream_t s, const PcgState* st, const double* gpc,
              const double* gterm, double2* spec, double* partials, const double2* tw,
              const GreenAna& ga, bool analytic) {
  if constexpr (D == 3) {
    if (analytic && fused_dif())
      return launchC_V<D, L, F, MODE, 2, true>(g, s, st, gpc, gterm, spec, partials, tw, ga);
  }
  if (fused_dif())
    return launchC_V<D, L, F, MODE, 1, true>(g, s, st, gpc, gterm, spec, partials, tw, ga);
  return launchC_V<D, L, F, MODE, 1, false>(g, s, st, gpc, gterm, spec, partials, tw, ga);
}
template <int L, int F>
int launchBCB_L(const FGeom& g, cudaStream_t s, const PcgState* st, const double* gpc,
                const double* gterm, double2* spec, double* partials, const double2* tw,
                unsigned* q) {
  constexpr int NT = BCB_NT;
  const size_t smem = sizeof(double) * bcb_bufd(L);
  auto k = passBCB<L, F>;
  static std::atomic<uint64_t> attr{0};
  static int per_sm_dev[64];
  const int dev = current_device();
  if (!(attr.load() & (1ull << dev))) {
    set_smem_once(k, smem, attr);
    JF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_dev[dev], k, NT, smem));
  }
  int sms = 0;
  JF_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int blocks = std::max(per_sm_dev[dev], 1) * sms;
  // q[0]: ticket counter, q[1]: sticky wait-timeout flag (cleared and checked
  // by jfftb_pcg), q[2 ...]: per-plane counters
  JF_CUDA(cudaMemsetAsync(q, 0, sizeof(unsigned), s));
  JF_CUDA(cudaMemsetAsync(q + 2, 0, sizeof(unsigned) * 3 * (size_t)g.K0, s));
  k<<<blocks, NT, smem, s>>>(g, st, gpc, gterm, spec, partials, tw, q);
  JF_LAUNCHED();
  return (int)(g.CS / L);
}

template <int M, int MODE>
void launchI_M(const FGeom& g, cudaStream_t s, const PcgState* st, const double2* zspec,
               const double* dinv, double* p, double* x, double* out, const double2* tw) {
  constexpr int TW = tw_i(M);
  constexpr int NT = passI_nt(M);
  const size_t smem = sizeof(double2) * TW * (M + 1);
  auto k = passI<M, MODE>;
  static std::atomic<uint64_t> attr{0};
  set_smem_once(k, smem, attr);
  dim3 grid((unsigned)(g.PS / TW) * g.L, g.nc);
  k<<<grid, NT, smem, s>>>(g, st, zspec, dinv, p, x, out, tw);
  JF_LAUNCHED();
}

#ifdef JF_FAST_BUILD  // A/B builds: fewer instantiations
#define JF_SIZE_SWITCH(L, CALL)                   \
  switch (L) {                                    \
    case 128: { constexpr int LL = 128; CALL; break; } \
    case 256: { constexpr int LL = 256; CALL; break; } \
    case 512: { constexpr int LL = 512; CALL; break; } \
    case 1024: { constexpr int LL = 1024; CALL; break; } \
    case 2048: { constexpr int LL = 2048; CALL; break; } \
    default: throw Error(JFFTB_EINVAL, "fused FFT: unsupported size (fast build)"); \
  }
#else
#define JF_SIZE_SWITCH(L, CALL)                   \
  switch (L) {                                    \
    case 16: { constexpr int LL = 16; CALL; break; }   \
    case 32: { constexpr int LL = 32; CALL; break; }   \
    case 64: { constexpr int LL = 64; CALL; break; }   \
    case 128: { constexpr int LL = 128; CALL; break; } \
    case 256: { constexpr int LL = 256; CALL; break; } \
    case 512: { constexpr int LL = 512; CALL; break; } \
    case 1024: { constexpr int LL = 1024; CALL; break; } \
    case 2048: { constexpr int LL = 2048; CALL; break; } \
    default: throw Error(JFFTB_EINVAL, "fused FFT: unsupported size"); \
  }
#endif

void launchA(const FGeom& g, cudaStream_t s, int F, int mode, const PcgState* st, double* r,
             const double* kp, const double* dinv, double2* spec, const double2* tw) {
  // F = 2 (green-jacobi): r' and s = D^-1/2 r' from one read of r
  require(F == 1 || (F == 2 && mode != FM_APPLY), "pass A: F = 2 needs INIT / ITER");
  const int n0 = g.n0;
  if (F == 2) {
    if (mode == FM_ITER) { JF_SIZE_SWITCH(n0, (launchA_M<LL / 2, 2, FM_ITER>(g, s, st, r, kp, dinv, spec, tw))); }
    else { JF_SIZE_SWITCH(n0, (launchA_M<LL / 2, 2, FM_INIT>(g, s, st, r, kp, dinv, spec, tw))); }
  } else if (mode == FM_ITER) { JF_SIZE_SWITCH(n0, (launchA_M<LL / 2, 1, FM_ITER>(g, s, st, r, kp, dinv, spec, tw))); }
  else if (mode == FM_INIT) { JF_SIZE_SWITCH(n0, (launchA_M<LL / 2, 1, FM_INIT>(g, s, st, r, kp, dinv, spec, tw))); }
  else { JF_SIZE_SWITCH(n0, (launchA_M<LL / 2, 1, FM_APPLY>(g, s, st, r, kp, dinv, spec, tw))); }
}
void launchB(const FGeom& g, cudaStream_t s, bool inv, bool pred, const PcgState* st,
             double2* spec, int comp0, int ncomp, const double2* tw) {
  const int n1 = g.n1;
  if (inv) {
    if (pred) { JF_SIZE_SWITCH(n1, (launchB_L<LL, true, true>(g, s, st, spec, comp0, ncomp, tw))); }
    else { JF_SIZE_SWITCH(n1, (launchB_L<LL, true, false>(g, s, st, spec, comp0, ncomp, tw))); }
  } else {
    if (pred) { JF_SIZE_SWITCH(n1, (launchB_L<LL, false, true>(g, s, st, spec, comp0, ncomp, tw))); }
    else { JF_SIZE_SWITCH(n1, (launchB_L<LL, false, false>(g, s, st, spec, comp0, ncomp, tw))); }
  }
}
int launchC(const FGeom& g, cudaStream_t s, int F, int mode, const PcgState* st,
            const double* gpc, const double* gterm, double2* spec, double* partials,
            const double2* tw, const GreenAna& ga, bool analytic) {
  const int nl = g.nlast;
  int blocks = 0;
  if (g.d == 3) {
    if (mode == FM_APPLY) { JF_SIZE_SWITCH(nl, (blocks = launchC_L<3, LL, 1, FM_APPLY>(g, s, st, gpc, gterm, spec, partials, tw, ga, analytic))); }
    else if (F == 2) { JF_SIZE_SWITCH(nl, (blocks = launchC_L<3, LL, 2, FM_ITER>(g, s, st, gpc, gterm, spec, partials, tw, ga, analytic))); }
    else { JF_SIZE_SWITCH(nl, (blocks = launchC_L<3, LL, 1, FM_ITER>(g, s, st, gpc, gterm, spec, partials, tw, ga, analytic))); }
  } else {
    if (mode == FM_APPLY) { JF_SIZE_SWITCH(nl, (blocks = launchC_L<2, LL, 1, FM_APPLY>(g, s, st, gpc, gterm, spec, partials, tw, ga, analytic))); }
    else if (F == 2) { JF_SIZE_SWITCH(nl, (blocks = launchC_L<2, LL, 2, FM_ITER>(g, s, st, gpc, gterm, spec, partials, tw, ga, analytic))); }
    else { JF_SIZE_SWITCH(nl, (blocks = launchC_L<2, LL, 1, FM_ITER>(g, s, st, gpc, gterm, spec, partials, tw, ga, analytic))); }
  }
  return blocks;
}
void launchI(const FGeom& g, cudaStream_t s, int mode, const PcgState* st, const double2* zspec,
             const double* dinv, double* p, double* x, double* out, const double2* tw) {
  const int n0 = g.n0;
  if (mode == FM_ITER) { JF_SIZE_SWITCH(n0, (launchI_M<LL / 2, FM_ITER>(g, s, st, zspec, dinv, p, x, out, tw))); }
  else if (mode == FM_INIT) { JF_SIZE_SWITCH(n0, (launchI_M<LL / 2, FM_INIT>(g, s, st, zspec, dinv, p, x, out, tw))); }
  else { JF_SIZE_SWITCH(n0, (launchI_M<LL / 2, FM_APPLY>(g, s, st, zspec, dinv, p, x, out, tw))); }
}

}  // namespace

// analytic Green blocks for this green operator (and the termination one)?
GreenAna green_ana(const Geom& geo, const jfftb_green* gpc) {
  GreenAna ga{};
  ga.lam = gpc->lambda_ref;
  ga.mu = gpc->mu_ref;
  ga.w = geo.w;
  for (int a = 0; a < 3; ++a) ga.h[a] = geo.hinv[a];
  return ga;
}
bool use_analytic(const Geom& geo, const jfftb_green* gpc, const jfftb_green* gterm) {
  return geo.d == 3 && green_analytic_enabled() &&
         gterm->lambda_ref == gpc->lambda_ref && gterm->mu_ref == gpc->mu_ref;
}

void launch_twiddles(cudaStream_t s, double2* tw) {
  twiddle_kernel<<<kTwN / 256, 256, 0, s>>>(tw);
  JF_LAUNCHED();
  twiddle_stage_kernel<<<dim3(kTwN / 256, 13, 3), 256, 0, s>>>(tw);
  JF_LAUNCHED();
}

bool fused_dif() {
  static const bool v = [] {
    const char* e = std::getenv("JFFTB_PASSC_DIF");
    return !(e && e[0] == '0');
  }();
  return v;
}

bool fused_supported(const Geom& g) {
  for (int a = 0; a < g.d; ++a) {
    const int n = g.n[a];
    if (n < 16 || n > 2048 || (n & (n - 1))) return false;
  }
  return true;
}

int64_t fused_spec_elems(const Geom& g) { return (int64_t)(g.n[0] / 2 + 1) * (g.N / g.n[0]); }

// apply the Green (dinv == null) or Green-Jacobi preconditioner through the
// fused passes: out = D G D r  (spec: d * CS complex scratch)
void fused_precond_apply(const Geom& geo, cudaStream_t s, const jfftb_green* green,
                         const double* dinv, const double* r, double* out, double2* spec,
                         const double2* tw) {
  const FGeom g = fgeom(geo);
  const double* gblocks = green->blocks;
  const GreenAna ga = green_ana(geo, green);
  const bool an = use_analytic(geo, green, green);
  launchA(g, s, 1, FM_APPLY, nullptr, const_cast<double*>(r), nullptr, dinv, spec, tw);
  if (g.d == 3) launchB(g, s, false, false, nullptr, spec, 0, g.d, tw);
  launchC(g, s, 1, FM_APPLY, nullptr, gblocks, gblocks, spec, nullptr, tw, ga, an);
  if (g.d == 3) launchB(g, s, true, false, nullptr, spec, 0, g.d, tw);
  launchI(g, s, FM_APPLY, nullptr, spec, dinv, nullptr, nullptr, out, tw);
}

// diagnostic: run the APPLY passes up to `upto` (1 A, 2 B, 3 C, 4 B', 5 I)
void fused_debug_apply(const Geom& geo, cudaStream_t s, const jfftb_green* green,
                       const double* dinv, const double* r, double* out, double2* spec,
                       const double2* tw, int upto) {
  const FGeom g = fgeom(geo);
  const double* gblocks = green->blocks;
  const GreenAna ga = green_ana(geo, green);
  const bool an = use_analytic(geo, green, green);
  launchA(g, s, 1, FM_APPLY, nullptr, const_cast<double*>(r), nullptr, dinv, spec, tw);
  if (upto >= 2 && g.d == 3) launchB(g, s, false, false, nullptr, spec, 0, g.d, tw);
  if (upto >= 3) launchC(g, s, 1, FM_APPLY, nullptr, gblocks, gblocks, spec, nullptr, tw, ga, an);
  if (upto >= 4 && g.d == 3) launchB(g, s, true, false, nullptr, spec, 0, g.d, tw);
  if (upto >= 5) launchI(g, s, FM_APPLY, nullptr, spec, dinv, nullptr, nullptr, out, tw);
}

// ---- the PCG stages (pcg.cu strings them together) ------------------------
// A: mode FUSED_INIT / FUSED_ITER with F = 1 (green) or 2 (green-jacobi);
//    FUSED_APPLY transforms r (dinv == null) for the quad-only termination
FGeom fgeom_b(const Geom& geo, const Batch& bt) {
  FGeom g = fgeom(geo);
  g.L = bt.L;
  g.vs = bt.vs;
  g.bss = bt.bss;
  return g;
}
void fused_stage_A(const Geom& geo, cudaStream_t s, int F, int mode, const PcgState* st,
                   double* r, const double* kp, const double* dinv, double2* spec,
                   const double2* tw, const Batch& bt) {
  launchA(fgeom_b(geo, bt), s, F, mode, st, r, kp, dinv, spec, tw);
}
// one component (dist.cu)
void fused_stage_A_comp(const Geom& geo, cudaStream_t s, int F, int mode, const PcgState* st,
                        double* r, const double* kp, const double* dinv, double2* spec,
                        const double2* tw, int comp) {
  FGeom g = fgeom(geo);
  g.c0 = comp;
  g.nc = 1;
  launchA(g, s, F, mode, st, r, kp, dinv, spec, tw);
}
void fused_stage_B(const Geom& geo, cudaStream_t s, bool inv, const PcgState* st,
                   double2* spec, int ncomp, const double2* tw, const Batch& bt) {
  const FGeom g = fgeom_b(geo, bt);
  if (g.d == 3) launchB(g, s, inv, true, st, spec, 0, ncomp, tw);
}
// returns the number of partial pairs written (per right-hand side)
int fused_stage_C(const Geom& geo, cudaStream_t s, int F, bool quad_only, const PcgState* st,
                  const jfftb_green* gpc_h, const jfftb_green* gterm_h, double2* spec,
                  double* partials, const double2* tw, const Batch& bt) {
  const FGeom g = fgeom_b(geo, bt);
  const double* gpc = gpc_h->blocks;
  const double* gterm = gterm_h->blocks;
  const GreenAna ga = green_ana(geo, gpc_h);
  const bool an = use_analytic(geo, gpc_h, gterm_h);
  if (quad_only) {
    int blocks = 0;
    if (g.d == 3) {
      JF_SIZE_SWITCH(g.nlast, (blocks = launchC_L<3, LL, 1, FM_QUAD>(g, s, st, gpc, gterm, spec, partials, tw, ga, an)));
    } else {
      JF_SIZE_SWITCH(g.nlast, (blocks = launchC_L<2, LL, 1, FM_QUAD>(g, s, st, gpc, gterm, spec, partials, tw, ga, an)));
    }
    return blocks;
  }
  return launchC(g, s, F, FM_ITER, st, gpc, gterm, spec, partials, tw, ga, an);
}
// Merged B / C / B' (passBCB): 3-D grids with n1 == n2, one solve, stored
// Green planes.  Opt-in (JFFTB_BCB=1): it halves the DRAM traffic of the three
// passes (ncu, 512^3 green-jacobi: 18.2 GB vs 33.8 GB per iteration) but runs
// slower than them (7.5 vs 6.5 ms): three items fit an SM and an item is a
// serial chain of barrier-separated stages (~8 us), while the separate
// passes each fill the SM for their own bottleneck (profiles/r02_ab_notes.md)
bool fused_bcb_supported(const Geom& geo) {
  const char* e = std::getenv("JFFTB_BCB");  // read per solve (tests switch it)
  const bool on = e && e[0] != '0';
  return on && geo.d == 3 && geo.n[1] == geo.n[2] && fused_supported(geo) && fused_dif() &&
         !green_analytic_enabled();
}
int64_t fused_bcb_partials(const Geom& geo) {
  return geo.d == 3 ? (int64_t)(geo.n[0] / 2 + 1) * geo.n[1] : 0;
}
// returns the number of partial pairs written; q: 2 + 3 K0 counters
int fused_stage_BCB(const Geom& geo, cudaStream_t s, int F, const PcgState* st,
                    const jfftb_green* gpc_h, const jfftb_green* gterm_h, double2* spec,
                    double* partials, const double2* tw, unsigned* q) {
  const FGeom g = fgeom(geo);
  const double* gpc = gpc_h->blocks;
  const double* gterm = gterm_h->blocks;
  int n = 0;
  if (F == 2) { JF_SIZE_SWITCH(g.nlast, (n = launchBCB_L<LL, 2>(g, s, st, gpc, gterm, spec, partials, tw, q))); }
  else { JF_SIZE_SWITCH(g.nlast, (n = launchBCB_L<LL, 1>(g, s, st, gpc, gterm, spec, partials, tw, q))); }
  return n;
}
void fused_stage_I(const Geom& geo, cudaStream_t s, int mode, const PcgState* st,
                   const double2* zspec, const double* dinv, double* p, double* x,
                   const double2* tw, const Batch& bt) {
  launchI(fgeom_b(geo, bt), s, mode, st, zspec, dinv, p, x, nullptr, tw);
}
int64_t fused_component_stride(const Geom& geo) { return fgeom(geo).CS; }

// ---- distributed solves (dist.cu) ------------------------------------------
// The spectral passes of one rank's k0-slab: frequency rows k0 in
// [k0lo, k0lo + kcnt) of the global grid `geo`, received from P = n1 / L1
// ranks into [src][field (nf)][k0][i1 local (L1)][i2] (one segment per source
// rank, field stride kcnt L1 n2, segment stride nf times that).
FGeom fgeom_slab(const Geom& geo, const SpecSlab& sl) {
  FGeom g = fgeom(geo);
  g.K0 = sl.kcnt;
  g.k0lo = sl.k0lo;
  g.CS = (int64_t)sl.kcnt * g.PS;  // elements per field (rows kcnt x n1)
  g.KS = (int64_t)sl.L1 * g.nlast;
  g.FS = (int64_t)sl.kcnt * g.KS;
  g.SS = (int64_t)sl.nf * g.FS;
  g.sh = ilog2c(sl.L1);
  return g;
}
void fused_stage_B_slab(const Geom& geo, const SpecSlab& sl, cudaStream_t s, bool inv,
                        const PcgState* st, double2* recv, int comp0, int ncomp,
                        const double2* tw) {
  launchB(fgeom_slab(geo, sl), s, inv, true, st, recv, comp0, ncomp, tw);
}
int fused_stage_C_slab(const Geom& geo, const SpecSlab& sl, cudaStream_t s, int F,
                       const PcgState* st, const double* green, double2* recv, double* partials,
                       const double2* tw) {
  const FGeom g = fgeom_slab(geo, sl);
  return launchC(g, s, F, FM_ITER, st, green, green, recv, partials, tw, GreenAna{}, false);
}
// pass I of a rank whose direction p lives in a halo-extended slab of
// n1 + 2 rows along axis 1 (geo: the rank's local real-space slab)
void fused_stage_I_ext(const Geom& geo, cudaStream_t s, int mode, const PcgState* st,
                       const double2* zspec, const double* dinv, double* p_ext, double* x,
                       const double2* tw, int comp) {
  FGeom g = fgeom(geo);
  if (comp >= 0) {
    g.c0 = comp;
    g.nc = 1;
  }
  g.pPS = (int64_t)(geo.n[1] + 2) * geo.n[2];
  g.pN = (int64_t)geo.n[0] * g.pPS;
  g.poff = geo.n[2];  // row 0 of the extended slab is the lower halo
  launchI(g, s, mode, st, zspec, dinv, p_ext, x, nullptr, tw);
}

}  // namespace jfftb
