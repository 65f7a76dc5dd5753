// Energy pairings of several load-case solutions (the
// consumer of pcg in topopt.py:98-196).
//
// For load cases g = 0..L-1 with displacement u_g and macroscopic strain
// Ebar_g, the total strain on simplex t of voxel x is eps_g = Ebar_g + B u_g
// (operators.py:79-83).  The reference pairs them as
//   P_gc(x) = sum_t eps_c(x, t)^T C0 eps_g(x, t)         (_strain_pairings,
//                                                         topopt.py:130-133)
//   Sigma_gc = (w / |Y|) sum_x rho(x) P_gc(x)            (_stress_matrix,
//                                                         topopt.py:136-141)
//   grad(x)  = sum_gc W_gc P_gc(x)                       (_stress_gradient,
//                                                         topopt.py:163-180,
//                                                         before its scale)
// with the isotropic C0: eps_c^T C0 eps_g = lam tr(eps_c) tr(eps_g) +
// 2 mu eps_c : eps_g.  One thread per voxel, every load's corner values read
// through L1; Sigma reduced per block in a fixed order (deterministic).
#include "common.cuh"

namespace jfftb {

namespace {

constexpr int kLcThreads = 128;
constexpr int kMaxLoads = 6;

// edge_base with a runtime simplex index (the tet loop is not unrolled)
template <int D>
__device__ __forceinline__ int d_edge_base(int t, int a) {
  int r = 0;
#pragma unroll
  for (int tt = 0; tt < n_simplex(D); ++tt)
    if (tt == t) r = edge_base(D, tt, a);
  return r;
}

struct LoadStrains {
  double e[kMaxLoads][3][3];  // Ebar_g as tensors
};

template <int D, int L>
__global__ void __launch_bounds__(kLcThreads)
    pairings_kernel(Geom g, const double* __restrict__ u, const double* __restrict__ rho,
                    double lam, double mu, LoadStrains E, const double* __restrict__ wgt,
                    double* __restrict__ field, double* __restrict__ partials) {
  constexpr int T = n_simplex(D);
  constexpr int K = L * (L + 1) / 2;
  constexpr int S = D == 2 ? 3 : 6;  // symmetric components (diagonal first)
  const int64_t N = g.N;
  const int n0 = g.n[0], n1 = g.n[1], n2 = D == 3 ? g.n[2] : 1;
  // pair weights, symmetrised: Wk = W_aa or W_ab + W_ba for the pair k = (a <= b)
  __shared__ double Wk[K];
  if (wgt && threadIdx.x == 0) {
    int k = 0;
    for (int a = 0; a < L; ++a)
      for (int b = a; b < L; ++b, ++k)
        Wk[k] = a == b ? wgt[a * L + a] : wgt[a * L + b] + wgt[b * L + a];
  }
  __syncthreads();
  double wsum[K];
#pragma unroll
  for (int k = 0; k < K; ++k) wsum[k] = 0.0;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < N;
       v += (int64_t)gridDim.x * blockDim.x) {
    int c[3];
    int64_t r = v;
    c[D - 1] = (int)(r % (D == 3 ? n2 : n1));
    r /= (D == 3 ? n2 : n1);
    if (D == 3) { c[1] = (int)(r % n1); r /= n1; }
    c[0] = (int)r;
    // corner index: bit j = +1 along axis j (periodic)
    int64_t cid[1 << D];
#pragma unroll
    for (int m = 0; m < (1 << D); ++m) {
      int64_t idx = 0;
#pragma unroll
      for (int a = 0; a < D; ++a) {
        const int na = a == 0 ? n0 : (a == 1 ? n1 : n2);
        int q = c[a] + ((m >> a) & 1);
        if (q == na) q = 0;
        idx = idx * na + q;
      }
      cid[m] = idx;
    }
    const double rv = rho[v];
    double fs = 0.0;
#pragma unroll 1
    for (int t = 0; t < T; ++t) {
      double eps[L][S];
#pragma unroll
      for (int l = 0; l < L; ++l) {
        const double* ul = u + (int64_t)l * D * N;
        double G[D][D];
#pragma unroll
        for (int a = 0; a < D; ++a) {
          const int o = d_edge_base<D>(t, a);
#pragma unroll
          for (int i = 0; i < D; ++i)
            G[i][a] = (__ldg(ul + i * N + cid[o | (1 << a)]) - __ldg(ul + i * N + cid[o])) *
                          g.hinv[a] + E.e[l][i][a];
        }
#pragma unroll
        for (int i = 0; i < D; ++i) eps[l][i] = G[i][i];
        if (D == 2) {
          eps[l][2] = 0.5 * (G[0][1] + G[1][0]);
        } else {
          eps[l][3] = 0.5 * (G[1][2] + G[2][1]);
          eps[l][4] = 0.5 * (G[0][2] + G[2][0]);
          eps[l][5] = 0.5 * (G[0][1] + G[1][0]);
        }
      }
      int k = 0;
#pragma unroll
      for (int a = 0; a < L; ++a)
#pragma unroll
        for (int b = a; b < L; ++b, ++k) {
          double tra = 0.0, trb = 0.0, dd = 0.0, od = 0.0;
#pragma unroll
          for (int i = 0; i < D; ++i) {
            tra += eps[a][i];
            trb += eps[b][i];
            dd += eps[a][i] * eps[b][i];
          }
#pragma unroll
          for (int i = D; i < S; ++i) od += eps[a][i] * eps[b][i];
          const double p = lam * tra * trb + 2.0 * mu * (dd + 2.0 * od);
          wsum[k] += rv * p;
          if (field) fs += Wk[k] * p;
        }
    }
    if (field) field[v] = fs;
  }
  // fixed-order block reduction of the K sums
  __shared__ double red[kLcThreads / 32][K];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    double s = wsum[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if (lane == 0) red[wid][k] = s;
  }
  __syncthreads();
  for (int k = threadIdx.x; k < K; k += blockDim.x) {
    double s = 0.0;
    for (int w = 0; w < kLcThreads / 32; ++w) s += red[w][k];
    partials[(int64_t)blockIdx.x * K + k] = s;
  }
}

template <int D, int L>
void launch_pairings_DL(const Geom& g, cudaStream_t s, const double* u, const double* rho,
                        double lam, double mu, const LoadStrains& E, const double* wgt,
                        double* field, double* partials) {
  pairings_kernel<D, L><<<kRedBlocks, kLcThreads, 0, s>>>(g, u, rho, lam, mu, E, wgt, field,
                                                          partials);
  JF_LAUNCHED();
}

}  // namespace

// u: L vector fields back to back; ebar: L Mandel vectors (3 or 6 entries
// each); wgt (device, L x L) and field may be null.  Writes kRedBlocks
// partial rows of L (L + 1) / 2 sums (a <= b, row-major) and returns K.
int launch_load_pairings(const Geom& g, cudaStream_t s, int L, const double* u,
                         const double* rho, double lam, double mu, const double* ebar,
                         const double* wgt, double* field, double* partials) {
  require(L >= 1 && L <= kMaxLoads, "1 to 6 load cases");
  LoadStrains E{};
  const int M = g.d == 2 ? 3 : 6;
  for (int l = 0; l < L; ++l) {
    const double* m = ebar + l * M;
    for (int i = 0; i < g.d; ++i) E.e[l][i][i] = m[i];
    if (g.d == 2) {
      E.e[l][0][1] = E.e[l][1][0] = m[2] / kSqrt2;
    } else {
      E.e[l][1][2] = E.e[l][2][1] = m[3] / kSqrt2;
      E.e[l][0][2] = E.e[l][2][0] = m[4] / kSqrt2;
      E.e[l][0][1] = E.e[l][1][0] = m[5] / kSqrt2;
    }
  }
#define JF_LC(DD, LL) \
  case LL: launch_pairings_DL<DD, LL>(g, s, u, rho, lam, mu, E, wgt, field, partials); break;
  if (g.d == 2) {
    switch (L) { JF_LC(2, 1) JF_LC(2, 2) JF_LC(2, 3) JF_LC(2, 4) JF_LC(2, 5) JF_LC(2, 6) }
  } else {
    switch (L) { JF_LC(3, 1) JF_LC(3, 2) JF_LC(3, 3) JF_LC(3, 4) JF_LC(3, 5) JF_LC(3, 6) }
  }
#undef JF_LC
  return L * (L + 1) / 2;
}

}  // namespace jfftb
