// Matrix-free P1 stiffness apply and its relatives (rhs, residual force,
// total strain, stress average) on the periodic grid.
//
// Replaces operators.py:43-101 / fem.py:41-111 (K u = B^T W rho C0 B u).
//
// KA design ("plane march"): a CTA owns a (BY x BX) column tile of voxels in
// the (axis1, axis2) plane -- axis 2 is the contiguous one -- and marches
// along axis 0.  Each thread owns one voxel column: per layer it reads its
// node of the next plane once from HBM (coalesced along axis 2), takes the
// other three corners of its voxel from shared memory, evaluates the voxel's
// d! simplices in registers (voxel_forces) and hands the corner forces that
// belong to neighbouring node columns over shared memory.  The lowest row and
// column of the tile are halo voxels, so a CTA emits (BY-1) x (BX-1) node
// columns and every node is written exactly once, with a fixed summation
// order (bitwise deterministic).  rho and u are read once per layer; out is
// written once: 2d+1 scalar fields of HBM traffic per apply.
#include "common.cuh"

namespace jfftb {

namespace {

// 3-D tile (threads), emits 31 x 7 columns (32 x 16 measured slower: 4.05 vs
// 3.80 ms at 512^3 -- one CTA of 16 warps hides less than two of 8)
#ifndef JF_ST_BY
#define JF_ST_BY 8
#endif
#ifndef JF_ST_MINB
#define JF_ST_MINB 2
#endif
constexpr int BX3 = 32, BY3 = JF_ST_BY;
constexpr int MINB3 = BY3 <= 8 ? JF_ST_MINB : 1;  // resident CTAs per SM the launch bounds target
constexpr int BX2 = 128;           // 2-D tile, emits 127 columns

__device__ __forceinline__ int wrapi(int i, int n) {
  i %= n;
  return i < 0 ? i + n : i;
}

__device__ __forceinline__ double block_sum(double v, double* red) {
  // deterministic block reduction (fixed tree); returns total in thread 0
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int tid = threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z);
  const int nthr = blockDim.x * blockDim.y * blockDim.z;
  const int lane = tid & 31, wid = tid >> 5;
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  double s = 0.0;
  if (wid == 0) {
    s = lane < (nthr >> 5) ? red[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  }
  return s;
}

struct EbarT {
  double e[3][3];
  double m[6];  // the Mandel vector itself
};

__host__ EbarT make_ebar(int d, const double* m) {
  EbarT E{};
  if (!m) return E;
  for (int k = 0; k < (d == 2 ? 3 : 6); ++k) E.m[k] = m[k];
  for (int i = 0; i < d; ++i) E.e[i][i] = m[i];
  if (d == 2) {
    E.e[0][1] = E.e[1][0] = m[2] / kSqrt2;
  } else {
    E.e[1][2] = E.e[2][1] = m[3] / kSqrt2;
    E.e[0][2] = E.e[2][0] = m[4] / kSqrt2;
    E.e[0][1] = E.e[1][0] = m[5] / kSqrt2;
  }
  return E;
}

// --------------------------------------------------------------------------
// 3-D plane-march stencil
// --------------------------------------------------------------------------
// One warp per tile row (BX3 = 32 lanes along the contiguous axis 2).  Per
// layer the displacement plane two layers ahead and the density layer one
// ahead stream global -> shared with cp.async (no registers held, latency
// hidden behind a whole layer of voxel math) into 3-deep rings; corner
// displacements are read from the ring, forces for the +x neighbour travel by
// warp shuffle and the combined +y forces through a double-buffered smem row.
// One __syncthreads per layer.
// ring depth: plane kk + RING - 1 is requested while layer kk is computed
#ifndef JF_ST_RING
#define JF_ST_RING 3
#endif
constexpr int RING = JF_ST_RING;
static_assert(RING == 3 || RING == 4, "plane ring of 3 or 4 slots");
constexpr int S3_U = RING * 3 * (BY3 + 1) * (BX3 + 1);  // u ring: [slot][comp][y][x]
constexpr int S3_R = RING * BY3 * BX3;                  // rho ring: [slot][y][x]
constexpr int S3_F = 2 * 2 * 3 * BY3 * BX3;          // +y hand-over: [buf][plane][comp][y][x]
constexpr size_t S3_BYTES = sizeof(double) * (S3_U + S3_R + S3_F + 32);

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
// predicated form: no branch around the copy (divergent branches around
// LDGSTS cost the march dozens of issue slots per layer)
__device__ __forceinline__ void cp_async8_if(void* smem, const void* gmem, bool on) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %2, 0;\n"
      " @p cp.async.ca.shared.global [%0], [%1], 8;\n}\n" ::"r"(s),
      "l"(gmem), "r"((int)on));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

template <int MODE, bool SCALE>
__global__ void __launch_bounds__(BX3* BY3, MINB3)
    stencil3d(Geom g, const double* __restrict__ u, const double* __restrict__ rho,
              double lam0, double mu0, EbarT E, double* __restrict__ out,
              double* __restrict__ partials, int chunk, int ext, int nchunks,
              int64_t bstride, const PcgState* __restrict__ st, int yoff, int ytot) {
  constexpr bool HAS_U = MODE != VOX_RHS;
  extern __shared__ double smem[];
  double(*U)[3][BY3 + 1][BX3 + 1] = reinterpret_cast<double(*)[3][BY3 + 1][BX3 + 1]>(smem);
  double(*R)[BY3][BX3] = reinterpret_cast<double(*)[BY3][BX3]>(smem + S3_U);
  double(*Fy)[2][3][BY3][BX3] =
      reinterpret_cast<double(*)[2][3][BY3][BX3]>(smem + S3_U + S3_R);
  double* red = smem + S3_U + S3_R + S3_F;

  const int n0 = g.n[0], n1 = g.n[1], n2 = g.n[2];
  const int64_t P = (int64_t)n1 * n2;
  // ext = 1 (distributed slabs, dist.cu): u and rho are halo-extended slabs
  // of n1 + 2 rows along axis 1 (input row = output row + 1, no wrap along
  // axis 1); out keeps the n1 rows
  const int64_t Pin = ext ? P + 2 * (int64_t)n2 : P, Nin = (int64_t)n0 * Pin;
  auto in_row = [&](int y) { return ext ? min(y + 1, n1 + 1) : wrapi(y, n1); };
  // PCG direction update predicated on the solve state (no work once done);
  // tile rows [yoff, yoff + gridDim.y) of ytot (a row group, pcg.cu)
  if (st && st->done) return;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int by = blockIdx.y + yoff;
  const int X0 = blockIdx.x * (BX3 - 1), Y0 = by * (BY3 - 1);
  // batched right-hand sides: blockIdx.z = rhs * nchunks + chunk; u and out
  // are bstride doubles apart (rho is shared)
  const int bl = (int)blockIdx.z / nchunks;
  if (u) u += bl * bstride;
  out += bl * bstride;
  const int k0 = ((int)blockIdx.z % nchunks) * chunk;
  const int k1 = min(k0 + chunk, n0);
  const int gx = X0 - 1 + tx, gy = Y0 - 1 + ty;
  const int c2 = wrapi(gx, n2);
  const bool outp = tx >= 1 && ty >= 1 && gx < n2 && gy < n1;
  const int c2h = wrapi(X0 - 1 + BX3, n2), c1h = in_row(Y0 - 1 + BY3);
  const int64_t col = (int64_t)(outp ? gy : 0) * n2 + c2;  // output column
  const int64_t cin = (int64_t)in_row(gy) * n2 + c2;       // input column
  // halo of a plane: column x = BX3 (BY3 values) and row y = BY3 (BX3 + 1
  // values) of each component, 3 * 41 copies spread over the first threads
  constexpr int HPC = BY3 + BX3 + 1;  // halo values per component
  const int tid = ty * BX3 + tx;
  const bool h_on = tid < 3 * HPC;
  int64_t h_src = 0;  // offset from the plane base (component included)
  int h_dst = 0;      // offset from the slot base, in doubles
  if (h_on) {
    const int hc = tid / HPC, e = tid % HPC;
    const int hy_ = e < BY3 ? e : BY3, hx_ = e < BY3 ? BX3 : e - BY3;
    h_src = (int64_t)hc * Nin + (int64_t)in_row(Y0 - 1 + hy_) * n2 + wrapi(X0 - 1 + hx_, n2);
    h_dst = (hc * (BY3 + 1) + hy_) * (BX3 + 1) + hx_;
  }
  (void)c2h;
  (void)c1h;

  double gs[3], fs[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) { gs[a] = g.hinv[a]; fs[a] = g.hinv[a]; }
  const double (*Eb)[3] = E.e;

  // async fetch of layer kk (unwrapped, -1 <= kk <= n0 + 2) into ring slot
  // (kk+3)%3; plane wrap by compare (no integer division in the march)
  auto plane_of = [&](int kk) { return kk < 0 ? kk + n0 : (kk >= n0 ? kk - n0 : kk); };
  auto slot_of = [](int kk) { return (kk + RING) % RING; };
  auto next_slot = [](int sl) { return sl == RING - 1 ? 0 : sl + 1; };
  auto fetch_u = [&](int kk, int s) {
    if (!HAS_U) return;
    const double* ub = u + (int64_t)plane_of(kk) * Pin;
#pragma unroll
    for (int i = 0; i < 3; ++i) cp_async8(&U[s][i][ty][tx], ub + i * Nin + cin);
    cp_async8_if(&U[s][0][0][0] + h_dst, ub + h_src, h_on);
  };
  auto fetch_r = [&](int kk, int s) {
    if (rho) cp_async8(&R[s][ty][tx], rho + (int64_t)plane_of(kk) * Pin + cin);
  };
  auto read_corners = [&](int s, double (&q)[4][3]) {
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      q[0][i] = U[s][i][ty][tx];
      q[1][i] = U[s][i][ty][tx + 1];
      q[2][i] = U[s][i][ty + 1][tx];
      q[3][i] = U[s][i][ty + 1][tx + 1];
    }
  };

  double uk[4][3], uk1[4][3];
#pragma unroll
  for (int q = 0; q < 4; ++q)
#pragma unroll
    for (int i = 0; i < 3; ++i) uk[q][i] = uk1[q][i] = 0.0;
  // prologue: group A = planes k0-1, k0 and rho(k0-1); then one group per
  // plane k0+i with rho(k0+i-1), i = 1 .. RING-2
  int s0 = slot_of(k0 - 1);                   // slot of layer kk (rotates by one)
  int s1 = next_slot(s0);
  fetch_u(k0 - 1, s0);
  fetch_u(k0, s1);
  fetch_r(k0 - 1, s0);
  cp_async_commit();
#pragma unroll
  for (int i = 1; i <= RING - 2; ++i) {
    fetch_u(k0 + i, slot_of(k0 - 1 + i + 1));
    fetch_r(k0 + i - 1, slot_of(k0 - 1 + i));
    cp_async_commit();
  }
  cp_async_wait<RING - 2>();
  __syncthreads();

  double nxt[3] = {0.0, 0.0, 0.0};
  double csum = 0.0;
  int64_t obase = (int64_t)plane_of(k0 - 1) * P + col;  // output index of layer kk
  for (int kk = k0 - 1, j = 0; kk < k1; ++kk, ++j) {
    const int b = j & 1;
    // slots: s0 = layer kk (u plane kk, rho kk), s1 = kk + 1; planes up to
    // kk + RING - 1 are in flight
    // Both corner planes are read from the ring (no register hand-over
    // between layers); the slots are refilled after this layer's barrier.
    if (HAS_U) {
      read_corners(s0, uk);
      read_corners(s1, uk1);
    }
    const double r = rho ? R[s0][ty][tx] : 1.0;
    double uc[8][3];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int q = (((c >> 1) & 1) << 1) | ((c >> 2) & 1);
#pragma unroll
      for (int i = 0; i < 3; ++i) uc[c][i] = (c & 1) ? uk1[q][i] : uk[q][i];
    }
    double f[8][3];
    voxel_forces<3, MODE, SCALE>(uc, lam0 * r, mu0 * r, gs, fs, Eb, f);
    double ak[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      // +x neighbour (lane - 1) hands over its corners (0,0,1), (1,0,1); its
      // (.,1,1) corners join our +y hand-over
      const double x0 = __shfl_up_sync(0xffffffffu, f[4][i], 1);
      const double x1 = __shfl_up_sync(0xffffffffu, f[5][i], 1);
      const double y0 = __shfl_up_sync(0xffffffffu, f[6][i], 1);
      const double y1 = __shfl_up_sync(0xffffffffu, f[7][i], 1);
      ak[i] = nxt[i] + f[0][i] + x0;
      nxt[i] = f[1][i] + x1;
#ifndef JF_ST_SEL
      // lane 0 is a halo column: whatever it hands over only reaches other
      // halo columns (never an output node), so no select is needed
      Fy[b][0][i][ty][tx] = f[2][i] + y0;
      Fy[b][1][i][ty][tx] = f[3][i] + y1;
#else
      Fy[b][0][i][ty][tx] = f[2][i] + (tx >= 1 ? y0 : 0.0);
      Fy[b][1][i][ty][tx] = f[3][i] + (tx >= 1 ? y1 : 0.0);
#endif
    }
    cp_async_wait<RING - 3>();  // plane kk+2 / rho(kk+1) landed (needed next layer)
    __syncthreads();     // ... and every warp is done reading slot s0
    if (ty >= 1) {
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        ak[i] += Fy[b][0][i][ty - 1][tx];
        nxt[i] += Fy[b][1][i][ty - 1][tx];
      }
    }
    if (kk >= k0 && outp) {
#pragma unroll
      for (int i = 0; i < 3; ++i) out[i * g.N + obase] = ak[i];
      if (MODE == VOX_K && partials)
        csum += uk[0][0] * ak[0] + uk[0][1] * ak[1] + uk[0][2] * ak[2];
    }
    obase += P;
    if (obase >= g.N) obase -= g.N;
    // refill: plane kk+RING takes plane kk's slot, rho(kk+RING-1) takes
    // rho(kk-1)'s
    if (kk + RING <= k1) fetch_u(kk + RING, s0);
    if (kk + RING - 1 < k1) fetch_r(kk + RING - 1, slot_of(kk + RING - 1));
    cp_async_commit();
    s0 = s1;
    s1 = next_slot(s1);
  }
  cp_async_wait<0>();
  if (MODE == VOX_K && partials) {
    const double s = block_sum(csum, red);
    if (threadIdx.x == 0 && threadIdx.y == 0)
      partials[blockIdx.x + gridDim.x * (by + ytot * blockIdx.z)] = s;
  }
}

// --------------------------------------------------------------------------
// 2-D plane-march stencil (axis 0 marched, axis 1 across threads)
// --------------------------------------------------------------------------
// Each thread owns one node column.  Its own node of plane k is loaded into
// registers three layers ahead (plain loads, no barrier), published to a
// double-buffered shared row for the neighbour on its left (and the tile's
// halo column by the last thread), and the forces for the +x neighbour travel
// through a double-buffered shared row that is read one layer later -- so a
// layer costs ONE barrier, and a node is finalised and written one layer
// after its last voxel.
template <int MODE, bool SCALE>
__global__ void __launch_bounds__(BX2)
    stencil2d(Geom g, const double* __restrict__ u, const double* __restrict__ rho,
              double lam0, double mu0, EbarT E, double* __restrict__ out,
              double* __restrict__ partials, int chunk, int) {
  constexpr bool HAS_U = MODE != VOX_RHS;
  __shared__ double U[2][2][BX2 + 1];   // [buf][comp][x]: node plane kk + 1
  __shared__ double F[2][2][2][BX2];    // [buf][plane][comp][x]: +x forces of layer kk
  __shared__ double red[32];
  const int n0 = g.n[0], n1 = g.n[1];
  const int tx = threadIdx.x;
  const int X0 = blockIdx.x * (BX2 - 1);
  const int k0 = blockIdx.y * chunk;
  const int k1 = min(k0 + chunk, n0);
  const int gx = X0 - 1 + tx;
  const int c1 = wrapi(gx, n1);
  const bool outp = tx >= 1 && gx < n1;
  const bool halo = tx == BX2 - 1;
  const int c1h = wrapi(X0 - 1 + BX2, n1);
  double gs[2] = {g.hinv[0], g.hinv[1]}, fs[2] = {g.hinv[0], g.hinv[1]};
  const double (*Eb)[3] = E.e;
  auto pl = [&](int k) { return k < 0 ? k + n0 : (k >= n0 ? k - n0 : k); };
  // own (and, for the last thread, halo-column) values of plane k
  struct Node {
    double v[2], h[2], r;
  };
  auto fetch = [&](int kk) {
    Node q{};
    const int64_t base = (int64_t)pl(kk) * n1;
    if (HAS_U) {
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        q.v[i] = __ldg(u + i * g.N + base + c1);
        q.h[i] = halo ? __ldg(u + i * g.N + base + c1h) : 0.0;
      }
    }
    q.r = rho ? __ldg(rho + base + c1) : 1.0;
    return q;
  };
  // prefetch ring: planes kk, kk + 1, kk + 2 (kk = k0 - 1 first)
  Node q0 = fetch(k0 - 1), q1 = fetch(k0), q2 = fetch(k0 + 1);
  double uk[2][2];  // corners of plane kk: own, +x
  if (HAS_U) {
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      U[1][i][tx] = q0.v[i];
      if (halo) U[1][i][BX2] = q0.h[i];
    }
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    uk[0][i] = HAS_U ? U[1][i][tx] : 0.0;
    uk[1][i] = HAS_U ? U[1][i][tx + 1] : 0.0;
  }
  double nxt[2] = {0.0, 0.0}, ak[2] = {0.0, 0.0}, pk[2] = {0.0, 0.0};
  double csum = 0.0;
  int64_t oidx = (int64_t)pl(k0 - 1) * n1 + c1;  // node of the pending output
  for (int kk = k0 - 1, j = 0; kk < k1; ++kk, ++j) {
    const int b = j & 1;
    // publish plane kk + 1, then request plane kk + 3
    if (HAS_U) {
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        U[b][i][tx] = q1.v[i];
        if (halo) U[b][i][BX2] = q1.h[i];
      }
    }
    const double rk = q0.r;
    q0 = q1;
    q1 = q2;
    if (kk + 3 <= k1) q2 = fetch(kk + 3);
    __syncthreads();  // U[b] written; F[b ^ 1] of layer kk - 1 written
    // finish node kk - 1 with the +x forces of layer kk - 1
    if (kk > k0 - 1) {
      if (tx >= 1) {
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          ak[i] = ak[i] + F[b ^ 1][0][i][tx - 1];
          nxt[i] = nxt[i] + F[b ^ 1][1][i][tx - 1];
        }
      }
      if (kk - 1 >= k0 && outp) {
        out[oidx] = ak[0];
        out[g.N + oidx] = ak[1];
        if (MODE == VOX_K && partials) csum += pk[0] * ak[0] + pk[1] * ak[1];
      }
      oidx += n1;
      if (oidx >= g.N) oidx -= g.N;
    }
    double uk1[2][2];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      uk1[0][i] = HAS_U ? q0.v[i] : 0.0;
      uk1[1][i] = HAS_U ? U[b][i][tx + 1] : 0.0;
    }
    double uc[4][2];
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
      for (int i = 0; i < 2; ++i) uc[c][i] = (c & 1) ? uk1[(c >> 1) & 1][i] : uk[(c >> 1) & 1][i];
    double f[4][2];
    voxel_forces<2, MODE, SCALE>(uc, lam0 * rk, mu0 * rk, gs, fs, Eb, f);
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      ak[i] = nxt[i] + f[0][i];
      nxt[i] = f[1][i];
      F[b][0][i][tx] = f[2][i];
      F[b][1][i][tx] = f[3][i];
      pk[i] = uk[0][i];
      uk[0][i] = uk1[0][i];
      uk[1][i] = uk1[1][i];
    }
  }
  // the last layer's node
  __syncthreads();
  {
    const int b = (k1 - k0) & 1;  // buffer of layer k1 - 1
    if (tx >= 1) {
#pragma unroll
      for (int i = 0; i < 2; ++i) ak[i] = ak[i] + F[b][0][i][tx - 1];
    }
    if (k1 - 1 >= k0 && outp) {
      out[oidx] = ak[0];
      out[g.N + oidx] = ak[1];
      if (MODE == VOX_K && partials) csum += pk[0] * ak[0] + pk[1] * ak[1];
    }
  }
  if (MODE == VOX_K && partials) {
    const double s = block_sum(csum, red);
    if (threadIdx.x == 0) partials[blockIdx.x + gridDim.x * blockIdx.y] = s;
  }
}

struct StencilLaunch {
  dim3 grid, block;
  int chunk;
};

StencilLaunch stencil_config(const Geom& g) {
  StencilLaunch L{};
  const int target = 4 * 148;
  if (g.d == 3) {
    // ~16 waves of 2 resident CTAs per SM; marches of >= 16 layers so the
    // per-chunk halo layer stays cheap
    const int bx = (g.n[2] + BX3 - 2) / (BX3 - 1), by = (g.n[1] + BY3 - 2) / (BY3 - 1);
    int chunks = (16 * MINB3 * 148 + bx * by - 1) / (bx * by);
    chunks = std::max(1, std::min(chunks, g.n[0] / 16));
    L.chunk = (g.n[0] + chunks - 1) / chunks;
    chunks = (g.n[0] + L.chunk - 1) / L.chunk;
    L.grid = dim3(bx, by, chunks);
    L.block = dim3(BX3, BY3, 1);
  } else {
    // ~12 blocks of BX2 threads per SM in flight
    const int bx = (g.n[1] + BX2 - 2) / (BX2 - 1);
    int chunks = (3 * target + bx - 1) / bx;
    chunks = std::max(1, std::min(chunks, g.n[0]));
    L.chunk = (g.n[0] + chunks - 1) / chunks;
    chunks = (g.n[0] + L.chunk - 1) / L.chunk;
    L.grid = dim3(bx, chunks, 1);
    L.block = dim3(BX2, 1, 1);
  }
  return L;
}

template <int MODE, bool SCALE>
void launch_mode(const Geom& g, cudaStream_t s, const StencilLaunch& L, const double* u,
                 const double* rho, double lam, double mu, const EbarT& E, double* out,
                 double* partials, int ext, int nb = 1, int64_t bstride = 0,
                 const PcgState* st = nullptr, int ty0 = 0, int ty1 = -1) {
  if (g.d == 3) {
    static std::atomic<uint64_t> attr{0};  // per template instance and device
    set_smem_once(stencil3d<MODE, SCALE>, S3_BYTES, attr);
    dim3 grid = L.grid;
    grid.z *= nb;
    if (ty1 < 0) ty1 = (int)L.grid.y;
    grid.y = ty1 - ty0;
    stencil3d<MODE, SCALE><<<grid, L.block, S3_BYTES, s>>>(g, u, rho, lam, mu, E, out, partials,
                                                           L.chunk, ext, L.grid.z, bstride, st,
                                                           ty0, (int)L.grid.y);
  }
  else
    stencil2d<MODE, SCALE><<<L.grid, L.block, 0, s>>>(g, u, rho, lam, mu, E, out, partials,
                                                      L.chunk, 0);
  JF_LAUNCHED();
}

}  // namespace

int stencil_blocks(const Geom& g) {
  StencilLaunch L = stencil_config(g);
  return L.grid.x * L.grid.y * L.grid.z;
}

int launch_stencil(const Geom& g, cudaStream_t s, int mode, const double* u, const double* rho,
                   double lam, double mu, const double* ebar_mandel, double* out,
                   double* curv_partials, int ext) {
  require(!ext || g.d == 3, "halo-extended slabs are 3-D only");
  StencilLaunch L = stencil_config(g);
  const EbarT E = make_ebar(g.d, ebar_mandel);
  if (mode == ST_K) {
    if (g.iso) {
      // fold the two 1/h factors and the weight into the Lame constants
      const double sc = g.w * g.hinv[0] * g.hinv[0];
      launch_mode<VOX_K, false>(g, s, L, u, rho, lam * sc, mu * sc, E, out, curv_partials, ext);
    } else {
      launch_mode<VOX_K, true>(g, s, L, u, rho, lam * g.w, mu * g.w, E, out, curv_partials, ext);
    }
  } else if (mode == ST_RHS) {
    // f = -B^T W rho C E : negate through the Lame constants
    launch_mode<VOX_RHS, true>(g, s, L, u, rho, -lam * g.w, -mu * g.w, E, out, nullptr, ext);
  } else {
    launch_mode<VOX_RES, true>(g, s, L, u, rho, -lam * g.w, -mu * g.w, E, out, nullptr, ext);
  }
  return L.grid.x * L.grid.y * L.grid.z;
}

int stencil_tile_rows(const Geom& g) { return g.d == 3 ? (int)stencil_config(g).grid.y : 1; }
int stencil_tile_height(const Geom& g) { return g.d == 3 ? BY3 - 1 : 0; }

// K p on the 3-D tile rows [ty0, ty1) (output rows [ty0, ty1) x (BY3 - 1)),
// predicated on the PCG state; partials land at the full launch's indices
void launch_stencil_rows(const Geom& g, cudaStream_t s, const double* u, const double* rho,
                         double lam, double mu, double* out, double* curv_partials,
                         const PcgState* st, int ty0, int ty1) {
  require(g.d == 3, "row-group stencil is 3-D");
  StencilLaunch L = stencil_config(g);
  const EbarT E = make_ebar(3, nullptr);
  if (g.iso) {
    const double sc = g.w * g.hinv[0] * g.hinv[0];
    launch_mode<VOX_K, false>(g, s, L, u, rho, lam * sc, mu * sc, E, out, curv_partials, 0, 1, 0,
                              st, ty0, ty1);
  } else {
    launch_mode<VOX_K, true>(g, s, L, u, rho, lam * g.w, mu * g.w, E, out, curv_partials, 0, 1, 0,
                             st, ty0, ty1);
  }
}

// K u for nb right-hand sides bstride doubles apart (3-D, one launch; the
// partials of rhs b start at b * stencil_blocks(g))
int launch_stencil_batch(const Geom& g, cudaStream_t s, const double* u, const double* rho,
                         double lam, double mu, double* out, double* curv_partials, int nb,
                         int64_t bstride) {
  require(g.d == 3 || nb == 1, "batched stencil is 3-D");
  if (nb == 1) return launch_stencil(g, s, ST_K, u, rho, lam, mu, nullptr, out, curv_partials);
  StencilLaunch L = stencil_config(g);
  const EbarT E = make_ebar(g.d, nullptr);
  if (g.iso) {
    const double sc = g.w * g.hinv[0] * g.hinv[0];
    launch_mode<VOX_K, false>(g, s, L, u, rho, lam * sc, mu * sc, E, out, curv_partials, 0, nb,
                              bstride);
  } else {
    launch_mode<VOX_K, true>(g, s, L, u, rho, lam * g.w, mu * g.w, E, out, curv_partials, 0, nb,
                             bstride);
  }
  return L.grid.x * L.grid.y * L.grid.z;
}

// --------------------------------------------------------------------------
// total strain E + B u at the quadrature points (operators.py:79-83)
// --------------------------------------------------------------------------
template <int D>
__global__ void total_strain_kernel(Geom g, const double* __restrict__ u, EbarT E,
                                    double* __restrict__ out) {
  constexpr int C = 1 << D, T = n_simplex(D), M = mandel_m(D);
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < g.N;
       v += (int64_t)gridDim.x * blockDim.x) {
    int idx[3];
    int64_t rem = v;
    for (int a = D - 1; a >= 0; --a) { idx[a] = rem % g.n[a]; rem /= g.n[a]; }
    double uc[C][D];
#pragma unroll
    for (int c = 0; c < C; ++c) {
      int64_t node = 0;
#pragma unroll
      for (int a = 0; a < D; ++a) {
        int ia = idx[a] + ((c >> a) & 1);
        if (ia == g.n[a]) ia = 0;
        node = node * g.n[a] + ia;
      }
#pragma unroll
      for (int i = 0; i < D; ++i) uc[c][i] = __ldg(u + i * g.N + node);
    }
#pragma unroll
    for (int t = 0; t < T; ++t) {
      double G[D][D];
#pragma unroll
      for (int a = 0; a < D; ++a) {
        const int o = edge_base(D, t, a);
#pragma unroll
        for (int i = 0; i < D; ++i) G[i][a] = (uc[o | (1 << a)][i] - uc[o][i]) / g.h[a];
      }
#pragma unroll
      for (int m = 0; m < M; ++m) {
        const int i = mandel_i(D, m), j = mandel_j(D, m);
        double e = (i == j) ? G[i][i] : (G[i][j] + G[j][i]) / kSqrt2;
        e += E.m[m];
        out[((int64_t)m * T + t) * g.N + v] = e;
      }
    }
  }
}

void launch_total_strain(const Geom& g, cudaStream_t s, const double* u, const double* ebar,
                         double* out) {
  const EbarT E = make_ebar(g.d, ebar);
  const int blocks = (int)std::min<int64_t>((g.N + 255) / 256, 148 * 16);
  if (g.d == 3) total_strain_kernel<3><<<blocks, 256, 0, s>>>(g, u, E, out);
  else total_strain_kernel<2><<<blocks, 256, 0, s>>>(g, u, E, out);
  JF_LAUNCHED();
}

// --------------------------------------------------------------------------
// sum_Q rho C0 (E + B u): per-block partials (M values each)
// --------------------------------------------------------------------------
template <int D>
__global__ void stress_sum_kernel(Geom g, const double* __restrict__ u,
                                  const double* __restrict__ rho, double lam, double mu,
                                  EbarT E, double* __restrict__ partials) {
  constexpr int C = 1 << D, T = n_simplex(D), M = mandel_m(D);
  __shared__ double red[32];
  double acc[M];
#pragma unroll
  for (int m = 0; m < M; ++m) acc[m] = 0.0;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < g.N;
       v += (int64_t)gridDim.x * blockDim.x) {
    int idx[3];
    int64_t rem = v;
    for (int a = D - 1; a >= 0; --a) { idx[a] = rem % g.n[a]; rem /= g.n[a]; }
    double uc[C][D];
#pragma unroll
    for (int c = 0; c < C; ++c) {
      int64_t node = 0;
#pragma unroll
      for (int a = 0; a < D; ++a) {
        int ia = idx[a] + ((c >> a) & 1);
        if (ia == g.n[a]) ia = 0;
        node = node * g.n[a] + ia;
      }
#pragma unroll
      for (int i = 0; i < D; ++i) uc[c][i] = u ? __ldg(u + i * g.N + node) : 0.0;
    }
    const double r = __ldg(rho + v);
    double vs[M];
#pragma unroll
    for (int m = 0; m < M; ++m) vs[m] = 0.0;
#pragma unroll
    for (int t = 0; t < T; ++t) {
      double G[D][D];
#pragma unroll
      for (int a = 0; a < D; ++a) {
        const int o = edge_base(D, t, a);
#pragma unroll
        for (int i = 0; i < D; ++i)
          G[i][a] = (uc[o | (1 << a)][i] - uc[o][i]) / g.h[a] + E.e[i][a];
      }
      double tr = 0.0;
#pragma unroll
      for (int a = 0; a < D; ++a) tr += G[a][a];
#pragma unroll
      for (int m = 0; m < M; ++m) {
        const int i = mandel_i(D, m), j = mandel_j(D, m);
        // Mandel stress of C0 eps: diag lam tr + 2 mu e_ii; shear 2 mu e_m
        vs[m] += (i == j) ? lam * tr + 2.0 * mu * G[i][i]
                          : 2.0 * mu * (G[i][j] + G[j][i]) / kSqrt2;
      }
    }
#pragma unroll
    for (int m = 0; m < M; ++m) acc[m] += r * vs[m];
  }
#pragma unroll
  for (int m = 0; m < M; ++m) {
    const double s = block_sum(acc[m], red);
    if (threadIdx.x == 0) partials[blockIdx.x * M + m] = s;
    __syncthreads();
  }
}

int launch_stress_sum(const Geom& g, cudaStream_t s, const double* u, const double* rho,
                      double lam, double mu, const double* ebar, double* partials) {
  const EbarT E = make_ebar(g.d, ebar);
  const int blocks = kRedBlocks;
  if (g.d == 3) stress_sum_kernel<3><<<blocks, 256, 0, s>>>(g, u, rho, lam, mu, E, partials);
  else stress_sum_kernel<2><<<blocks, 256, 0, s>>>(g, u, rho, lam, mu, E, partials);
  JF_LAUNCHED();
  return blocks;
}

}  // namespace jfftb
