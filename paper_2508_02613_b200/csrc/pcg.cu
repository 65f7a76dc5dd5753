// PCG recurrence on device (solver.py:64-140).
//
// One iteration = stencil K p (+ fused <p, Kp> partials) -> alpha ->
// fused x/r update (+ D^-1/2 r, + <r, z> partials for jacobi/none) -> forward
// FFT -> fused Green block solve + Parseval quadratic forms -> termination /
// beta -> inverse FFT -> fused p update.  All scalars (alpha, beta, rz, the
// Green norm, the iteration count and the convergence flag) live on the
// device; every kernel of an iteration is predicated on `done`, so the host
// never needs a result before launching the next iteration.
#include <cstdlib>

#include "common.cuh"

namespace jfftb {

namespace {

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double block_sum1(double v, double* red) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  double s = 0.0;
  if (wid == 0) {
    s = lane < (int)(blockDim.x >> 5) ? red[lane] : 0.0;
    s = warp_sum(s);
  }
  return s;
}

// fixed-order sum of partials[b*stride + j], b < count, in one 1024-thread block
__device__ double sum_strided(const double* p, int count, int stride, int j, double* red) {
  // four independent running sums per thread (fixed order, loads in flight)
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  const int step = blockDim.x;
  int b = threadIdx.x;
  for (; b + 3 * step < count; b += 4 * step) {
    a0 += p[(int64_t)b * stride + j];
    a1 += p[(int64_t)(b + step) * stride + j];
    a2 += p[(int64_t)(b + 2 * step) * stride + j];
    a3 += p[(int64_t)(b + 3 * step) * stride + j];
  }
  for (; b < count; b += step) a0 += p[(int64_t)b * stride + j];
  double s = (a0 + a1) + (a2 + a3);
  s = block_sum1(s, red);
  __syncthreads();
  return s;  // valid in thread 0
}

// one block per right-hand side (blockIdx.x); pb: partials between them
__global__ void alpha_kernel(PcgState* st, const double* __restrict__ partials, int count,
                             int stride, int64_t pb) {
  __shared__ double red[32];
  st += blockIdx.x;
  partials += blockIdx.x * pb;
  if (st->done) {
    if (threadIdx.x == 0) st->xupd = 0;
    return;
  }
  const double curv = sum_strided(partials, count, stride, 0, red);
  if (threadIdx.x == 0) {
    st->curv = curv;
    st->xupd = 0;
    if (!isfinite(curv)) {
      st->status = JFFTB_ENONFINITE;
      st->done = 1;
    } else if (curv <= 0.0) {
      st->status = JFFTB_ECURVATURE;
      st->done = 1;
    } else {
      st->alpha = st->rz / curv;
      st->xupd = 1;
    }
  }
}

// x += alpha p ; r -= alpha Kp ; kind-specific extras (INIT: no x/r update)
template <int KIND, bool INIT>
__global__ void __launch_bounds__(256)
    update_kernel(int64_t n, const PcgState* __restrict__ st, double* __restrict__ x,
                  double* __restrict__ r, const double* __restrict__ p,
                  const double* __restrict__ kp, const double* __restrict__ dinv,
                  double* __restrict__ sz, double* __restrict__ partials) {
  __shared__ double red[32];
  if (st->done) return;
  const double alpha = st->alpha;
  double acc = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double ri = r[i];
    if (!INIT) {
      x[i] = x[i] + alpha * p[i];
      ri = ri - alpha * kp[i];
      r[i] = ri;
    }
    if (KIND == JFFTB_PC_GREEN_JACOBI) sz[i] = dinv[i] * ri;
    if (KIND == JFFTB_PC_JACOBI) {
      const double zi = dinv[i] * (dinv[i] * ri);
      sz[i] = zi;
      acc = fma(ri, zi, acc);
    }
    if (KIND == JFFTB_PC_NONE) acc = fma(ri, ri, acc);
  }
  if (KIND == JFFTB_PC_JACOBI || KIND == JFFTB_PC_NONE) {
    acc = block_sum1(acc, red);
    if (threadIdx.x == 0) partials[blockIdx.x] = acc;
  }
}

// termination test + beta (solver.py:122-135); INIT = the k = 0 check (99-110)
template <int KIND, bool INIT>
__global__ void finalize_kernel(PcgState* st, const double* __restrict__ spart, int scount,
                                int sstride, const double* __restrict__ upart, int ucount,
                                double* __restrict__ hist, int64_t sb = 0, int hb = 0) {
  __shared__ double red[32];
  // one block per right-hand side: sb partials, hb history entries apart
  st += blockIdx.x;
  spart += blockIdx.x * sb;
  hist += (int64_t)blockIdx.x * hb;
  if (st->done) return;
  const double q0 = sum_strided(spart, scount, sstride, 0, red);
  const double q1 = sum_strided(spart, scount, sstride, 1, red);
  double u0 = 0.0;
  if (KIND == JFFTB_PC_JACOBI || KIND == JFFTB_PC_NONE) u0 = sum_strided(upart, ucount, 1, 0, red);
  if (threadIdx.x != 0) return;
  int it = st->iters;
  if (!INIT) st->iters = ++it;
  const double g2 = q0;
  if (!isfinite(g2)) {
    st->status = JFFTB_ENONFINITE;
    st->done = 1;
    return;
  }
  hist[it] = g2;
  st->gnorm2 = g2;
  if (g2 <= st->eta) {
    st->done = 1;
    return;
  }
  const double rz_new = (KIND == JFFTB_PC_JACOBI || KIND == JFFTB_PC_NONE) ? u0 : q1;
  if (!isfinite(rz_new)) {
    st->status = JFFTB_ENONFINITE;
    st->done = 1;
    return;
  }
  if (!INIT) st->beta = rz_new / st->rz;
  st->rz = rz_new;
  if (it >= st->max_iter) st->done = 1;  // iteration cap: reported, not raised
}

// p = beta p + z  (INIT: p = z); z = D^-1/2 z' (green-jacobi), z' (green),
// r (none), D^-1 r (jacobi, precomputed in sz)
template <int KIND, bool INIT>
__global__ void __launch_bounds__(256)
    pupdate_kernel(int64_t n, const PcgState* __restrict__ st, double* __restrict__ p,
                   const double* __restrict__ zsrc, const double* __restrict__ dinv) {
  if (st->done) return;
  const double beta = st->beta;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double z = zsrc[i];
    if (KIND == JFFTB_PC_GREEN_JACOBI) z = dinv[i] * z;
    p[i] = INIT ? z : beta * p[i] + z;
  }
}

}  // namespace


static void run_fwd_fft(jfftb_grid* g, int batch2, double* in, double2* out) {
  cufftHandle plan = batch2 ? g->plan_fwd_2d : g->plan_fwd_d;
  JF_CUFFT(cufftSetStream(plan, g->stream));
  JF_CUFFT(cufftExecD2Z(plan, in, (cufftDoubleComplex*)out));
}
static void run_inv_fft(jfftb_grid* g, double2* in, double* out) {
  JF_CUFFT(cufftSetStream(g->plan_inv_d, g->stream));
  JF_CUFFT(cufftExecZ2D(g->plan_inv_d, (cufftDoubleComplex*)in, out));
}

static int grid_n(int64_t n) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, kRedBlocks));
}

// one pass of the preconditioner + termination functional; INIT = k = 0
template <int KIND, bool INIT>
static void pcg_precond_phase(jfftb_grid* g, jfftb_jacobi* jac, jfftb_green* gpc,
                              jfftb_green* gterm, const PcgBuffers& B) {
  const Geom& geo = g->geo;
  const int64_t n = geo.d * geo.N;
  cudaStream_t s = g->stream;
  const double* dinv = jac ? jac->inv_sqrt : nullptr;
  double* r = B.rs;
  double* sz = B.rs + n;
  update_kernel<KIND, INIT><<<kRedBlocks, 256, 0, s>>>(n, B.st, B.x, r, B.p, B.kp, dinv, sz,
                                                       B.upart);
  JF_LAUNCHED();
  if (!INIT) prof_mark(g);
  const int mode = KIND == JFFTB_PC_GREEN_JACOBI ? 1 : (KIND == JFFTB_PC_GREEN ? 0 : 2);
  run_fwd_fft(g, KIND == JFFTB_PC_GREEN_JACOBI, B.rs, B.spec);
  if (!INIT) prof_mark(g);
  launch_pcg_spectral(geo, s, mode, (mode == 2 ? gterm : gpc)->blocks, gterm->blocks, B.spec,
                      B.st, B.spart);
  if (!INIT) prof_mark(g);
  finalize_kernel<KIND, INIT><<<1, 1024, 0, s>>>(B.st, B.spart, kRedBlocks, 2, B.upart,
                                                 kRedBlocks, B.hist);
  JF_LAUNCHED();
  if (!INIT) prof_mark(g);
  const double* zsrc = r;
  if (KIND == JFFTB_PC_GREEN_JACOBI) {
    run_inv_fft(g, B.spec + geo.d * geo.Nh, sz);
    zsrc = sz;
  } else if (KIND == JFFTB_PC_GREEN) {
    run_inv_fft(g, B.spec, sz);
    zsrc = sz;
  } else if (KIND == JFFTB_PC_JACOBI) {
    zsrc = sz;
  }
  if (!INIT) prof_mark(g);
  pupdate_kernel<KIND, INIT><<<grid_n(n), 256, 0, s>>>(n, B.st, B.p, zsrc, dinv);
  JF_LAUNCHED();
  if (!INIT) {
    prof_mark(g);
    prof_end_iter(g);
  }
}

// The end of an iteration (3-D fused spectral kinds): pass I writes the new
// direction p_{k+1} (and x), then the NEXT iteration's stencil K p_{k+1} runs
// right away, predicated on the PCG state like every other pass, so the
// iterations queued past convergence cost nothing.  (Running the stencil in
// row groups on a side stream alongside pass I was measured: no gain at
// 512^3 -- 18.30 vs 18.14 ms per iteration -- the two do not co-reside on an
// SM and the board is power-capped.)
static void tail_I_KA(jfftb_op* op, jfftb_grid* g, int mode, const PcgBuffers& B,
                      const double2* z, const double* dinv) {
  const Geom& geo = g->geo;
  cudaStream_t s = g->stream;
  fused_stage_I(geo, s, mode, B.st, z, dinv, B.p, B.x, g->twiddle, Batch{});
  if (!g->prof)
    launch_stencil_rows(geo, s, B.p, op->rho, op->lambda0, op->mu0, B.kp, B.kpart, B.st, 0,
                        stencil_tile_rows(geo));
}

// Fused-spectral variant (power-of-two grids): green / green-jacobi run the
// five fused passes of fused.cu, the x update rides on the last one (pass I);
// none / jacobi keep their elementwise update and get the termination
// functional from a quad-only spectral pass.
template <int KIND, bool INIT>
static void pcg_precond_phase_fused(jfftb_op* op, jfftb_grid* g, jfftb_jacobi* jac,
                                    jfftb_green* gpc, jfftb_green* gterm, const PcgBuffers& B) {
  const Geom& geo = g->geo;
  const int64_t n = geo.d * geo.N;
  cudaStream_t s = g->stream;
  const double* dinv = jac ? jac->inv_sqrt : nullptr;
  const double2* tw = g->twiddle;
  double* r = B.rs;
  double* sz = B.rs + n;
  constexpr bool GJ = KIND == JFFTB_PC_GREEN_JACOBI;
  constexpr bool SPECTRAL_PC = GJ || KIND == JFFTB_PC_GREEN;
  constexpr int F = GJ ? 2 : 1;
  const bool bcb = SPECTRAL_PC && B.bcbq && fused_bcb_supported(geo);
  int scount;
  if (SPECTRAL_PC) {
    // r' = r - alpha Kp and its transform; green-jacobi adds s = D^-1/2 r'
    fused_stage_A(geo, s, F, INIT ? FUSED_INIT : FUSED_ITER, B.st, r, B.kp, dinv, B.spec, tw,
                  Batch{});
    if (!INIT) prof_mark(g);
    if (bcb) {
      // B, C and B' in one persistent kernel (the "spectral" stage of the profile)
      if (!INIT) prof_mark(g);
      scount = fused_stage_BCB(geo, s, F, B.st, gpc, gterm, B.spec, B.spart, tw, B.bcbq);
    } else {
      fused_stage_B(geo, s, false, B.st, B.spec, F * geo.d, tw, Batch{});
      if (!INIT) prof_mark(g);
      scount = fused_stage_C(geo, s, F, false, B.st, gpc, gterm, B.spec, B.spart, tw, Batch{});
    }
  } else {
    update_kernel<KIND, INIT><<<kRedBlocks, 256, 0, s>>>(n, B.st, B.x, r, B.p, B.kp, dinv, sz,
                                                         B.upart);
    JF_LAUNCHED();
    if (!INIT) prof_mark(g);
    fused_stage_A(geo, s, 1, FUSED_APPLY, B.st, r, nullptr, nullptr, B.spec, tw, Batch{});
    fused_stage_B(geo, s, false, B.st, B.spec, geo.d, tw, Batch{});
    if (!INIT) prof_mark(g);
    scount = fused_stage_C(geo, s, 1, true, B.st, gterm, gterm, B.spec, B.spart, tw, Batch{});
  }
  if (!INIT) prof_mark(g);
  finalize_kernel<KIND, INIT><<<1, 1024, 0, s>>>(B.st, B.spart, scount, 2, B.upart,
                                                 kRedBlocks, B.hist);
  JF_LAUNCHED();
  if (!INIT) prof_mark(g);
  if (SPECTRAL_PC) {
    double2* z = B.spec + (GJ ? geo.d * fused_component_stride(geo) : 0);
    if (!bcb) fused_stage_B(geo, s, true, B.st, z, geo.d, tw, Batch{});
    if (!INIT) prof_mark(g);
    if (g->geo.d == 3) {
      // pass I, then the next iteration's stencil
      tail_I_KA(op, g, INIT ? FUSED_INIT : FUSED_ITER, B, z, GJ ? dinv : nullptr);
    } else {
      fused_stage_I(geo, s, INIT ? FUSED_INIT : FUSED_ITER, B.st, z, GJ ? dinv : nullptr, B.p,
                    B.x, tw, Batch{});
    }
  } else {
    if (!INIT) prof_mark(g);
    pupdate_kernel<KIND, INIT><<<grid_n(n), 256, 0, s>>>(n, B.st, B.p,
                                                         KIND == JFFTB_PC_JACOBI ? sz : r, dinv);
    JF_LAUNCHED();
  }
  if (!INIT) {
    prof_mark(g);
    prof_end_iter(g);
  }
}

// the fused 3-D spectral kinds compute K p at the end of the previous
// iteration (tail_I_KA)
template <int KIND>
static constexpr bool ka_in_tail() {
  return KIND == JFFTB_PC_GREEN || KIND == JFFTB_PC_GREEN_JACOBI;
}

template <int KIND>
static void pcg_iteration(jfftb_op* op, jfftb_jacobi* jac, jfftb_green* gpc,
                          jfftb_green* gterm, const PcgBuffers& B) {
  jfftb_grid* g = op->grid;
  cudaStream_t s = g->stream;
  const bool tail = ka_in_tail<KIND>() && g->fused && g->geo.d == 3;
  prof_mark(g);
  if (!tail || g->prof)
    launch_stencil(g->geo, s, ST_K, B.p, op->rho, op->lambda0, op->mu0, nullptr, B.kp, B.kpart);
  prof_mark(g);
  alpha_kernel<<<1, 1024, 0, s>>>(B.st, B.kpart, B.kcount, 1, 0);
  JF_LAUNCHED();
  prof_mark(g);
  if (g->fused) pcg_precond_phase_fused<KIND, false>(op, g, jac, gpc, gterm, B);
  else pcg_precond_phase<KIND, false>(g, jac, gpc, gterm, B);
}

template <int KIND>
static void pcg_init(jfftb_op* op, jfftb_jacobi* jac, jfftb_green* gpc, jfftb_green* gterm,
                     const PcgBuffers& B) {
  if (op->grid->fused) pcg_precond_phase_fused<KIND, true>(op, op->grid, jac, gpc, gterm, B);
  else pcg_precond_phase<KIND, true>(op->grid, jac, gpc, gterm, B);
}

// ---- batched right-hand sides (jfftb_pcg_batch): the fused passes of the
// spectral kinds with one launch per stage for all L solves (grid dimension
// per right-hand side, per-solve device state); rho, D^-1/2 and the Green
// planes are shared by the L solves of a launch
template <int KIND, bool INIT>
static void pcg_phase_batch(jfftb_grid* g, jfftb_jacobi* jac, jfftb_green* gpc, jfftb_green* gterm,
                            const PcgBuffers& B, const Batch& bt) {
  const Geom& geo = g->geo;
  cudaStream_t s = g->stream;
  const double* dinv = jac ? jac->inv_sqrt : nullptr;
  const double2* tw = g->twiddle;
  constexpr bool GJ = KIND == JFFTB_PC_GREEN_JACOBI;
  constexpr int F = GJ ? 2 : 1;
  fused_stage_A(geo, s, F, INIT ? FUSED_INIT : FUSED_ITER, B.st, B.rs, B.kp, dinv, B.spec, tw, bt);
  fused_stage_B(geo, s, false, B.st, B.spec, F * geo.d, tw, bt);
  const int scount = fused_stage_C(geo, s, F, false, B.st, gpc, gterm, B.spec, B.spart, tw, bt);
  finalize_kernel<KIND, INIT><<<bt.L, 1024, 0, s>>>(B.st, B.spart, scount, 2, B.upart, kRedBlocks,
                                                    B.hist, 2 * (int64_t)scount, B.hstride);
  JF_LAUNCHED();
  double2* z = B.spec + (GJ ? geo.d * fused_component_stride(geo) : 0);
  fused_stage_B(geo, s, true, B.st, z, geo.d, tw, bt);
  fused_stage_I(geo, s, INIT ? FUSED_INIT : FUSED_ITER, B.st, z, GJ ? dinv : nullptr, B.p, B.x, tw,
                bt);
}

void pcg_dispatch_batch(int kind, bool init, jfftb_op* op, jfftb_jacobi* jac, jfftb_green* gpc,
                        jfftb_green* gterm, const PcgBuffers& B, const Batch& bt) {
  jfftb_grid* g = op->grid;
  require(g->fused && (kind == JFFTB_PC_GREEN || kind == JFFTB_PC_GREEN_JACOBI),
          "batched solves run the fused spectral kinds");
  if (!init) {
    launch_stencil_batch(g->geo, g->stream, B.p, op->rho, op->lambda0, op->mu0, B.kp, B.kpart, bt.L,
                         bt.vs);
    alpha_kernel<<<bt.L, 1024, 0, g->stream>>>(B.st, B.kpart, B.kcount, 1, B.kcount);
    JF_LAUNCHED();
  }
  if (kind == JFFTB_PC_GREEN_JACOBI) {
    init ? pcg_phase_batch<JFFTB_PC_GREEN_JACOBI, true>(g, jac, gpc, gterm, B, bt)
         : pcg_phase_batch<JFFTB_PC_GREEN_JACOBI, false>(g, jac, gpc, gterm, B, bt);
  } else {
    init ? pcg_phase_batch<JFFTB_PC_GREEN, true>(g, jac, gpc, gterm, B, bt)
         : pcg_phase_batch<JFFTB_PC_GREEN, false>(g, jac, gpc, gterm, B, bt);
  }
}

void launch_alpha(cudaStream_t s, PcgState* st, const double* partials, int count, int stride) {
  alpha_kernel<<<1, 1024, 0, s>>>(st, partials, count, stride, 0);
  JF_LAUNCHED();
}

void launch_finalize(int kind, bool init, cudaStream_t s, PcgState* st, const double* spart,
                     int scount, int sstride, double* hist) {
  require(kind == JFFTB_PC_GREEN || kind == JFFTB_PC_GREEN_JACOBI,
          "finalize: spectral kinds only");
  if (kind == JFFTB_PC_GREEN) {
    init ? finalize_kernel<JFFTB_PC_GREEN, true><<<1, 1024, 0, s>>>(st, spart, scount, sstride, nullptr, 0, hist)
         : finalize_kernel<JFFTB_PC_GREEN, false><<<1, 1024, 0, s>>>(st, spart, scount, sstride, nullptr, 0, hist);
  } else {
    init ? finalize_kernel<JFFTB_PC_GREEN_JACOBI, true><<<1, 1024, 0, s>>>(st, spart, scount, sstride, nullptr, 0, hist)
         : finalize_kernel<JFFTB_PC_GREEN_JACOBI, false><<<1, 1024, 0, s>>>(st, spart, scount, sstride, nullptr, 0, hist);
  }
  JF_LAUNCHED();
}

void pcg_dispatch(int kind, bool init, jfftb_op* op, jfftb_jacobi* jac, jfftb_green* gpc,
                  jfftb_green* gterm, const PcgBuffers& B) {
  switch (kind) {
    case JFFTB_PC_NONE:
      init ? pcg_init<JFFTB_PC_NONE>(op, jac, gpc, gterm, B)
           : pcg_iteration<JFFTB_PC_NONE>(op, jac, gpc, gterm, B);
      break;
    case JFFTB_PC_GREEN:
      init ? pcg_init<JFFTB_PC_GREEN>(op, jac, gpc, gterm, B)
           : pcg_iteration<JFFTB_PC_GREEN>(op, jac, gpc, gterm, B);
      break;
    case JFFTB_PC_JACOBI:
      init ? pcg_init<JFFTB_PC_JACOBI>(op, jac, gpc, gterm, B)
           : pcg_iteration<JFFTB_PC_JACOBI>(op, jac, gpc, gterm, B);
      break;
    default:
      init ? pcg_init<JFFTB_PC_GREEN_JACOBI>(op, jac, gpc, gterm, B)
           : pcg_iteration<JFFTB_PC_GREEN_JACOBI>(op, jac, gpc, gterm, B);
      break;
  }
}

}  // namespace jfftb
