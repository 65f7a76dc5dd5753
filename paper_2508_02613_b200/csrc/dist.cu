// Distributed (slab-decomposed) 3-D PCG: solver.py:64-140 with the fused
// Green / Green-Jacobi passes of fused.cu running per rank and the three
// exchange steps of the iteration as collectives.
//
// Decomposition (P ranks, n1 % P == 0, L1 = n1 / P):
//   real space  rank r owns axis-1 rows [r L1, (r + 1) L1) and all of axes 0
//               and 2: the stencil (one halo row of p per side), pass A
//               (axis-0 R2C of r' and s = D^-1/2 r') and pass I (axis-0 C2R,
//               x / p update) are local;
//   k space     rank r owns axis-0 frequency rows [k0lo_r, k0lo_r + kcnt_r)
//               of the n0/2 + 1 half-spectrum rows and all of axes 1 and 2:
//               pass B (axis-1 FFT), pass C (axis-2 FFT, Green block solve
//               with the k0-slab's Green planes, Parseval sums, inverse) and
//               pass B' are local.
// Per iteration: one halo exchange (two rows of p), one all-to-all of the
// 2d (green-jacobi) or d (green) half spectra after pass A and one of the d
// z^ spectra before pass I, and two all-gathers of per-rank partial sums
// (curvature; Green norm and rz).  Every rank sums the gathered partials in
// rank order, so alpha, beta and the termination decision are bitwise
// identical everywhere and no host synchronisation happens inside an
// iteration.  The all-to-all chunks are contiguous on both sides: pass A
// writes [field][k0][local columns], the receiver keeps one segment per
// source rank and passes B / C address the segments directly (fused.cu
// FGeom::row_off), so nothing is repacked.
//
// Transports: NCCL (one process per GPU, libnccl loaded at run time) or a
// loopback communicator that holds all P ranks in one process on one device
// (device-to-device copies, ranks issued one after the other on one stream,
// no kernel ever waits on another rank's): the decomposition is tested on a
// single GPU that way.
#include <dlfcn.h>
#include <nccl.h>

#include <chrono>
#include <cmath>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "fft.cuh"

namespace jfftb {
namespace {

// ---- NCCL, resolved at run time (the library never links it) --------------
struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    // prefer the copy already in the process (torch's), else the loader's
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW);
    if (!h) return a;
    auto sym = [&](const char* n) { return dlsym(h, n); };
    a.GetUniqueId = (decltype(a.GetUniqueId))sym("ncclGetUniqueId");
    a.CommInitRank = (decltype(a.CommInitRank))sym("ncclCommInitRank");
    a.CommDestroy = (decltype(a.CommDestroy))sym("ncclCommDestroy");
    a.GroupStart = (decltype(a.GroupStart))sym("ncclGroupStart");
    a.GroupEnd = (decltype(a.GroupEnd))sym("ncclGroupEnd");
    a.Send = (decltype(a.Send))sym("ncclSend");
    a.Recv = (decltype(a.Recv))sym("ncclRecv");
    a.AllGather = (decltype(a.AllGather))sym("ncclAllGather");
    a.GetErrorString = (decltype(a.GetErrorString))sym("ncclGetErrorString");
    return a;
  }();
  if (!api.GetUniqueId || !api.CommInitRank || !api.Send || !api.Recv || !api.AllGather ||
      !api.GroupStart || !api.GroupEnd)
    throw Error(JFFTB_ECUDA, "libnccl.so.2 could not be loaded");
  return api;
}

#define JF_NCCL(call)                                                                  \
  do {                                                                                 \
    ncclResult_t r_ = (call);                                                          \
    if (r_ != ncclSuccess)                                                             \
      throw ::jfftb::Error(JFFTB_ECUDA, std::string(#call) + ": " +                    \
                                            (nccl().GetErrorString ? nccl().GetErrorString(r_) \
                                                                   : "nccl error"));   \
  } while (0)

template <class F>
int guarded(F&& f) {
  try {
    f();
    return JFFTB_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return JFFTB_ECUDA;
  }
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) JF_CUDA(cudaSetDevice(dev));
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

// ---- small kernels -----------------------------------------------------------
int nblocks(int64_t n) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 16));
}

// comb probe of the Jacobi diagonal (preconditioners.py:109-115) on a
// halo-extended slab: ones on component alpha at nodes whose GLOBAL index
// parities equal offs (row e of the slab is global row row0 + e, mod n1)
__global__ void comb_ext_kernel(double* __restrict__ comb, int n0, int rows, int n2, int n1,
                                int row0, int alpha, int offs) {
  const int64_t per = (int64_t)n0 * rows * n2;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < 3 * per;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int comp = (int)(i / per);
    int64_t rem = i % per;
    const int i2 = (int)(rem % n2);
    rem /= n2;
    const int e = (int)(rem % rows);
    const int i0 = (int)(rem / rows);
    int g1 = (row0 + e) % n1;
    if (g1 < 0) g1 += n1;
    const bool on = comp == alpha && (i0 & 1) == (offs & 1) && (g1 & 1) == ((offs >> 1) & 1) &&
                    (i2 & 1) == ((offs >> 2) & 1);
    comb[i] = on ? 1.0 : 0.0;
  }
}
__global__ void comb_take_kernel(double* __restrict__ diag, const double* __restrict__ resp,
                                 int n0, int L1, int n2, int row0, int alpha, int offs) {
  const int64_t per = (int64_t)n0 * L1 * n2;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < per;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int i2 = (int)(v % n2);
    const int e = (int)((v / n2) % L1);
    const int i0 = (int)(v / ((int64_t)n2 * L1));
    const int g1 = row0 + e;
    if ((i0 & 1) == (offs & 1) && (g1 & 1) == ((offs >> 1) & 1) && (i2 & 1) == ((offs >> 2) & 1))
      diag[alpha * per + v] = resp[alpha * per + v];
  }
}
__global__ void jacobi_finish_kernel(double* __restrict__ diag, int64_t n, int* bad) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double v = diag[i];
    if (!(v >= 0.0) || !isfinite(v)) *bad = 1;
    if (v == 0.0) v = 1.0;
    diag[i] = 1.0 / sqrt(v);
  }
}
// x -= (sum over ranks of the gathered per-component sums, rank order) / N
__global__ void sub_gathered_mean_kernel(double* __restrict__ x, int64_t Nl,
                                         const double* __restrict__ gath, int P, double invN) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < 3 * Nl;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i / Nl);
    double s = 0.0;
    for (int q = 0; q < P; ++q) s += gath[q * 4 + c];
    x[i] -= s * invN;
  }
}
__global__ void comp_sum3_kernel(const double* __restrict__ x, int64_t Nl,
                                 double* __restrict__ part) {
  __shared__ double red[32];
  for (int c = 0; c < 3; ++c) {
    double s = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < Nl;
         i += (int64_t)gridDim.x * blockDim.x)
      s += x[c * Nl + i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) red[wid] = s;
    __syncthreads();
    if (wid == 0) {
      s = lane < (int)(blockDim.x >> 5) ? red[lane] : 0.0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
      if (lane == 0) part[blockIdx.x * 3 + c] = s;
    }
    __syncthreads();
  }
}

}  // namespace
}  // namespace jfftb

using namespace jfftb;

struct jfftb_comm {
  int world = 1;
  int rank = 0;      // this process's rank (NCCL); 0 for the loopback
  int device = 0;
  bool local = false;  // loopback: all ranks in this process
  ncclComm_t nc = nullptr;
};

namespace {

// one rank's device state
struct Rank {
  int r = 0;
  int k0lo = 0, kcnt = 0;
  double *rho_ext = nullptr, *dinv = nullptr, *x = nullptr, *rs = nullptr, *p_ext = nullptr,
         *kp = nullptr;
  double2 *spec = nullptr, *recv = nullptr;
  double* green = nullptr;
  double* hbuf = nullptr;  // halo staging: send lo, send hi, recv lo, recv hi (NCCL)
  double* part = nullptr;  // block partials (stencil / pass C / sums)
  double* mine = nullptr;  // this rank's reduced partials (4 doubles)
  double* gath = nullptr;  // gathered partials [P][4]
  PcgState* st = nullptr;
  double* hist = nullptr;
  int hist_cap = 0;
  std::vector<void*> allocs;
  double* alloc(size_t bytes) {
    void* p = nullptr;
    JF_CUDA(cudaMalloc(&p, bytes));
    allocs.push_back(p);
    return static_cast<double*>(p);
  }
};

}  // namespace

struct jfftb_dist {
  jfftb_comm* comm = nullptr;
  int n[3] = {0, 0, 0};
  double h[3] = {0, 0, 0};
  int P = 1, L1 = 0, kind = JFFTB_PC_GREEN_JACOBI;
  double lam0 = 0, mu0 = 0, lamr = 0, mur = 0;
  Geom gl{};      // one rank's real-space slab (n0, L1, n2)
  Geom gg{};      // the global grid
  cudaStream_t stream = nullptr;
  // exchange stream: the per-component all-to-alls run here, gated by events,
  // while `stream` transforms the next component (precond_phase)
  cudaStream_t xstream = nullptr;
  cudaEvent_t ev_c[3] = {nullptr, nullptr, nullptr};  // component c computed (stream)
  cudaEvent_t ev_x[3] = {nullptr, nullptr, nullptr};  // component c exchanged (xstream)
  bool overlap = true;
  double2* tw = nullptr;
  double* shared_gath = nullptr;  // loopback: the all-gather buffer all ranks share
  PcgState* host_st = nullptr;
  std::vector<Rank> ranks;        // 1 (NCCL) or P (loopback)
  int kcount = 0;                 // stencil partials per rank
  ~jfftb_dist() {
    for (auto& rk : ranks) {
      for (void* p : rk.allocs) cudaFree(p);
      if (rk.hist) cudaFree(rk.hist);
    }
    if (shared_gath) cudaFree(shared_gath);
    if (tw) cudaFree(tw);
    if (host_st) cudaFreeHost(host_st);
    for (int c = 0; c < 3; ++c) {
      if (ev_c[c]) cudaEventDestroy(ev_c[c]);
      if (ev_x[c]) cudaEventDestroy(ev_x[c]);
    }
    if (xstream) cudaStreamDestroy(xstream);
    if (stream) cudaStreamDestroy(stream);
  }
  int nf() const { return kind == JFFTB_PC_GREEN_JACOBI ? 6 : 3; }
  int64_t Nl() const { return gl.N; }
  int64_t Next() const { return (int64_t)n[0] * (L1 + 2) * n[2]; }
  int64_t PSl() const { return (int64_t)L1 * n[2]; }
  int K0() const { return n[0] / 2 + 1; }
  SpecSlab slab(const Rank& rk) const { return SpecSlab{rk.k0lo, rk.kcnt, L1, nf()}; }
  int k0lo_of(int q) const { return q * (n[0] / 2 / P); }
  int kcnt_of(int q) const { return n[0] / 2 / P + (q == P - 1 ? 1 : 0); }
};

namespace {

// ---- transport ---------------------------------------------------------------
struct P2P {
  int from, to;  // ranks
  const void* src;
  void* dst;     // for the loopback both are filled; for NCCL only the local side
  size_t bytes;
};

// a batch of point-to-point transfers between ranks.  Loopback: device copies
// (both ends are in this process).  NCCL: the local rank's sends and receives
// in one group (self transfers are copies).
void run_p2p(jfftb_dist* D, const std::vector<P2P>& xs, cudaStream_t s = nullptr) {
  jfftb_comm* c = D->comm;
  if (!s) s = D->stream;
  if (c->local) {
    for (const auto& x : xs)
      if (x.bytes && x.src != x.dst)
        JF_CUDA(cudaMemcpyAsync(x.dst, x.src, x.bytes, cudaMemcpyDeviceToDevice, s));
    return;
  }
  const NcclApi& N = nccl();
  JF_NCCL(N.GroupStart());
  for (const auto& x : xs) {
    if (!x.bytes) continue;
    if (x.from == c->rank && x.to == c->rank) {
      if (x.src != x.dst)
        JF_CUDA(cudaMemcpyAsync(x.dst, x.src, x.bytes, cudaMemcpyDeviceToDevice, s));
    } else if (x.from == c->rank) {
      JF_NCCL(N.Send(x.src, x.bytes, ncclUint8, x.to, c->nc, s));
    } else if (x.to == c->rank) {
      JF_NCCL(N.Recv(x.dst, x.bytes, ncclUint8, x.from, c->nc, s));
    }
  }
  JF_NCCL(N.GroupEnd());
}

// every rank's `m` (<= 4) partial sums in rk.mine -> rk.gath[P][4] on every rank
void allgather(jfftb_dist* D) {
  if (D->comm->local) return;  // the ranks wrote straight into the shared buffer
  Rank& rk = D->ranks[0];
  JF_NCCL(nccl().AllGather(rk.mine, rk.gath, 4, ncclDouble, D->comm->nc, D->stream));
}

// rank q (global index) is local here?
Rank* local_rank(jfftb_dist* D, int q) {
  if (D->comm->local) return &D->ranks[q];
  return D->ranks[0].r == q ? &D->ranks[0] : nullptr;
}

// halo rows of a halo-extended field (3 components, or 1 for rho): row 0
// <- the lower neighbour's last row, row L1 + 1 <- the upper neighbour's first
void halo_exchange(jfftb_dist* D, int ncomp, double* (*field)(Rank&)) {
  const int P = D->P, L1 = D->L1, n0 = D->n[0], n2 = D->n[2];
  const size_t rowb = (size_t)n2 * sizeof(double);
  const size_t pitch = (size_t)(L1 + 2) * n2 * sizeof(double);
  const int h = ncomp * n0;  // (component, i0) rows of one halo row
  cudaStream_t s = D->stream;
  if (D->comm->local) {
    for (auto& rk : D->ranks) {
      Rank& lo = D->ranks[(rk.r - 1 + P) % P];
      Rank& hi = D->ranks[(rk.r + 1) % P];
      double* f = field(rk);
      JF_CUDA(cudaMemcpy2DAsync(f, pitch, field(lo) + (size_t)L1 * n2, pitch, rowb, h,
                                cudaMemcpyDeviceToDevice, s));
      JF_CUDA(cudaMemcpy2DAsync(f + (size_t)(L1 + 1) * n2, pitch, field(hi) + n2, pitch, rowb, h,
                                cudaMemcpyDeviceToDevice, s));
    }
    return;
  }
  Rank& rk = D->ranks[0];
  double* f = field(rk);
  const size_t hb = (size_t)h * n2;
  double *send_lo = rk.hbuf, *send_hi = rk.hbuf + hb, *recv_lo = rk.hbuf + 2 * hb,
         *recv_hi = rk.hbuf + 3 * hb;
  // pack my first and last rows
  JF_CUDA(cudaMemcpy2DAsync(send_lo, rowb, f + n2, pitch, rowb, h, cudaMemcpyDeviceToDevice, s));
  JF_CUDA(cudaMemcpy2DAsync(send_hi, rowb, f + (size_t)L1 * n2, pitch, rowb, h,
                            cudaMemcpyDeviceToDevice, s));
  const int lo = (rk.r - 1 + P) % P, hi = (rk.r + 1) % P;
  // posting order fixes the NCCL match per peer pair (also when lo == hi)
  std::vector<P2P> xs = {{rk.r, hi, send_hi, nullptr, hb * sizeof(double)},
                         {rk.r, lo, send_lo, nullptr, hb * sizeof(double)},
                         {lo, rk.r, nullptr, recv_lo, hb * sizeof(double)},
                         {hi, rk.r, nullptr, recv_hi, hb * sizeof(double)}};
  if (P == 1) {
    xs = {{0, 0, send_hi, recv_lo, hb * sizeof(double)}, {0, 0, send_lo, recv_hi, hb * sizeof(double)}};
  }
  run_p2p(D, xs);
  JF_CUDA(cudaMemcpy2DAsync(f, pitch, recv_lo, rowb, rowb, h, cudaMemcpyDeviceToDevice, s));
  JF_CUDA(cudaMemcpy2DAsync(f + (size_t)(L1 + 1) * n2, pitch, recv_hi, rowb, rowb, h,
                            cudaMemcpyDeviceToDevice, s));
}

double* f_p(Rank& r) { return r.p_ext; }
double* f_rho(Rank& r) { return r.rho_ext; }

// forward all-to-all: rank r's pass-A spectra rows [k0lo_q, +kcnt_q) of
// every field -> rank q's segment r
// (the fields of component c: c, and d + c for green-jacobi; c < 0: all)
void alltoall_fwd(jfftb_dist* D, int c = -1, cudaStream_t s = nullptr) {
  const int P = D->P, nf = D->nf();
  const int64_t PSl = D->PSl(), CSl = (int64_t)D->K0() * PSl;
  std::vector<P2P> xs;
  for (int r = 0; r < P; ++r)
    for (int q = 0; q < P; ++q) {
      Rank* R = local_rank(D, r);
      Rank* Q = local_rank(D, q);
      if (!R && !Q) continue;
      const int k0lo = D->k0lo_of(q), kc = D->kcnt_of(q);
      const int64_t FS = (int64_t)kc * PSl, SS = nf * FS;
      for (int f = 0; f < nf; ++f) {
        if (c >= 0 && f % 3 != c) continue;
        xs.push_back({r, q, R ? R->spec + f * CSl + (int64_t)k0lo * PSl : nullptr,
                      Q ? Q->recv + r * SS + f * FS : nullptr, sizeof(double2) * FS});
      }
    }
  run_p2p(D, xs, s);
}

// backward: rank q's z^ fields (comps zq.. zq + 2) of segment r -> rank r's
// spectra rows [k0lo_q, +kcnt_q)
// (component cc of z^ only when cc >= 0)
void alltoall_bwd(jfftb_dist* D, int zq, int cc = -1, cudaStream_t s = nullptr) {
  const int P = D->P, nf = D->nf();
  const int64_t PSl = D->PSl(), CSl = (int64_t)D->K0() * PSl;
  std::vector<P2P> xs;
  for (int q = 0; q < P; ++q)
    for (int r = 0; r < P; ++r) {
      Rank* Q = local_rank(D, q);
      Rank* R = local_rank(D, r);
      if (!R && !Q) continue;
      const int k0lo = D->k0lo_of(q), kc = D->kcnt_of(q);
      const int64_t FS = (int64_t)kc * PSl, SS = nf * FS;
      for (int c = 0; c < 3; ++c) {
        if (cc >= 0 && c != cc) continue;
        xs.push_back({q, r, Q ? Q->recv + r * SS + (zq + c) * FS : nullptr,
                      R ? R->spec + (zq + c) * CSl + (int64_t)k0lo * PSl : nullptr,
                      sizeof(double2) * FS});
      }
    }
  run_p2p(D, xs, s);
}

// one PCG phase after the stencil: A, exchange, B, C, gather, finalize, B',
// exchange, I  (INIT: the k = 0 pass, no update).
//
// With more than one rank the two all-to-alls are pipelined against the
// passes on either side, component by component: pass A of component c + 1
// runs while component c's spectra travel (exchange stream, gated by events),
// pass B starts on the fields of a component as soon as they have landed,
// and on the way back pass B' / the exchange / pass I of the three z^
// components overlap the same way.  Only pass C needs every field.  The data
// and the arithmetic are those of the unpipelined schedule (JFFTB_DIST_OVERLAP=0),
// so the results are bitwise the same.
void precond_phase(jfftb_dist* D, bool init) {
  const bool GJ = D->kind == JFFTB_PC_GREEN_JACOBI;
  const int F = GJ ? 2 : 1, d = 3;
  cudaStream_t s = D->stream;
  const int mode = init ? FUSED_INIT : FUSED_ITER;
  const bool ov = D->overlap && D->P > 1;
  cudaStream_t sx = D->xstream;
  const int zq = GJ ? d : 0;
  const int64_t CSl = (int64_t)D->K0() * D->PSl();
  if (ov) {
    for (int c = 0; c < d; ++c) {
      for (auto& rk : D->ranks)
        fused_stage_A_comp(D->gl, s, F, mode, rk.st, rk.rs, rk.kp, GJ ? rk.dinv : nullptr, rk.spec,
                           D->tw, c);
      JF_CUDA(cudaEventRecord(D->ev_c[c], s));
      JF_CUDA(cudaStreamWaitEvent(sx, D->ev_c[c], 0));
      alltoall_fwd(D, c, sx);
      JF_CUDA(cudaEventRecord(D->ev_x[c], sx));
    }
    for (int c = 0; c < d; ++c) {
      JF_CUDA(cudaStreamWaitEvent(s, D->ev_x[c], 0));
      for (auto& rk : D->ranks)
        for (int f = 0; f < F; ++f)
          fused_stage_B_slab(D->gg, D->slab(rk), s, false, rk.st, rk.recv, f * d + c, 1, D->tw);
    }
  } else {
    for (auto& rk : D->ranks)
      fused_stage_A(D->gl, s, F, mode, rk.st, rk.rs, rk.kp, GJ ? rk.dinv : nullptr, rk.spec, D->tw,
                    Batch{});
    alltoall_fwd(D);
    for (auto& rk : D->ranks)
      fused_stage_B_slab(D->gg, D->slab(rk), s, false, rk.st, rk.recv, 0, F * d, D->tw);
  }
  for (auto& rk : D->ranks) {
    const int cnt =
        fused_stage_C_slab(D->gg, D->slab(rk), s, F, rk.st, rk.green, rk.recv, rk.part, D->tw);
    launch_sum_partials(s, rk.part, cnt, 2, rk.mine);
  }
  allgather(D);
  for (auto& rk : D->ranks) launch_finalize(D->kind, init, s, rk.st, rk.gath, D->P, 4, rk.hist);
  if (ov) {
    for (int c = 0; c < d; ++c) {
      for (auto& rk : D->ranks)
        fused_stage_B_slab(D->gg, D->slab(rk), s, true, rk.st, rk.recv, zq + c, 1, D->tw);
      JF_CUDA(cudaEventRecord(D->ev_c[c], s));
      JF_CUDA(cudaStreamWaitEvent(sx, D->ev_c[c], 0));
      alltoall_bwd(D, zq, c, sx);
      JF_CUDA(cudaEventRecord(D->ev_x[c], sx));
    }
    for (int c = 0; c < d; ++c) {
      JF_CUDA(cudaStreamWaitEvent(s, D->ev_x[c], 0));
      for (auto& rk : D->ranks)
        fused_stage_I_ext(D->gl, s, mode, rk.st, rk.spec + zq * CSl, GJ ? rk.dinv : nullptr,
                          rk.p_ext, rk.x, D->tw, c);
    }
  } else {
    for (auto& rk : D->ranks)
      fused_stage_B_slab(D->gg, D->slab(rk), s, true, rk.st, rk.recv, zq, d, D->tw);
    alltoall_bwd(D, zq);
    for (auto& rk : D->ranks)
      fused_stage_I_ext(D->gl, s, mode, rk.st, rk.spec + zq * CSl, GJ ? rk.dinv : nullptr,
                        rk.p_ext, rk.x, D->tw);
  }
}

void iteration(jfftb_dist* D) {
  cudaStream_t s = D->stream;
  halo_exchange(D, 3, f_p);
  for (auto& rk : D->ranks) {
    const int cnt = launch_stencil(D->gl, s, ST_K, rk.p_ext, rk.rho_ext, D->lam0, D->mu0, nullptr,
                                   rk.kp, rk.part, 1);
    launch_sum_partials(s, rk.part, cnt, 1, rk.mine);
  }
  allgather(D);
  for (auto& rk : D->ranks) launch_alpha(s, rk.st, rk.gath, D->P, 4);
  precond_phase(D, false);
}

void ensure_history(jfftb_dist* D, int max_iter) {
  for (auto& rk : D->ranks)
    if (rk.hist_cap < max_iter + 1) {
      if (rk.hist) cudaFree(rk.hist);
      rk.hist = nullptr;
      rk.hist_cap = 0;
      JF_CUDA(cudaMalloc(&rk.hist, sizeof(double) * std::max(max_iter + 1, 1024)));
      rk.hist_cap = std::max(max_iter + 1, 1024);
    }
}

size_t field_bytes(jfftb_dist* D) { return sizeof(double) * 3 * D->Nl(); }

}  // namespace

extern "C" {

int jfftb_comm_unique_id(char* id128) {
  return guarded([&] {
    require(id128 != nullptr, "null id buffer");
    ncclUniqueId id;
    JF_NCCL(nccl().GetUniqueId(&id));
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
    std::memcpy(id128, &id, sizeof(id));
  });
}

int jfftb_comm_create_nccl(const char* id128, int rank, int world, int device, jfftb_comm** out) {
  return guarded([&] {
    require(id128 && out, "null argument");
    require(world >= 1 && rank >= 0 && rank < world, "invalid rank / world size");
    DeviceGuard dg(device);
    ncclUniqueId id;
    std::memcpy(&id, id128, sizeof(id));
    auto* c = new jfftb_comm();
    c->world = world;
    c->rank = rank;
    c->device = device;
    try {
      JF_NCCL(nccl().CommInitRank(&c->nc, world, id, rank));
    } catch (...) {
      delete c;
      throw;
    }
    *out = c;
  });
}

int jfftb_comm_create_local(int world, int device, jfftb_comm** out) {
  return guarded([&] {
    require(out != nullptr, "null argument");
    require(world >= 1 && world <= 64, "invalid world size");
    auto* c = new jfftb_comm();
    c->world = world;
    c->device = device;
    c->local = true;
    *out = c;
  });
}

int jfftb_comm_destroy(jfftb_comm* c) {
  return guarded([&] {
    if (!c) return;
    if (c->nc) nccl().CommDestroy(c->nc);
    delete c;
  });
}

int jfftb_dist_create(jfftb_comm* comm, const int64_t* n, const double* lengths, const double* rho,
                      int where, double lambda0, double mu0, double lambda_ref, double mu_ref,
                      int kind, jfftb_dist** out) {
  return guarded([&] {
    require(comm && n && lengths && rho && out, "null argument");
    require(kind == JFFTB_PC_GREEN || kind == JFFTB_PC_GREEN_JACOBI,
            "distributed solves support the green and green-jacobi kinds");
    require(where == JFFTB_HOST || where == JFFTB_DEVICE, "where must be HOST or DEVICE");
    require(mu_ref > 0.0 && lambda_ref + mu_ref > 0.0, "stiffness not positive definite");
    const int P = comm->world;
    for (int a = 0; a < 3; ++a) {
      require(n[a] >= 16 && n[a] <= 2048 && (n[a] & (n[a] - 1)) == 0,
              "distributed solves need power-of-two grids, 16 <= n <= 2048");
      require(lengths[a] > 0.0 && std::isfinite(lengths[a]), "cell side lengths must be positive");
    }
    require(n[1] % P == 0 && n[1] / P >= 16, "n1 / world must be an integer >= 16");
    require(n[0] / 2 % P == 0 && n[0] / 2 / P >= 1, "n0 / 2 must be divisible by the world size");
    DeviceGuard dg(comm->device);
    auto* D = new jfftb_dist();
    try {
      D->comm = comm;
      D->P = P;
      D->kind = kind;
      D->lam0 = lambda0;
      D->mu0 = mu0;
      D->lamr = lambda_ref;
      D->mur = mu_ref;
      for (int a = 0; a < 3; ++a) {
        D->n[a] = (int)n[a];
        D->h[a] = lengths[a] / (double)n[a];
      }
      D->L1 = D->n[1] / P;
      auto mk = [&](int n1) {
        Geom g{};
        g.d = 3;
        g.n[0] = D->n[0];
        g.n[1] = n1;
        g.n[2] = D->n[2];
        g.N = (int64_t)g.n[0] * g.n[1] * g.n[2];
        g.nh = g.n[2] / 2 + 1;
        g.Nh = g.N / g.n[2] * g.nh;
        for (int a = 0; a < 3; ++a) {
          g.h[a] = D->h[a];
          g.hinv[a] = 1.0 / D->h[a];
        }
        g.w = D->h[0] * D->h[1] * D->h[2] / 6.0;
        g.iso = D->h[0] == D->h[1] && D->h[1] == D->h[2];
        return g;
      };
      D->gl = mk(D->L1);
      D->gg = mk(D->n[1]);
      JF_CUDA(cudaStreamCreateWithFlags(&D->stream, cudaStreamNonBlocking));
      JF_CUDA(cudaStreamCreateWithFlags(&D->xstream, cudaStreamNonBlocking));
      for (int c = 0; c < 3; ++c) {
        JF_CUDA(cudaEventCreateWithFlags(&D->ev_c[c], cudaEventDisableTiming));
        JF_CUDA(cudaEventCreateWithFlags(&D->ev_x[c], cudaEventDisableTiming));
      }
      if (const char* e = std::getenv("JFFTB_DIST_OVERLAP")) D->overlap = e[0] != '0';
      JF_CUDA(cudaMalloc(&D->tw, sizeof(double2) * kTwiddleN));
      launch_twiddles(D->stream, D->tw);
      JF_CUDA(cudaMallocHost(&D->host_st, sizeof(PcgState)));
      D->kcount = stencil_blocks(D->gl);
      const int nloc = comm->local ? P : 1;
      if (comm->local) JF_CUDA(cudaMalloc(&D->shared_gath, sizeof(double) * 4 * P));
      const int64_t Nl = D->Nl(), Next = D->Next(), PSl = D->PSl();
      const int nf = D->nf();
      D->ranks.resize(nloc);
      for (int i = 0; i < nloc; ++i) {
        Rank& rk = D->ranks[i];
        rk.r = comm->local ? i : comm->rank;
        rk.k0lo = D->k0lo_of(rk.r);
        rk.kcnt = D->kcnt_of(rk.r);
        rk.rho_ext = rk.alloc(sizeof(double) * Next);
        rk.dinv = rk.alloc(sizeof(double) * 3 * Nl);
        rk.x = rk.alloc(sizeof(double) * 3 * Nl);
        rk.rs = rk.alloc(sizeof(double) * 6 * Nl);
        rk.p_ext = rk.alloc(sizeof(double) * 3 * Next);
        JF_CUDA(cudaMemsetAsync(rk.p_ext, 0, sizeof(double) * 3 * Next, D->stream));
        rk.kp = rk.alloc(sizeof(double) * 3 * Nl);
        rk.spec = reinterpret_cast<double2*>(rk.alloc(sizeof(double2) * nf * D->K0() * PSl));
        // one rank: the received layout [src][field][k0][i1][i2] IS pass A's
        // [field][k0][columns], so the spectra are not exchanged at all
        rk.recv = P == 1 ? rk.spec
                         : reinterpret_cast<double2*>(rk.alloc(
                               sizeof(double2) * (size_t)nf * rk.kcnt * D->n[1] * D->n[2]));
        rk.green = rk.alloc(sizeof(double) * 9 * (size_t)rk.kcnt * D->n[1] * D->n[2]);
        if (!comm->local) rk.hbuf = rk.alloc(sizeof(double) * 4 * 3 * D->n[0] * D->n[2]);
        rk.part = rk.alloc(sizeof(double) * std::max(D->kcount, 2 * kFusedMaxBlocks + 8 * kRedBlocks));
        if (comm->local) {
          rk.gath = D->shared_gath;
          rk.mine = D->shared_gath + 4 * rk.r;
        } else {
          rk.mine = rk.alloc(sizeof(double) * 4);
          rk.gath = rk.alloc(sizeof(double) * 4 * P);
        }
        rk.st = reinterpret_cast<PcgState*>(rk.alloc(sizeof(PcgState)));
        // density: the rank's slab (n0, L1, n2) into the interior rows
        const double* src = rho + (comm->local ? (size_t)i * Nl : 0);
        JF_CUDA(cudaMemcpy2DAsync(rk.rho_ext + D->n[2], sizeof(double) * (D->L1 + 2) * D->n[2],
                                  src, sizeof(double) * PSl, sizeof(double) * PSl, D->n[0],
                                  where == JFFTB_HOST ? cudaMemcpyHostToDevice
                                                      : cudaMemcpyDeviceToDevice,
                                  D->stream));
      }
      halo_exchange(D, 1, f_rho);
      // Green planes of each rank's k0-slab (preconditioners.py:50-80): the
      // impulse responses of K_ref on a 4^3 cell of the same pixel size
      Geom sm = D->gg;
      sm.n[0] = sm.n[1] = sm.n[2] = 4;
      sm.N = 64;
      sm.nh = 3;
      sm.Nh = 48;
      double *imp = nullptr, *resp = nullptr;
      JF_CUDA(cudaMalloc(&imp, sizeof(double) * 3 * 64));
      JF_CUDA(cudaMalloc(&resp, sizeof(double) * 9 * 64));
      for (int beta = 0; beta < 3; ++beta) {
        JF_CUDA(cudaMemsetAsync(imp, 0, sizeof(double) * 3 * 64, D->stream));
        const double one = 1.0;
        JF_CUDA(cudaMemcpyAsync(imp + beta * 64, &one, sizeof(double), cudaMemcpyHostToDevice,
                                D->stream));
        launch_stencil(sm, D->stream, ST_K, imp, nullptr, lambda_ref, mu_ref, nullptr,
                       resp + beta * 3 * 64, nullptr);
        JF_CUDA(cudaStreamSynchronize(D->stream));
      }
      for (auto& rk : D->ranks)
        launch_green_setup(D->gg, D->stream, resp, 4 | (4 << 8) | (4 << 16), rk.green, 1,
                           (int64_t)rk.kcnt * D->n[1] * D->n[2], fused_dif(), rk.k0lo);
      JF_CUDA(cudaStreamSynchronize(D->stream));
      cudaFree(imp);
      cudaFree(resp);
      // Jacobi diagonal: d 2^d comb probes through the slab stencil
      // (preconditioners.py:97-119); combs are built from global indices, so
      // they need no exchange
      if (kind == JFFTB_PC_GREEN_JACOBI) {
        double *comb = nullptr, *kresp = nullptr;
        int* bad = nullptr;
        JF_CUDA(cudaMalloc(&comb, sizeof(double) * 3 * Next));
        JF_CUDA(cudaMalloc(&kresp, sizeof(double) * 3 * Nl));
        JF_CUDA(cudaMalloc(&bad, sizeof(int)));
        JF_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), D->stream));
        for (auto& rk : D->ranks) {
          const int row0 = rk.r * D->L1 - 1;
          for (int alpha = 0; alpha < 3; ++alpha)
            for (int offs = 0; offs < 8; ++offs) {
              comb_ext_kernel<<<nblocks(3 * Next), 256, 0, D->stream>>>(
                  comb, D->n[0], D->L1 + 2, D->n[2], D->n[1], row0, alpha, offs);
              JF_LAUNCHED();
              launch_stencil(D->gl, D->stream, ST_K, comb, rk.rho_ext, lambda0, mu0, nullptr, kresp,
                             nullptr, 1);
              comb_take_kernel<<<nblocks(Nl), 256, 0, D->stream>>>(
                  rk.dinv, kresp, D->n[0], D->L1, D->n[2], rk.r * D->L1, alpha, offs);
              JF_LAUNCHED();
            }
          jacobi_finish_kernel<<<nblocks(3 * Nl), 256, 0, D->stream>>>(rk.dinv, 3 * Nl, bad);
          JF_LAUNCHED();
        }
        int hbad = 0;
        JF_CUDA(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, D->stream));
        JF_CUDA(cudaStreamSynchronize(D->stream));
        cudaFree(comb);
        cudaFree(kresp);
        cudaFree(bad);
        require(!hbad, "probed diagonal has negative or non-finite entries");
      }
      JF_CUDA(cudaStreamSynchronize(D->stream));
    } catch (...) {
      delete D;
      throw;
    }
    *out = D;
  });
}

int jfftb_dist_destroy(jfftb_dist* D) {
  return guarded([&] {
    if (!D) return;
    DeviceGuard dg(D->comm->device);
    cudaStreamSynchronize(D->stream);
    delete D;
  });
}

// f = -B^T W rho C0 E on every local slab (operators.py:61-76)
int jfftb_dist_assemble_rhs(jfftb_dist* D, const double* eps_bar, double* out, int where) {
  return guarded([&] {
    require(D && eps_bar && out, "null argument");
    for (int k = 0; k < 6; ++k) require(std::isfinite(eps_bar[k]), "macroscopic strain must be finite");
    DeviceGuard dg(D->comm->device);
    const size_t fb = field_bytes(D);
    double* tmp = nullptr;
    JF_CUDA(cudaMalloc(&tmp, fb));
    for (size_t i = 0; i < D->ranks.size(); ++i) {
      Rank& rk = D->ranks[i];
      launch_stencil(D->gl, D->stream, ST_RHS, nullptr, rk.rho_ext, D->lam0, D->mu0, eps_bar, tmp,
                     nullptr, 1);
      JF_CUDA(cudaMemcpyAsync(reinterpret_cast<char*>(out) + i * fb, tmp, fb,
                              where == JFFTB_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice,
                              D->stream));
    }
    JF_CUDA(cudaStreamSynchronize(D->stream));
    cudaFree(tmp);
  });
}

int jfftb_dist_jacobi_export(jfftb_dist* D, double* out, int where) {
  return guarded([&] {
    require(D && out, "null argument");
    require(D->kind == JFFTB_PC_GREEN_JACOBI, "no Jacobi diagonal for this kind");
    DeviceGuard dg(D->comm->device);
    const size_t fb = field_bytes(D);
    for (size_t i = 0; i < D->ranks.size(); ++i)
      JF_CUDA(cudaMemcpyAsync(reinterpret_cast<char*>(out) + i * fb, D->ranks[i].dinv, fb,
                              where == JFFTB_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice,
                              D->stream));
    JF_CUDA(cudaStreamSynchronize(D->stream));
  });
}

// pcg (solver.py:64-140) over the local slabs: rhs / x_out hold the local
// ranks' slabs back to back (one slab for NCCL, P for the loopback);
// history_out (host) receives the (rank-identical) residual history
int jfftb_dist_pcg(jfftb_dist* D, const double* rhs, int where, double eta, int max_iter,
                   double* x_out, double* history_out, int* iterations, int* terminated,
                   double* wall_s) {
  const auto t0 = std::chrono::steady_clock::now();
  return guarded([&] {
    require(D && rhs && history_out && iterations && terminated, "null argument");
    require(max_iter >= 0, "max_iter must be >= 0");
    require(where == JFFTB_HOST || where == JFFTB_DEVICE, "where must be HOST or DEVICE");
    DeviceGuard dg(D->comm->device);
    cudaStream_t s = D->stream;
    ensure_history(D, max_iter);
    const size_t fb = field_bytes(D);
    const cudaMemcpyKind h2d = where == JFFTB_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
    PcgState h0{};
    h0.eta = eta;
    h0.max_iter = max_iter;
    *D->host_st = h0;
    for (size_t i = 0; i < D->ranks.size(); ++i) {
      Rank& rk = D->ranks[i];
      JF_CUDA(cudaMemcpyAsync(rk.st, D->host_st, sizeof(PcgState), cudaMemcpyHostToDevice, s));
      JF_CUDA(cudaMemsetAsync(rk.x, 0, fb, s));
      JF_CUDA(cudaMemcpyAsync(rk.rs, reinterpret_cast<const char*>(rhs) + i * fb, fb, h2d, s));
    }
    auto poll = [&]() {
      JF_CUDA(cudaMemcpyAsync(D->host_st, D->ranks[0].st, sizeof(PcgState), cudaMemcpyDeviceToHost, s));
      JF_CUDA(cudaStreamSynchronize(s));
      return D->host_st->done != 0;
    };
    precond_phase(D, true);
    bool done = poll();
    int batch = 1;
    while (!done) {
      for (int k = 0; k < batch; ++k) iteration(D);
      done = poll();
      batch = std::min(batch * 2, 8);
    }
    const PcgState hs = *D->host_st;
    *iterations = hs.iters;
    JF_CUDA(cudaMemcpyAsync(history_out, D->ranks[0].hist, sizeof(double) * (hs.iters + 1),
                            cudaMemcpyDeviceToHost, s));
    JF_CUDA(cudaStreamSynchronize(s));
    if (hs.status != JFFTB_OK)
      throw Error(hs.status, hs.status == JFFTB_ECURVATURE
                                 ? "non-positive search-direction curvature in PCG"
                                 : "PCG recurrence became non-finite");
    *terminated = hs.gnorm2 <= eta ? JFFTB_CONVERGED : JFFTB_ITERATION_CAP;
    // mean subtraction over the whole grid (solver.py:138)
    for (auto& rk : D->ranks) {
      comp_sum3_kernel<<<kRedBlocks, 256, 0, s>>>(rk.x, D->Nl(), rk.part);
      JF_LAUNCHED();
      launch_sum_partials(s, rk.part, kRedBlocks, 3, rk.mine);
    }
    allgather(D);
    const double invN = 1.0 / ((double)D->n[0] * D->n[1] * D->n[2]);
    for (size_t i = 0; i < D->ranks.size(); ++i) {
      Rank& rk = D->ranks[i];
      sub_gathered_mean_kernel<<<nblocks(3 * D->Nl()), 256, 0, s>>>(rk.x, D->Nl(), rk.gath, D->P,
                                                                    invN);
      JF_LAUNCHED();
      if (x_out)
        JF_CUDA(cudaMemcpyAsync(reinterpret_cast<char*>(x_out) + i * fb, rk.x, fb,
                                where == JFFTB_HOST ? cudaMemcpyDeviceToHost
                                                    : cudaMemcpyDeviceToDevice,
                                s));
    }
    JF_CUDA(cudaStreamSynchronize(s));
    if (wall_s)
      *wall_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  });
}

int jfftb_dist_info(jfftb_dist* D, int64_t* info8) {
  return guarded([&] {
    require(D && info8, "null argument");
    info8[0] = D->P;
    info8[1] = D->L1;
    info8[2] = (int64_t)D->ranks.size();
    info8[3] = D->ranks[0].r;
    info8[4] = D->ranks[0].k0lo;
    info8[5] = D->ranks[0].kcnt;
    info8[6] = D->Nl();
    info8[7] = D->comm->local ? 1 : 0;
  });
}

}  // extern "C"
