// C ABI of libjfftb200.so (include/jfftb200.h): handle lifetime, host/device
// staging, preconditioner setup, and the PCG driver loop.
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "fft.cuh"

namespace jfftb {


namespace {

thread_local std::string g_last_error;
thread_local int64_t g_launches = 0;

// RAII device buffer on a stream
struct DevBuf {
  void* ptr = nullptr;
  DevBuf() = default;
  explicit DevBuf(size_t bytes) { reset(bytes); }
  void reset(size_t bytes) {
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    if (bytes) JF_CUDA(cudaMalloc(&ptr, bytes));
  }
  ~DevBuf() {
    if (ptr) cudaFree(ptr);
  }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  template <class T>
  T* as() const {
    return static_cast<T*>(ptr);
  }
};

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

template <class F>
int guarded(F&& f) {
  try {
    f();
    return JFFTB_OK;
  } catch (const Error& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return JFFTB_ECUDA;
  } catch (...) {
    g_last_error = "unknown error";
    return JFFTB_ECUDA;
  }
}

// Stage an input array onto the device: device pointers pass through, host
// arrays are copied into `tmp`.
const double* stage_in(jfftb_grid* g, const double* src, size_t count, int where, DevBuf& tmp) {
  require(src != nullptr, "null input array");
  if (where == JFFTB_DEVICE) return src;
  require(where == JFFTB_HOST, "where must be JFFTB_HOST or JFFTB_DEVICE");
  tmp.reset(count * sizeof(double));
  copy_h2d(g, tmp.ptr, src, count * sizeof(double), g->stream);
  return tmp.as<double>();
}
double* stage_out(double* dst, size_t count, int where, DevBuf& tmp) {
  require(dst != nullptr, "null output array");
  if (where == JFFTB_DEVICE) return dst;
  require(where == JFFTB_HOST, "where must be JFFTB_HOST or JFFTB_DEVICE");
  tmp.reset(count * sizeof(double));
  return tmp.as<double>();
}
void finish_out(jfftb_grid* g, double* dst, const double* dev, size_t count, int where) {
  if (where == JFFTB_HOST) copy_d2h(g, dst, dev, count * sizeof(double), g->stream);
}

double* ensure_partials(jfftb_grid* g, int count) {
  if (g->partials_cap < count) {
    if (g->partials) JF_CUDA(cudaFree(g->partials));
    JF_CUDA(cudaMalloc(&g->partials, sizeof(double) * count));
    g->partials_cap = count;
  }
  return g->partials;
}

void ensure_plans(jfftb_grid* g) {
  if (g->plans_ready) return;
  const Geom& geo = g->geo;
  long long n[3] = {geo.n[0], geo.n[1], geo.n[2]};
  size_t w1 = 0, w2 = 0, w3 = 0;
  JF_CUFFT(cufftCreate(&g->plan_fwd_d));
  JF_CUFFT(cufftCreate(&g->plan_inv_d));
  JF_CUFFT(cufftCreate(&g->plan_fwd_2d));
  for (cufftHandle h : {g->plan_fwd_d, g->plan_inv_d, g->plan_fwd_2d})
    JF_CUFFT(cufftSetAutoAllocation(h, 0));
  JF_CUFFT(cufftMakePlanMany64(g->plan_fwd_d, geo.d, n, nullptr, 1, geo.N, nullptr, 1, geo.Nh,
                               CUFFT_D2Z, geo.d, &w1));
  JF_CUFFT(cufftMakePlanMany64(g->plan_inv_d, geo.d, n, nullptr, 1, geo.Nh, nullptr, 1, geo.N,
                               CUFFT_Z2D, geo.d, &w2));
  JF_CUFFT(cufftMakePlanMany64(g->plan_fwd_2d, geo.d, n, nullptr, 1, geo.N, nullptr, 1, geo.Nh,
                               CUFFT_D2Z, 2 * geo.d, &w3));
  g->fft_work_bytes = std::max(std::max(w1, w2), w3);
  if (g->fft_work_bytes) JF_CUDA(cudaMalloc(&g->fft_work, g->fft_work_bytes));
  for (cufftHandle h : {g->plan_fwd_d, g->plan_inv_d, g->plan_fwd_2d})
    JF_CUFFT(cufftSetWorkArea(h, g->fft_work));
  g->plans_ready = true;
}

__global__ void scale_kernel(double* x, double a, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    x[i] *= a;
}

__global__ void check_rho_kernel(const double* rho, int64_t n, int* bad) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    if (!(rho[i] >= 0.0)) *bad = 1;  // negative or NaN
}

// ---------------------------------------------------------------------------
// Jacobi probing (preconditioners.py:97-119)
// ---------------------------------------------------------------------------
__global__ void comb_kernel(double* __restrict__ comb, Geom g, int alpha, int offs) {
  // comb = 0 except ones on component alpha at nodes with i_a % 2 == o_a
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < g.d * g.N;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int comp = (int)(i / g.N);
    int64_t rem = i % g.N;
    bool on = comp == alpha;
    for (int a = g.d - 1; a >= 0; --a) {
      const int ia = (int)(rem % g.n[a]);
      rem /= g.n[a];
      on = on && ((ia & 1) == ((offs >> a) & 1));
    }
    comb[i] = on ? 1.0 : 0.0;
  }
}
__global__ void comb_extract_kernel(double* __restrict__ diag, const double* __restrict__ resp,
                                    Geom g, int alpha, int offs) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < g.N;
       v += (int64_t)gridDim.x * blockDim.x) {
    int64_t rem = v;
    bool on = true;
    for (int a = g.d - 1; a >= 0; --a) {
      const int ia = (int)(rem % g.n[a]);
      rem /= g.n[a];
      on = on && ((ia & 1) == ((offs >> a) & 1));
    }
    if (on) diag[alpha * g.N + v] = resp[alpha * g.N + v];
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

int nblk(int64_t n) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 16));
}

int read_flag(jfftb_grid* g, int* dflag) {
  int h = 0;
  JF_CUDA(cudaMemcpyAsync(&h, dflag, sizeof(int), cudaMemcpyDeviceToHost, g->stream));
  JF_CUDA(cudaStreamSynchronize(g->stream));
  return h;
}

// PCG workspace, allocated once per grid (and regrown only for a longer
// history): x, [r; s], p, Kp, 2d half spectra, state, history, partials
PcgBuffers pcg_workspace(jfftb_grid* g, int kcount, int max_iter) {
  const Geom& geo = g->geo;
  const int64_t n = geo.d * geo.N;
  auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
  const size_t need_hist = sizeof(double) * (size_t)(max_iter + 1);
  const int64_t nspec = std::max<int64_t>(geo.Nh, spec_elems(g));
  const bool bcb = g->fused && fused_bcb_supported(geo);
  const int sblocks = (int)std::max<int64_t>(std::max(kRedBlocks, kFusedMaxBlocks),
                                             bcb ? fused_bcb_partials(geo) : 0);
  const size_t qbytes = sizeof(unsigned) * (2 + 3 * (size_t)(geo.n[0] / 2 + 1));
  const size_t fixed = al(sizeof(double) * n) * 3 + al(sizeof(double) * 2 * n) +
                       al(sizeof(double2) * 2 * geo.d * nspec) + al(sizeof(PcgState)) +
                       al(sizeof(double) * (kcount + 2 * sblocks + kRedBlocks)) + al(qbytes);
  const size_t total = fixed + al(need_hist);
  if (g->ws_bytes < total) {
    if (g->ws) JF_CUDA(cudaFree(g->ws));
    g->ws = nullptr;
    g->ws_bytes = 0;
    JF_CUDA(cudaMalloc(&g->ws, total + al(sizeof(double) * 1024)));  // history headroom
    g->ws_bytes = total + al(sizeof(double) * 1024);
  }
  if (!g->ws_host) JF_CUDA(cudaMallocHost(&g->ws_host, sizeof(PcgState)));
  char* p = static_cast<char*>(g->ws);
  auto take = [&](size_t b) {
    char* q = p;
    p += al(b);
    return q;
  };
  PcgBuffers B{};
  B.x = (double*)take(sizeof(double) * n);
  B.rs = (double*)take(sizeof(double) * 2 * n);
  B.p = (double*)take(sizeof(double) * n);
  B.kp = (double*)take(sizeof(double) * n);
  B.spec = (double2*)take(sizeof(double2) * 2 * geo.d * nspec);
  B.st = (PcgState*)take(sizeof(PcgState));
  B.kpart = (double*)take(sizeof(double) * (kcount + 2 * sblocks + kRedBlocks));
  B.spart = B.kpart + kcount;
  B.upart = B.spart + 2 * sblocks;
  B.kcount = kcount;
  B.bcbq = bcb ? (unsigned*)take(qbytes) : nullptr;
  if (!bcb) take(qbytes);
  B.hist = (double*)p;
  return B;
}

// workspace of a batched solve (L right-hand sides; spectral kinds on the
// fused path): per solve x, r, p, Kp (d N each), 2d spectra, state, history
PcgBuffers pcg_workspace_batch(jfftb_grid* g, int kcount, int max_iter, int L, Batch& bt) {
  const Geom& geo = g->geo;
  const int64_t n = geo.d * geo.N;
  auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
  const int64_t nspec = spec_elems(g);
  const int hstride = max_iter + 1;
  const size_t total = al(sizeof(double) * n * L) * 4 + al(sizeof(double2) * 2 * geo.d * nspec * L) +
                       al(sizeof(PcgState) * L) +
                       al(sizeof(double) * ((size_t)kcount * L + 2 * kFusedMaxBlocks + kRedBlocks)) +
                       al(sizeof(double) * hstride * L);
  if (g->wsb_bytes < total) {
    if (g->wsb) JF_CUDA(cudaFree(g->wsb));
    g->wsb = nullptr;
    g->wsb_bytes = 0;
    JF_CUDA(cudaMalloc(&g->wsb, total));
    g->wsb_bytes = total;
  }
  if (g->wsb_L < L) {
    if (g->wsb_host) JF_CUDA(cudaFreeHost(g->wsb_host));
    g->wsb_host = nullptr;
    JF_CUDA(cudaMallocHost(&g->wsb_host, sizeof(PcgState) * L));
    g->wsb_L = L;
  }
  char* p = static_cast<char*>(g->wsb);
  auto take = [&](size_t b) {
    char* q = p;
    p += al(b);
    return q;
  };
  PcgBuffers B{};
  B.x = (double*)take(sizeof(double) * n * L);
  B.rs = (double*)take(sizeof(double) * n * L);
  B.p = (double*)take(sizeof(double) * n * L);
  B.kp = (double*)take(sizeof(double) * n * L);
  B.spec = (double2*)take(sizeof(double2) * 2 * geo.d * nspec * L);
  B.st = (PcgState*)take(sizeof(PcgState) * L);
  B.kpart = (double*)take(sizeof(double) * ((size_t)kcount * L + 2 * kFusedMaxBlocks + kRedBlocks));
  B.spart = B.kpart + (size_t)kcount * L;
  B.upart = B.spart + 2 * kFusedMaxBlocks;
  B.kcount = kcount;
  B.hist = (double*)take(sizeof(double) * hstride * L);
  B.hstride = hstride;
  bt.L = L;
  bt.vs = n;
  bt.bss = 2 * geo.d * nspec;
  return B;
}

bool graphs_enabled() {
  static const bool v = [] {
    const char* e = std::getenv("JFFTB_GRAPHS");
    return !(e && e[0] == '0');
  }();
  return v;
}

void drop_iteration_graph(jfftb_grid* g) {
  if (g->iter_graph) cudaGraphExecDestroy(g->iter_graph);
  g->iter_graph = nullptr;
  g->iter_kind = -1;
}

// replay (capturing first if needed) one PCG iteration as a CUDA graph; the
// graph bakes in every pointer of the iteration, so it is keyed on them
void run_iteration_graph(jfftb_grid* g, int kind, jfftb_op* op, jfftb_jacobi* jac,
                         jfftb_green* gpc, jfftb_green* gterm, const PcgBuffers& B) {
  constexpr int kIterKey = jfftb_grid::kIterKey;
  const void* key[kIterKey] = {op, op->rho, jac, jac ? jac->inv_sqrt : nullptr, gpc->blocks,
                               gterm->blocks, B.x, B.st, B.hist, g->stream, B.bcbq};
  const double lame[6] = {op->lambda0, op->mu0, gpc->lambda_ref, gpc->mu_ref,
                          gterm->lambda_ref, gterm->mu_ref};
  bool hit = g->iter_graph != nullptr && g->iter_kind == kind;
  for (int i = 0; hit && i < 6; ++i) hit = g->iter_lame[i] == lame[i];
  for (int i = 0; hit && i < kIterKey; ++i) hit = g->iter_key[i] == key[i];
  if (!hit) {
    drop_iteration_graph(g);
    cudaGraph_t graph = nullptr;
    const int64_t before = g_launches;
    // capture on the grid's own stream (the caller's may be the legacy
    // default stream, which cannot be captured); the graph is launched on
    // the caller's stream below
    cudaStream_t user = g->stream;
    JF_CUDA(cudaStreamSynchronize(user));
    g->stream = g->own_stream;
    JF_CUDA(cudaStreamBeginCapture(g->stream, cudaStreamCaptureModeThreadLocal));
    try {
      pcg_dispatch(kind, false, op, jac, gpc, gterm, B);
    } catch (...) {
      cudaStreamEndCapture(g->stream, &graph);
      if (graph) cudaGraphDestroy(graph);
      g->stream = user;
      throw;
    }
    const cudaError_t ec = cudaStreamEndCapture(g->stream, &graph);
    g->stream = user;
    JF_CUDA(ec);
    g->iter_launches = (int)(g_launches - before);
    g_launches = before;
    const cudaError_t e = cudaGraphInstantiate(&g->iter_graph, graph, 0);
    cudaGraphDestroy(graph);
    JF_CUDA(e);
    for (int i = 0; i < kIterKey; ++i) g->iter_key[i] = key[i];
    g->iter_kind = kind;
    for (int i = 0; i < 6; ++i) g->iter_lame[i] = lame[i];
  }
  JF_CUDA(cudaGraphLaunch(g->iter_graph, g->stream));
  count_launch(g->iter_launches);
}

// precondition r (device, d*N) into out (device) for kind (-1 = jacobi half)
void precond_device(int kind, jfftb_green* green, jfftb_jacobi* jac, jfftb_grid* g,
                    const double* r, double* out) {
  const Geom& geo = g->geo;
  const int64_t n = geo.d * geo.N;
  cudaStream_t s = g->stream;
  auto need_jac = [&]() { require(jac != nullptr, "kind needs an assembled Jacobi diagonal"); };
  auto need_green = [&]() { require(green != nullptr, "kind needs an assembled Green operator"); };
  if (kind == JFFTB_PC_NONE) {
    launch_copy(s, out, r, n);
  } else if (kind == -1) {
    need_jac();
    launch_mul(s, out, jac->inv_sqrt, r, n);
  } else if (kind == JFFTB_PC_JACOBI) {
    need_jac();
    launch_mul2(s, out, jac->inv_sqrt, r, n);
  } else if (kind == JFFTB_PC_GREEN || kind == JFFTB_PC_GREEN_JACOBI) {
    need_green();
    if (kind == JFFTB_PC_GREEN_JACOBI) need_jac();
    if (g->fused) {
      DevBuf spec(sizeof(double2) * geo.d * spec_elems(g));
      fused_precond_apply(geo, s, green,
                          kind == JFFTB_PC_GREEN_JACOBI ? jac->inv_sqrt : nullptr, r, out,
                          spec.as<double2>(), g->twiddle);
      JF_CUDA(cudaStreamSynchronize(s));  // spec is freed on return
      return;
    }
    ensure_plans(g);
    DevBuf spec(sizeof(double2) * geo.d * geo.Nh);
    DevBuf tmp(kind == JFFTB_PC_GREEN_JACOBI ? sizeof(double) * n : 0);
    const double* src = r;
    if (kind == JFFTB_PC_GREEN_JACOBI) {
      launch_mul(s, tmp.as<double>(), jac->inv_sqrt, r, n);
      src = tmp.as<double>();
    }
    JF_CUFFT(cufftSetStream(g->plan_fwd_d, s));
    JF_CUFFT(cufftExecD2Z(g->plan_fwd_d, const_cast<double*>(src), spec.as<cufftDoubleComplex>()));
    launch_green_apply(geo, s, green->blocks, spec.as<double2>(), spec.as<double2>(), 1);
    JF_CUFFT(cufftSetStream(g->plan_inv_d, s));
    JF_CUFFT(cufftExecZ2D(g->plan_inv_d, spec.as<cufftDoubleComplex>(), out));
    if (kind == JFFTB_PC_GREEN_JACOBI) launch_mul(s, out, jac->inv_sqrt, out, n);
    JF_CUDA(cudaStreamSynchronize(s));  // spec/tmp are freed on return
  } else {
    require(false, "unknown preconditioner kind");
  }
}

}  // namespace

void set_last_error(const std::string& m) { g_last_error = m; }
void count_launch(int n) { g_launches += n; }

void prof_mark(jfftb_grid* g) {
  if (!g->prof) return;
  cudaEvent_t e;
  if (g->ev_free.empty()) {
    JF_CUDA(cudaEventCreate(&e));
  } else {
    e = g->ev_free.back();
    g->ev_free.pop_back();
  }
  JF_CUDA(cudaEventRecord(e, g->stream));
  g->ev_cur.push_back(e);
}

void prof_end_iter(jfftb_grid* g) {
  if (!g->prof) return;
  g->ev_pending.push_back(g->ev_cur);
  g->ev_cur.clear();
  ++g->prof_seq;
}

// Accumulate the stage times of issued iterations whose sequence number is
// <= real_iters (the solve's true iteration count); the stream must be idle.
void prof_collect(jfftb_grid* g, int64_t real_iters, bool final) {
  if (!g->prof) return;
  size_t keep = 0;
  std::vector<std::vector<cudaEvent_t>> rest;
  for (auto& ev : g->ev_pending) {
    const int64_t seq = g->prof_done_seq + 1;
    if (seq <= real_iters && ev.size() == JFFTB_N_STAGES + 1) {
      for (int k = 0; k < JFFTB_N_STAGES; ++k) {
        float ms = 0.f;
        JF_CUDA(cudaEventElapsedTime(&ms, ev[k], ev[k + 1]));
        g->prof_ms[k] += ms;
      }
      ++g->prof_iters;
      ++g->prof_done_seq;
      for (auto e : ev) g->ev_free.push_back(e);
    } else if (final) {
      for (auto e : ev) g->ev_free.push_back(e);
    } else {
      rest.push_back(ev);
      ++keep;
    }
  }
  g->ev_pending.swap(rest);
  if (final) {
    g->prof_seq = g->prof_done_seq = 0;
    for (auto e : g->ev_cur) g->ev_free.push_back(e);
    g->ev_cur.clear();
  }
  (void)keep;
}

}  // namespace jfftb

using namespace jfftb;

extern "C" {

const char* jfftb_last_error(void) { return g_last_error.c_str(); }
int jfftb_version(void) { return 100; }
int64_t jfftb_launch_count(int reset) {
  const int64_t v = g_launches;
  if (reset) g_launches = 0;
  return v;
}

int jfftb_grid_create(int d, const int64_t* n, const double* lengths, int device,
                      jfftb_grid** out) {
  return guarded([&] {
    require(out != nullptr && n != nullptr && lengths != nullptr, "null argument");
    require(d == 2 || d == 3, "only d = 2 and d = 3 are supported");
    int ndev = 0;
    JF_CUDA(cudaGetDeviceCount(&ndev));
    require(device >= 0 && device < ndev, "invalid CUDA device");
    Geom geo{};
    geo.d = d;
    geo.N = 1;
    for (int a = 0; a < 3; ++a) geo.n[a] = 1;
    for (int a = 0; a < d; ++a) {
      require(n[a] >= 2 && n[a] < (1 << 20), "grid needs n >= 2 nodes per direction");
      require(lengths[a] > 0.0 && std::isfinite(lengths[a]), "cell side lengths must be positive");
      geo.n[a] = (int)n[a];
      geo.N *= n[a];
      geo.h[a] = lengths[a] / (double)n[a];
      geo.hinv[a] = 1.0 / geo.h[a];
    }
    geo.nh = geo.n[d - 1] / 2 + 1;
    geo.Nh = geo.N / geo.n[d - 1] * geo.nh;
    double vol = 1.0;
    for (int a = 0; a < d; ++a) vol *= geo.h[a];
    geo.w = vol / (d == 2 ? 2.0 : 6.0);
    geo.iso = true;
    for (int a = 1; a < d; ++a) geo.iso = geo.iso && geo.h[a] == geo.h[0];
    DeviceGuard dg(device);
    auto* g = new jfftb_grid();
    g->geo = geo;
    g->device = device;
    if (cudaStreamCreateWithFlags(&g->own_stream, cudaStreamNonBlocking) != cudaSuccess) {
      delete g;
      throw Error(JFFTB_ECUDA, "cudaStreamCreate failed");
    }
    g->stream = g->own_stream;
    JF_CUDA(cudaMalloc(&g->dscal, 64 * sizeof(double)));
    // JFFTB_DISABLE_FUSED=1 forces the cuFFT spectral path (A/B testing)
    const char* nofuse = std::getenv("JFFTB_DISABLE_FUSED");
    g->fused = fused_supported(geo) && !(nofuse && nofuse[0] == '1');
    if (g->fused) {
      JF_CUDA(cudaMalloc(&g->twiddle, sizeof(double2) * kTwiddleN));
      launch_twiddles(g->own_stream, g->twiddle);
      JF_CUDA(cudaStreamSynchronize(g->own_stream));
    }
    *out = g;
  });
}

namespace {
void grid_free(jfftb_grid* g) {
    DeviceGuard dg(g->device);
    cudaStreamSynchronize(g->stream);
    if (g->plans_ready) {
      cufftDestroy(g->plan_fwd_d);
      cufftDestroy(g->plan_inv_d);
      cufftDestroy(g->plan_fwd_2d);
    }
    if (g->fft_work) cudaFree(g->fft_work);
    if (g->partials) cudaFree(g->partials);
    if (g->dscal) cudaFree(g->dscal);
    if (g->ws) cudaFree(g->ws);
    if (g->ws_host) cudaFreeHost(g->ws_host);
    if (g->wsb) cudaFree(g->wsb);
    if (g->wsb_host) cudaFreeHost(g->wsb_host);
    if (g->twiddle) cudaFree(g->twiddle);
    free_host_staging(g);
    drop_iteration_graph(g);
    prof_collect(g, 0, true);
    for (auto e : g->ev_free) cudaEventDestroy(e);
    cudaStreamDestroy(g->own_stream);
    delete g;
}
void grid_release(jfftb_grid* g) {
  if (g->refs.fetch_sub(1) == 1 && g->closed.load()) grid_free(g);
}
void op_free(jfftb_op* op) {
  jfftb_grid* g = op->grid;
  {
    DeviceGuard dg(g->device);
    cudaStreamSynchronize(g->stream);
    drop_iteration_graph(g);  // it bakes in op->rho
    cudaFree(op->rho);
  }
  delete op;
  grid_release(g);
}
void op_release(jfftb_op* op) {
  if (op->refs.fetch_sub(1) == 1 && op->closed.load()) op_free(op);
}
}  // namespace

// Destroying a grid (or an operator) that still has live children -- an
// operator, a Green operator, a Jacobi diagonal -- defers the release to the
// last child's destroy, so handles may be dropped in any order.
int jfftb_grid_destroy(jfftb_grid* g) {
  return guarded([&] {
    if (!g) return;
    g->closed.store(true);
    if (g->refs.load() == 0) grid_free(g);
  });
}

int jfftb_grid_set_stream(jfftb_grid* g, void* stream) {
  return guarded([&] {
    require(g != nullptr, "null grid");
    g->stream = stream ? (cudaStream_t)stream : g->own_stream;
  });
}

int jfftb_grid_synchronize(jfftb_grid* g) {
  return guarded([&] {
    require(g != nullptr, "null grid");
    DeviceGuard dg(g->device);
    JF_CUDA(cudaStreamSynchronize(g->stream));
  });
}

int jfftb_fft_forward(jfftb_grid* g, const double* u, double* spec, int where) {
  return guarded([&] {
    require(g != nullptr, "null grid");
    DeviceGuard dg(g->device);
    const Geom& geo = g->geo;
    ensure_plans(g);
    DevBuf tin, tout;
    const double* du = stage_in(g, u, geo.d * geo.N, where, tin);
    double* ds = stage_out(spec, 2 * geo.d * geo.Nh, where, tout);
    JF_CUFFT(cufftSetStream(g->plan_fwd_d, g->stream));
    JF_CUFFT(cufftExecD2Z(g->plan_fwd_d, const_cast<double*>(du), (cufftDoubleComplex*)ds));
    finish_out(g, spec, ds, 2 * geo.d * geo.Nh, where);
    JF_CUDA(cudaStreamSynchronize(g->stream));
  });
}

int jfftb_fft_inverse(jfftb_grid* g, const double* spec, double* u, int where) {
  return guarded([&] {
    require(g != nullptr, "null grid");
    DeviceGuard dg(g->device);
    const Geom& geo = g->geo;
    ensure_plans(g);
    DevBuf tin, tout, work(sizeof(double2) * geo.d * geo.Nh);
    const double* ds = stage_in(g, spec, 2 * geo.d * geo.Nh, where, tin);
    double* du = stage_out(u, geo.d * geo.N, where, tout);
    // Z2D overwrites its input: transform a copy
    JF_CUDA(cudaMemcpyAsync(work.ptr, ds, sizeof(double2) * geo.d * geo.Nh,
                            cudaMemcpyDeviceToDevice, g->stream));
    JF_CUFFT(cufftSetStream(g->plan_inv_d, g->stream));
    JF_CUFFT(cufftExecZ2D(g->plan_inv_d, work.as<cufftDoubleComplex>(), du));
    scale_kernel<<<nblk(geo.d * geo.N), 256, 0, g->stream>>>(du, 1.0 / (double)geo.N,
                                                              geo.d * geo.N);
    JF_LAUNCHED();
    finish_out(g, u, du, geo.d * geo.N, where);
    JF_CUDA(cudaStreamSynchronize(g->stream));
  });
}

int jfftb_op_create(jfftb_grid* g, const double* rho, int where, double lambda0, double mu0,
                    jfftb_op** out) {
  return guarded([&] {
    require(g != nullptr && out != nullptr, "null argument");
    require(std::isfinite(lambda0) && std::isfinite(mu0), "non-finite material");
    DeviceGuard dg(g->device);
    const Geom& geo = g->geo;
    DevBuf tin;
    const double* dr = stage_in(g, rho, geo.N, where, tin);
    double* own = nullptr;
    JF_CUDA(cudaMalloc(&own, sizeof(double) * geo.N));
    JF_CUDA(cudaMemcpyAsync(own, dr, sizeof(double) * geo.N, cudaMemcpyDeviceToDevice, g->stream));
    int* bad = (int*)g->dscal;
    JF_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), g->stream));
    check_rho_kernel<<<nblk(geo.N), 256, 0, g->stream>>>(own, geo.N, bad);
    JF_LAUNCHED();
    if (read_flag(g, bad)) {
      cudaFree(own);
      throw Error(JFFTB_EINVAL, "negative density");
    }
    auto* op = new jfftb_op();
    g->refs.fetch_add(1);
    op->grid = g;
    op->rho = own;
    op->lambda0 = lambda0;
    op->mu0 = mu0;
    *out = op;
  });
}

int jfftb_op_destroy(jfftb_op* op) {
  return guarded([&] {
    if (!op) return;
    op->closed.store(true);
    if (op->refs.load() == 0) op_free(op);
  });
}

int jfftb_apply_system(jfftb_op* op, const double* u, double* out, int where) {
  return guarded([&] {
    require(op != nullptr, "null operator");
    jfftb_grid* g = op->grid;
    DeviceGuard dg(g->device);
    const int64_t n = g->geo.d * g->geo.N;
    DevBuf tin, tout;
    const double* du = stage_in(g, u, n, where, tin);
    double* dout = stage_out(out, n, where, tout);
    require(du != dout, "apply_system cannot run in place");
    launch_stencil(g->geo, g->stream, ST_K, du, op->rho, op->lambda0, op->mu0, nullptr, dout,
                   nullptr);
    finish_out(g, out, dout, n, where);
  });
}

static void check_ebar(int d, const double* eps_bar) {
  require(eps_bar != nullptr, "null macroscopic strain");
  const int m = d == 2 ? 3 : 6;
  for (int k = 0; k < m; ++k)
    require(std::isfinite(eps_bar[k]), "macroscopic strain must be finite");
}

int jfftb_assemble_rhs(jfftb_op* op, const double* eps_bar, double* out, int where) {
  return guarded([&] {
    require(op != nullptr, "null operator");
    jfftb_grid* g = op->grid;
    check_ebar(g->geo.d, eps_bar);
    DeviceGuard dg(g->device);
    const int64_t n = g->geo.d * g->geo.N;
    DevBuf tout;
    double* dout = stage_out(out, n, where, tout);
    launch_stencil(g->geo, g->stream, ST_RHS, nullptr, op->rho, op->lambda0, op->mu0, eps_bar,
                   dout, nullptr);
    finish_out(g, out, dout, n, where);
  });
}

int jfftb_total_strain(jfftb_op* op, const double* u, const double* eps_bar, double* out,
                       int where) {
  return guarded([&] {
    require(op != nullptr, "null operator");
    jfftb_grid* g = op->grid;
    check_ebar(g->geo.d, eps_bar);
    DeviceGuard dg(g->device);
    const Geom& geo = g->geo;
    const int M = geo.d == 2 ? 3 : 6, T = geo.d == 2 ? 2 : 6;
    DevBuf tin, tout;
    const double* du = stage_in(g, u, geo.d * geo.N, where, tin);
    double* dout = stage_out(out, (size_t)M * T * geo.N, where, tout);
    launch_total_strain(geo, g->stream, du, eps_bar, dout);
    finish_out(g, out, dout, (size_t)M * T * geo.N, where);
  });
}

int jfftb_residual_force(jfftb_op* op, const double* u, const double* eps_bar, double* out,
                         int where) {
  return guarded([&] {
    require(op != nullptr, "null operator");
    jfftb_grid* g = op->grid;
    check_ebar(g->geo.d, eps_bar);
    DeviceGuard dg(g->device);
    const int64_t n = g->geo.d * g->geo.N;
    DevBuf tin, tout;
    const double* du = stage_in(g, u, n, where, tin);
    double* dout = stage_out(out, n, where, tout);
    require(du != dout, "residual_force cannot run in place");
    launch_stencil(g->geo, g->stream, ST_RES, du, op->rho, op->lambda0, op->mu0, eps_bar, dout,
                   nullptr);
    finish_out(g, out, dout, n, where);
  });
}

int jfftb_homogenized_stress(jfftb_op* op, const double* u, const double* eps_bar,
                             double* sigma_out, int where) {
  return guarded([&] {
    require(op != nullptr && sigma_out != nullptr, "null argument");
    jfftb_grid* g = op->grid;
    check_ebar(g->geo.d, eps_bar);
    DeviceGuard dg(g->device);
    const Geom& geo = g->geo;
    const int M = geo.d == 2 ? 3 : 6;
    DevBuf tin;
    const double* du = stage_in(g, u, geo.d * geo.N, where, tin);
    double* part = ensure_partials(g, kRedBlocks * M + M);
    const int cnt = launch_stress_sum(geo, g->stream, du, op->rho, op->lambda0, op->mu0,
                                      eps_bar, part);
    launch_sum_partials(g->stream, part, cnt, M, part + kRedBlocks * M);
    double sums[6];
    JF_CUDA(cudaMemcpyAsync(sums, part + kRedBlocks * M, sizeof(double) * M,
                            cudaMemcpyDeviceToHost, g->stream));
    JF_CUDA(cudaStreamSynchronize(g->stream));
    double vol = 1.0;
    for (int a = 0; a < geo.d; ++a) vol *= geo.h[a] * geo.n[a];
    const double scale = geo.w / vol;
    for (int m = 0; m < M; ++m) sigma_out[m] = scale * sums[m];
  });
}

int jfftb_green_create(jfftb_grid* g, double lambda_ref, double mu_ref, jfftb_green** out) {
  return guarded([&] {
    require(g != nullptr && out != nullptr, "null argument");
    require(mu_ref > 0.0 && lambda_ref + mu_ref > 0.0,
            "stiffness not positive definite");
    DeviceGuard dg(g->device);
    const Geom& geo = g->geo;
    // impulse responses of K_ref (rho = 1) on a small periodic grid that has
    // the same pixel size: the stencil radius is 1, so for n >= 3 the
    // response around node 0 is identical to the full grid's
    Geom sm = geo;
    int m[3] = {1, 1, 1};
    sm.N = 1;
    for (int a = 0; a < geo.d; ++a) {
      m[a] = std::min(geo.n[a], 4);
      sm.n[a] = m[a];
      sm.N *= m[a];
    }
    sm.nh = sm.n[geo.d - 1] / 2 + 1;
    sm.Nh = sm.N / sm.n[geo.d - 1] * sm.nh;
    const int d = geo.d;
    DevBuf imp(sizeof(double) * d * sm.N), resp(sizeof(double) * d * d * sm.N);
    for (int beta = 0; beta < d; ++beta) {
      JF_CUDA(cudaMemsetAsync(imp.ptr, 0, sizeof(double) * d * sm.N, g->stream));
      const double one = 1.0;
      JF_CUDA(cudaMemcpyAsync(imp.as<double>() + beta * sm.N, &one, sizeof(double),
                              cudaMemcpyHostToDevice, g->stream));
      launch_stencil(sm, g->stream, ST_K, imp.as<double>(), nullptr, lambda_ref, mu_ref, nullptr,
                     resp.as<double>() + (int64_t)beta * d * sm.N, nullptr);
    }
    auto* gr = new jfftb_green();
    gr->grid = g;
    gr->lambda_ref = lambda_ref;
    gr->mu_ref = mu_ref;
    const int np = green_planes(d);
    const int64_t nfreq = spec_elems(g);
    gr->nfreq = nfreq;
    if (cudaMalloc(&gr->blocks, sizeof(double) * np * nfreq) != cudaSuccess) {
      delete gr;
      throw Error(JFFTB_ECUDA, "cudaMalloc failed for Green blocks");
    }
    const int layout = g->fused ? 1 : 0;
    launch_green_setup(geo, g->stream, resp.as<double>(), m[0] | (m[1] << 8) | (m[2] << 16),
                       gr->blocks, layout, nfreq, layout == 1 && fused_dif());
    JF_CUDA(cudaStreamSynchronize(g->stream));
    g->refs.fetch_add(1);
    *out = gr;
  });
}

int jfftb_green_destroy(jfftb_green* green) {
  return guarded([&] {
    if (!green) return;
    jfftb_grid* g = green->grid;
    {
      DeviceGuard dg(g->device);
      cudaStreamSynchronize(g->stream);
      drop_iteration_graph(g);  // it bakes in the Green planes
      cudaFree(green->blocks);
    }
    delete green;
    grid_release(g);
  });
}

int jfftb_green_export_blocks(jfftb_green* green, double* out) {
  return guarded([&] {
    require(green != nullptr && out != nullptr, "null argument");
    jfftb_grid* g = green->grid;
    DeviceGuard dg(g->device);
    const Geom& geo = g->geo;
    const int d = geo.d, np = green_planes(d);
    const int64_t nfreq = spec_elems(g);
    std::vector<double> packed((size_t)np * nfreq);
    JF_CUDA(cudaMemcpyAsync(packed.data(), green->blocks, sizeof(double) * np * nfreq,
                            cudaMemcpyDeviceToHost, g->stream));
    JF_CUDA(cudaStreamSynchronize(g->stream));
    for (int64_t f = 0; f < geo.Nh; ++f) {
      double* o = out + f * 2 * d * d;
      // numpy order (last axis halved); the fused layout halves axis 0, so the
      // other half is reached through G(-q) = conj G(q)
      int64_t src = f;
      double conj = 1.0;
      if (g->fused) {
        int q[3] = {0, 0, 0};
        int64_t rem = f;
        q[d - 1] = (int)(rem % geo.nh);
        rem /= geo.nh;
        for (int a = d - 2; a >= 0; --a) { q[a] = (int)(rem % geo.n[a]); rem /= geo.n[a]; }
        if (2 * q[0] > geo.n[0]) {
          for (int a = 0; a < d; ++a) q[a] = (geo.n[a] - q[a]) % geo.n[a];
          conj = -1.0;
        }
        if (fused_dif()) q[d - 1] = dif_pos(geo.n[d - 1], q[d - 1]);  // in-place pass C slots
        src = q[0];
        for (int a = 1; a < d; ++a) src = src * geo.n[a] + q[a];
      }
      for (int a = 0; a < d; ++a) {
        o[2 * (a * d + a)] = packed[a * nfreq + src];
        o[2 * (a * d + a) + 1] = 0.0;
      }
      int k = 0;
      for (int a = 0; a < d; ++a)
        for (int b = a + 1; b < d; ++b, ++k) {
          const double re = packed[(d + 2 * k) * nfreq + src];
          const double im = conj * packed[(d + 2 * k + 1) * nfreq + src];
          o[2 * (a * d + b)] = re;
          o[2 * (a * d + b) + 1] = im;
          o[2 * (b * d + a)] = re;
          o[2 * (b * d + a) + 1] = -im;
        }
    }
  });
}

int jfftb_apply_green(jfftb_green* green, const double* r, double* out, int where) {
  return jfftb_apply_precond(JFFTB_PC_GREEN, green, nullptr, r, out, where);
}

int jfftb_jacobi_create(jfftb_op* op, jfftb_jacobi** out) {
  return guarded([&] {
    require(op != nullptr && out != nullptr, "null argument");
    jfftb_grid* g = op->grid;
    const Geom& geo = g->geo;
    for (int a = 0; a < geo.d; ++a)
      require(geo.n[a] % 2 == 0, "diagonal probing requires an even node count");
    DeviceGuard dg(g->device);
    const int64_t n = geo.d * geo.N;
    DevBuf comb(sizeof(double) * n), resp(sizeof(double) * n);
    double* diag = nullptr;
    JF_CUDA(cudaMalloc(&diag, sizeof(double) * n));
    try {
      for (int alpha = 0; alpha < geo.d; ++alpha)
        for (int offs = 0; offs < (1 << geo.d); ++offs) {
          comb_kernel<<<nblk(n), 256, 0, g->stream>>>(comb.as<double>(), geo, alpha, offs);
          JF_LAUNCHED();
          launch_stencil(geo, g->stream, ST_K, comb.as<double>(), op->rho, op->lambda0, op->mu0,
                         nullptr, resp.as<double>(), nullptr);
          comb_extract_kernel<<<nblk(geo.N), 256, 0, g->stream>>>(diag, resp.as<double>(), geo,
                                                                  alpha, offs);
          JF_LAUNCHED();
        }
      int* bad = (int*)g->dscal;
      JF_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), g->stream));
      jacobi_finish_kernel<<<nblk(n), 256, 0, g->stream>>>(diag, n, bad);
      JF_LAUNCHED();
      if (read_flag(g, bad))
        throw Error(JFFTB_EINVAL, "probed diagonal has negative or non-finite entries");
    } catch (...) {
      cudaFree(diag);
      throw;
    }
    auto* j = new jfftb_jacobi();
    op->refs.fetch_add(1);
    j->op = op;
    j->grid = g;
    j->inv_sqrt = diag;
    *out = j;
  });
}

int jfftb_jacobi_from_array(jfftb_grid* g, const double* inv_sqrt, int where, jfftb_jacobi** out) {
  return guarded([&] {
    require(g != nullptr && inv_sqrt != nullptr && out != nullptr, "null argument");
    DeviceGuard dg(g->device);
    const int64_t n = g->geo.d * g->geo.N;
    DevBuf tin;
    const double* src = stage_in(g, inv_sqrt, n, where, tin);
    double* diag = nullptr;
    JF_CUDA(cudaMalloc(&diag, sizeof(double) * n));
    JF_CUDA(cudaMemcpyAsync(diag, src, sizeof(double) * n, cudaMemcpyDeviceToDevice, g->stream));
    JF_CUDA(cudaStreamSynchronize(g->stream));
    auto* j = new jfftb_jacobi();
    g->refs.fetch_add(1);
    j->op = nullptr;
    j->grid = g;
    j->inv_sqrt = diag;
    *out = j;
  });
}

int jfftb_jacobi_destroy(jfftb_jacobi* jac) {
  return guarded([&] {
    if (!jac) return;
    jfftb_op* op = jac->op;
    jfftb_grid* g = jac->grid;
    {
      DeviceGuard dg(g->device);
      cudaStreamSynchronize(g->stream);
      drop_iteration_graph(g);  // it bakes in D^-1/2
      cudaFree(jac->inv_sqrt);
    }
    delete jac;
    if (op) op_release(op);
    else grid_release(g);
  });
}

int jfftb_jacobi_export(jfftb_jacobi* jac, double* out, int where) {
  return guarded([&] {
    require(jac != nullptr, "null jacobi");
    jfftb_grid* g = jac->grid;
    DeviceGuard dg(g->device);
    const int64_t n = g->geo.d * g->geo.N;
    require(out != nullptr, "null output");
    if (where == JFFTB_HOST) {
      copy_d2h(g, out, jac->inv_sqrt, sizeof(double) * n, g->stream);
    } else {
      JF_CUDA(cudaMemcpyAsync(out, jac->inv_sqrt, sizeof(double) * n, cudaMemcpyDeviceToDevice,
                              g->stream));
      JF_CUDA(cudaStreamSynchronize(g->stream));
    }
  });
}

int jfftb_apply_precond(int kind, jfftb_green* green, jfftb_jacobi* jac, const double* r,
                        double* out, int where) {
  return guarded([&] {
    jfftb_grid* g = green ? green->grid : (jac ? jac->grid : nullptr);
    require(g != nullptr, "preconditioner needs a Green operator or a Jacobi diagonal");
    if (green && jac) require(green->grid == jac->grid, "grid mismatch");
    DeviceGuard dg(g->device);
    const int64_t n = g->geo.d * g->geo.N;
    DevBuf tin, tout;
    const double* dr = stage_in(g, r, n, where, tin);
    double* dout = stage_out(out, n, where, tout);
    precond_device(kind, green, jac, g, dr, dout);
    finish_out(g, out, dout, n, where);
  });
}

int jfftb_pcg(jfftb_op* op, int kind, jfftb_green* green_pc, jfftb_jacobi* jac,
              jfftb_green* green_term, const double* rhs, int where, double eta, int max_iter,
              double* x_out, double* history_out, int* iterations, int* terminated,
              double* wall_s) {
  const auto t0 = std::chrono::steady_clock::now();
  return guarded([&] {
    require(op != nullptr && green_term != nullptr, "pcg needs an operator and a Green operator");
    require(history_out && iterations && terminated, "null output argument");
    require(kind >= JFFTB_PC_NONE && kind <= JFFTB_PC_GREEN_JACOBI, "unknown preconditioner");
    require(max_iter >= 0, "max_iter must be >= 0");
    jfftb_grid* g = op->grid;
    require(green_term->grid == g, "Green operator lives on a different grid");
    if (kind == JFFTB_PC_GREEN || kind == JFFTB_PC_GREEN_JACOBI)
      require(green_pc != nullptr && green_pc->grid == g, "kind needs an assembled Green operator");
    if (kind == JFFTB_PC_JACOBI || kind == JFFTB_PC_GREEN_JACOBI)
      require(jac != nullptr && jac->grid == g, "kind needs an assembled Jacobi diagonal");
    if (!green_pc) green_pc = green_term;
    DeviceGuard dg(g->device);
    const Geom& geo = g->geo;
    cudaStream_t s = g->stream;
    if (!g->fused) ensure_plans(g);  // the fused passes need no cuFFT plans
    const int64_t n = geo.d * geo.N;
    require(rhs != nullptr, "null right-hand side");
    require(where == JFFTB_HOST || where == JFFTB_DEVICE, "where must be HOST or DEVICE");

    // workspace: one allocation cached on the grid and reused by every solve
    const int kcount = stencil_blocks(geo);
    PcgBuffers B = pcg_workspace(g, kcount, max_iter);
    PcgState* hs = g->ws_host;
    if (B.bcbq) JF_CUDA(cudaMemsetAsync(B.bcbq, 0, 2 * sizeof(unsigned), s));

    // fault in a pageable solution array on host threads while the device
    // iterates, so the final d2h is a plain staged memcpy
    HostPrefault prefault(where == JFFTB_HOST ? x_out : nullptr, sizeof(double) * n);

    PcgState h0{};
    h0.eta = eta;
    h0.max_iter = max_iter;
    *hs = h0;
    JF_CUDA(cudaMemcpyAsync(B.st, hs, sizeof(PcgState), cudaMemcpyHostToDevice, s));
    JF_CUDA(cudaMemsetAsync(B.x, 0, sizeof(double) * n, s));
    if (where == JFFTB_HOST)
      copy_h2d(g, B.rs, rhs, sizeof(double) * n, s);
    else
      JF_CUDA(cudaMemcpyAsync(B.rs, rhs, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
    auto poll = [&]() {
      JF_CUDA(cudaMemcpyAsync(hs, B.st, sizeof(PcgState), cudaMemcpyDeviceToHost, s));
      JF_CUDA(cudaStreamSynchronize(s));
      return hs->done != 0;
    };
    prof_collect(g, 0, true);  // drop leftovers of an aborted solve
    pcg_dispatch(kind, true, op, jac, green_pc, green_term, B);
    bool done = poll();
    // host loop: iterations are predicated on the device flag, so a few can
    // be queued ahead of each poll; the batch grows while the solve runs
    int batch = 1;
    // After the first (uncaptured) iteration, further iterations replay one
    // captured CUDA graph: one launch instead of ~10 and shorter gaps between
    // the kernels.  Not while the stage profiler records events.
    const bool graphs = g->fused && !g->prof && graphs_enabled();
    bool first = true;
    while (!done) {
      for (int k = 0; k < batch; ++k) {
        if (graphs && !first) {
          run_iteration_graph(g, kind, op, jac, green_pc, green_term, B);
        } else {
          pcg_dispatch(kind, false, op, jac, green_pc, green_term, B);
        }
        first = false;
      }
      done = poll();
      prof_collect(g, hs->iters, false);
      batch = std::min(batch * 2, 8);
    }
    prof_collect(g, hs->iters, true);
    const int it = hs->iters;
    *iterations = it;
    JF_CUDA(cudaMemcpyAsync(history_out, B.hist, sizeof(double) * (it + 1),
                            cudaMemcpyDeviceToHost, s));
    unsigned bcb_flag = 0;
    if (B.bcbq)
      JF_CUDA(cudaMemcpyAsync(&bcb_flag, B.bcbq + 1, sizeof(unsigned), cudaMemcpyDeviceToHost, s));
    JF_CUDA(cudaStreamSynchronize(s));
    if (bcb_flag)
      throw Error(JFFTB_ECUDA, "merged spectral pass: a work item's producers never arrived");
    if (hs->status != JFFTB_OK) {
      if (wall_s)
        *wall_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      throw Error(hs->status, hs->status == JFFTB_ECURVATURE
                                  ? "non-positive search-direction curvature in PCG"
                                  : "PCG recurrence became non-finite");
    }
    *terminated = (hs->gnorm2 <= eta) ? JFFTB_CONVERGED : JFFTB_ITERATION_CAP;
    launch_sub_mean(geo, s, B.x, ensure_partials(g, kRedBlocks * 3 + 3));
    prefault.wait();
    if (x_out) {
      if (where == JFFTB_HOST)
        copy_d2h(g, x_out, B.x, sizeof(double) * n, s);
      else
        JF_CUDA(cudaMemcpyAsync(x_out, B.x, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
    }
    JF_CUDA(cudaStreamSynchronize(s));
    if (wall_s)
      *wall_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  });
}

int jfftb_pcg_batch(jfftb_op* op, int kind, jfftb_green* green_pc, jfftb_jacobi* jac,
                    jfftb_green* green_term, int nrhs, const double* rhs, int where, double eta,
                    int max_iter, double* x_out, double* history_out, int* iterations,
                    int* terminated, double* wall_s) {
  const auto t0 = std::chrono::steady_clock::now();
  return guarded([&] {
    require(op != nullptr && green_term != nullptr, "pcg needs an operator and a Green operator");
    require(rhs && history_out && iterations && terminated, "null argument");
    require(nrhs >= 1 && nrhs <= 64, "1 to 64 right-hand sides");
    require(max_iter >= 0, "max_iter must be >= 0");
    require(where == JFFTB_HOST || where == JFFTB_DEVICE, "where must be HOST or DEVICE");
    jfftb_grid* g = op->grid;
    require(g->fused && g->geo.d == 3 &&
                (kind == JFFTB_PC_GREEN || kind == JFFTB_PC_GREEN_JACOBI),
            "batched solves run the fused 3-D spectral kinds (use jfftb_pcg otherwise)");
    require(green_term->grid == g && green_pc != nullptr && green_pc->grid == g,
            "Green operators live on a different grid");
    if (kind == JFFTB_PC_GREEN_JACOBI)
      require(jac != nullptr && jac->grid == g, "kind needs an assembled Jacobi diagonal");
    DeviceGuard dg(g->device);
    const Geom& geo = g->geo;
    cudaStream_t s = g->stream;
    const int64_t n = geo.d * geo.N;
    Batch bt;
    PcgBuffers B = pcg_workspace_batch(g, stencil_blocks(geo), max_iter, nrhs, bt);
    PcgState* hs = g->wsb_host;
    for (int l = 0; l < nrhs; ++l) {
      PcgState h0{};
      h0.eta = eta;
      h0.max_iter = max_iter;
      hs[l] = h0;
    }
    JF_CUDA(cudaMemcpyAsync(B.st, hs, sizeof(PcgState) * nrhs, cudaMemcpyHostToDevice, s));
    JF_CUDA(cudaMemsetAsync(B.x, 0, sizeof(double) * n * nrhs, s));
    if (where == JFFTB_HOST)
      copy_h2d(g, B.rs, rhs, sizeof(double) * n * nrhs, s);
    else
      JF_CUDA(cudaMemcpyAsync(B.rs, rhs, sizeof(double) * n * nrhs, cudaMemcpyDeviceToDevice, s));
    auto poll = [&]() {
      JF_CUDA(cudaMemcpyAsync(hs, B.st, sizeof(PcgState) * nrhs, cudaMemcpyDeviceToHost, s));
      JF_CUDA(cudaStreamSynchronize(s));
      for (int l = 0; l < nrhs; ++l)
        if (!hs[l].done) return false;
      return true;
    };
    pcg_dispatch_batch(kind, true, op, jac, green_pc, green_term, B, bt);
    bool done = poll();
    int batch = 1;
    while (!done) {
      for (int k = 0; k < batch; ++k)
        pcg_dispatch_batch(kind, false, op, jac, green_pc, green_term, B, bt);
      done = poll();
      batch = std::min(batch * 2, 8);
    }
    int status = JFFTB_OK;
    for (int l = 0; l < nrhs; ++l) {
      iterations[l] = hs[l].iters;
      terminated[l] = hs[l].gnorm2 <= eta ? JFFTB_CONVERGED : JFFTB_ITERATION_CAP;
      JF_CUDA(cudaMemcpyAsync(history_out + (size_t)l * (max_iter + 1), B.hist + (size_t)l * B.hstride,
                              sizeof(double) * (hs[l].iters + 1), cudaMemcpyDeviceToHost, s));
      if (hs[l].status != JFFTB_OK && status == JFFTB_OK) status = hs[l].status;
    }
    JF_CUDA(cudaStreamSynchronize(s));
    if (status != JFFTB_OK)
      throw Error(status, status == JFFTB_ECURVATURE
                              ? "non-positive search-direction curvature in PCG"
                              : "PCG recurrence became non-finite");
    double* part = ensure_partials(g, kRedBlocks * 3 + 3);
    for (int l = 0; l < nrhs; ++l) launch_sub_mean(geo, s, B.x + (size_t)l * n, part);
    if (x_out) {
      if (where == JFFTB_HOST)
        copy_d2h(g, x_out, B.x, sizeof(double) * n * nrhs, s);
      else
        JF_CUDA(cudaMemcpyAsync(x_out, B.x, sizeof(double) * n * nrhs, cudaMemcpyDeviceToDevice, s));
    }
    JF_CUDA(cudaStreamSynchronize(s));
    if (wall_s)
      *wall_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  });
}

int jfftb_debug_fused_apply(jfftb_green* green, jfftb_jacobi* jac, int upto, const double* r,
                            double* out) {
  return guarded([&] {
    require(green != nullptr && r != nullptr && out != nullptr, "null argument");
    jfftb_grid* g = green->grid;
    require(g->fused, "grid has no fused spectral path");
    DeviceGuard dg(g->device);
    const Geom& geo = g->geo;
    const int64_t n = geo.d * geo.N, ns = spec_elems(g);
    DevBuf din(sizeof(double) * n), dout(sizeof(double) * n),
        spec(sizeof(double2) * geo.d * ns);
    JF_CUDA(cudaMemcpyAsync(din.ptr, r, sizeof(double) * n, cudaMemcpyHostToDevice, g->stream));
    fused_debug_apply(geo, g->stream, green, jac ? jac->inv_sqrt : nullptr,
                      din.as<double>(), dout.as<double>(), spec.as<double2>(), g->twiddle, upto);
    if (upto >= 5)
      JF_CUDA(cudaMemcpyAsync(out, dout.ptr, sizeof(double) * n, cudaMemcpyDeviceToHost,
                              g->stream));
    else
      JF_CUDA(cudaMemcpyAsync(out, spec.ptr, sizeof(double2) * geo.d * ns,
                              cudaMemcpyDeviceToHost, g->stream));
    JF_CUDA(cudaStreamSynchronize(g->stream));
  });
}

int jfftb_profile_start(jfftb_grid* g) {
  return guarded([&] {
    require(g != nullptr, "null grid");
    g->prof = true;
    for (int k = 0; k < JFFTB_N_STAGES; ++k) g->prof_ms[k] = 0.0;
    g->prof_iters = 0;
  });
}

int jfftb_profile_read(jfftb_grid* g, double* stage_ms, int64_t* iterations, int stop) {
  return guarded([&] {
    require(g != nullptr && stage_ms != nullptr && iterations != nullptr, "null argument");
    for (int k = 0; k < JFFTB_N_STAGES; ++k) stage_ms[k] = g->prof_ms[k];
    *iterations = g->prof_iters;
    if (stop) g->prof = false;
  });
}

/* ---- input generators (generators.cu; microstructures.py:73-115) ------ */
}  // extern "C"
namespace {
// run `body` on a device copy of a host scalar field (or in place on a
// device field) and copy the result back
template <class F>
void scalar_inout(jfftb_grid* g, double* field, int where, F&& body) {
  require(field != nullptr, "null field");
  const int64_t n = g->geo.N;
  if (where == JFFTB_DEVICE) {
    body(field);
    return;
  }
  require(where == JFFTB_HOST, "where must be JFFTB_HOST or JFFTB_DEVICE");
  DevBuf tmp(sizeof(double) * n);
  copy_h2d(g, tmp.ptr, field, sizeof(double) * n, g->stream);
  body(tmp.as<double>());
  copy_d2h(g, field, tmp.ptr, sizeof(double) * n, g->stream);
}
double* minmax_of(jfftb_grid* g, const double* field) {
  double* part = ensure_partials(g, gen_partials(g->geo) + 2);
  double* mm = part + gen_partials(g->geo);
  launch_minmax(g->geo, g->stream, field, part, mm);
  return mm;
}
}  // namespace
extern "C" {

int jfftb_binomial_filter(jfftb_grid* g, double* field, int passes, int where) {
  return guarded([&] {
    require(g != nullptr, "null grid");
    require(passes >= 0, "filter passes must be >= 0");
    DeviceGuard dg(g->device);
    scalar_inout(g, field, where, [&](double* f) {
      if (passes == 0) return;
      DevBuf scratch(sizeof(double) * g->geo.N);
      launch_binomial_filter(g->geo, g->stream, f, scratch.as<double>(), passes);
      JF_CUDA(cudaStreamSynchronize(g->stream));
    });
  });
}

int jfftb_field_minmax(jfftb_grid* g, const double* field, double* minmax2, int where) {
  return guarded([&] {
    require(g != nullptr && minmax2 != nullptr, "null argument");
    DeviceGuard dg(g->device);
    DevBuf tin;
    const double* f = stage_in(g, field, g->geo.N, where, tin);
    double* mm = minmax_of(g, f);
    JF_CUDA(cudaMemcpyAsync(minmax2, mm, 2 * sizeof(double), cudaMemcpyDeviceToHost, g->stream));
    JF_CUDA(cudaStreamSynchronize(g->stream));
  });
}

int jfftb_rescale_contrast(jfftb_grid* g, double* field, double chi, int where) {
  return guarded([&] {
    require(g != nullptr, "null grid");
    require(chi >= 1.0, "total phase contrast must be >= 1");
    DeviceGuard dg(g->device);
    const double soft = std::isinf(chi) ? 0.0 : 1.0 / chi;
    scalar_inout(g, field, where, [&](double* f) {
      double* mm = minmax_of(g, f);
      double h[2];
      JF_CUDA(cudaMemcpyAsync(h, mm, sizeof(h), cudaMemcpyDeviceToHost, g->stream));
      JF_CUDA(cudaStreamSynchronize(g->stream));
      require(h[1] > h[0], "cannot rescale a constant field to a target contrast");
      launch_rescale(g->geo, g->stream, f, mm, soft);
    });
  });
}

int jfftb_threshold(jfftb_grid* g, double* field, double chi, int where) {
  return guarded([&] {
    require(g != nullptr, "null grid");
    require(chi >= 1.0, "total phase contrast must be >= 1");
    DeviceGuard dg(g->device);
    const double soft = std::isinf(chi) ? 0.0 : 1.0 / chi;
    scalar_inout(g, field, where, [&](double* f) { launch_threshold(g->geo, g->stream, f, soft); });
  });
}

int jfftb_simp_projection(jfftb_grid* g, double* field, double beta, double emin, int where) {
  return guarded([&] {
    require(g != nullptr, "null grid");
    require(std::isfinite(beta) && beta > 0.0, "projection sharpness must be finite and > 0");
    require(std::isfinite(emin) && emin >= 0.0, "void stiffness must be finite and >= 0");
    DeviceGuard dg(g->device);
    scalar_inout(g, field, where, [&](double* f) {
      double* part = ensure_partials(g, gen_partials(g->geo) + 2);
      launch_simp(g->geo, g->stream, f, part, part + gen_partials(g->geo), beta, emin);
      JF_CUDA(cudaStreamSynchronize(g->stream));
    });
  });
}

int jfftb_field_layout(jfftb_grid* g, const double* src, double* dst, int planes, int to_c,
                       int where) {
  return guarded([&] {
    require(g != nullptr, "null grid");
    require(planes >= 1, "planes must be >= 1");
    DeviceGuard dg(g->device);
    const size_t n = (size_t)planes * g->geo.N;
    DevBuf tin, tout;
    const double* ds = stage_in(g, src, n, where, tin);
    double* dd = stage_out(dst, n, where, tout);
    require(ds != dd, "field layout conversion cannot run in place");
    launch_fortran_to_c(g->geo, g->stream, ds, dd, planes, to_c != 0);
    finish_out(g, dst, dd, n, where);
    if (where == JFFTB_DEVICE) JF_CUDA(cudaStreamSynchronize(g->stream));
  });
}

int jfftb_load_pairings(jfftb_op* op, int nload, const double* u, const double* ebar,
                        const double* weights, double* sigma_out, double* field_out,
                        int where) {
  return guarded([&] {
    require(op != nullptr && ebar != nullptr && sigma_out != nullptr, "null argument");
    require(nload >= 1 && nload <= 6, "1 to 6 load cases");
    jfftb_grid* g = op->grid;
    const Geom& geo = g->geo;
    const int M = geo.d == 2 ? 3 : 6;
    for (int l = 0; l < nload; ++l) check_ebar(geo.d, ebar + l * M);
    DeviceGuard dg(g->device);
    DevBuf tin, tout, dw;
    const double* du = stage_in(g, u, (size_t)nload * geo.d * geo.N, where, tin);
    double* dfield = field_out ? stage_out(field_out, geo.N, where, tout) : nullptr;
    if (field_out) {
      require(weights != nullptr, "the pairing field needs load-pair weights");
      dw.reset(sizeof(double) * nload * nload);
      JF_CUDA(cudaMemcpyAsync(dw.ptr, weights, sizeof(double) * nload * nload,
                              cudaMemcpyHostToDevice, g->stream));
    }
    const int K = nload * (nload + 1) / 2;
    double* part = ensure_partials(g, kRedBlocks * K + K);
    launch_load_pairings(geo, g->stream, nload, du, op->rho, op->lambda0, op->mu0, ebar,
                         dw.as<double>(), dfield, part);
    launch_sum_partials(g->stream, part, kRedBlocks, K, part + kRedBlocks * K);
    std::vector<double> sums(K);
    JF_CUDA(cudaMemcpyAsync(sums.data(), part + kRedBlocks * K, sizeof(double) * K,
                            cudaMemcpyDeviceToHost, g->stream));
    JF_CUDA(cudaStreamSynchronize(g->stream));
    double vol = 1.0;
    for (int a = 0; a < geo.d; ++a) vol *= geo.h[a] * geo.n[a];
    const double scale = geo.w / vol;
    for (int a = 0, k = 0; a < nload; ++a)
      for (int b = a; b < nload; ++b, ++k)
        sigma_out[a * nload + b] = sigma_out[b * nload + a] = scale * sums[k];
    if (field_out) finish_out(g, field_out, dfield, geo.N, where);
  });
}

}  // extern "C"
