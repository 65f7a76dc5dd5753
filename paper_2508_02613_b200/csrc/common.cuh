// Shared internals of libjfftb200.so: handle structs, error plumbing and the
// per-voxel finite-element force routine used by every stencil kernel.
#pragma once

#include <cuda_runtime.h>
#include <cufft.h>
#include <stdint.h>

#include <stdexcept>
#include <string>
#include <atomic>
#include <thread>
#include <vector>

#include "../../include/jfftb200.h"

namespace jfftb {

// ---------------------------------------------------------------------------
// errors: C++ exceptions inside, int status codes at the C boundary
// ---------------------------------------------------------------------------
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void set_last_error(const std::string& msg);
void count_launch(int n = 1);

#define JF_CUDA(call)                                                          \
  do {                                                                         \
    cudaError_t e_ = (call);                                                   \
    if (e_ != cudaSuccess)                                                     \
      throw ::jfftb::Error(JFFTB_ECUDA, std::string(#call) + ": " +            \
                                            cudaGetErrorString(e_));           \
  } while (0)

#define JF_CUFFT(call)                                                         \
  do {                                                                         \
    cufftResult r_ = (call);                                                   \
    if (r_ != CUFFT_SUCCESS)                                                   \
      throw ::jfftb::Error(JFFTB_ECUDA, std::string(#call) + ": cufft error " + \
                                            std::to_string((int)r_));          \
  } while (0)

#define JF_LAUNCHED()                                                          \
  do {                                                                         \
    ::jfftb::count_launch();                                                   \
    JF_CUDA(cudaGetLastError());                                               \
  } while (0)

inline void require(bool ok, const std::string& msg) {
  if (!ok) throw Error(JFFTB_EINVAL, msg);
}

inline int current_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev & 63;
}

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) is per device context:
// `done` (one static per kernel instance) keeps one bit per device id
template <class K>
void set_smem_once(K kernel, size_t bytes, std::atomic<uint64_t>& done) {
  const uint64_t bit = 1ull << current_device();
  if (done.load() & bit) return;
  if (bytes > 48 * 1024)
    JF_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  done.fetch_or(bit);
}

// ---------------------------------------------------------------------------
// geometry passed by value to kernels
// ---------------------------------------------------------------------------
struct Geom {
  int d;
  int n[3];        // nodes per axis (axis 0 slowest)
  int64_t N;       // nodes
  int nh;          // n[d-1]/2 + 1
  int64_t Nh;      // half-spectrum entries per component
  double h[3];     // pixel size per axis
  double hinv[3];
  double w;        // quadrature weight prod(h)/d!
  bool iso;        // all h equal
};

// persistent device scalars of one PCG solve
struct PcgState {
  double rz, curv, alpha, beta, gnorm2, rz_new, eta;
  int done;     // 1 once converged / capped / aborted
  int iters;    // search-direction updates so far
  int status;   // JFFTB_OK / JFFTB_ENONFINITE / JFFTB_ECURVATURE
  int max_iter;
  int xupd;     // fused path: this iteration's alpha is valid (x += alpha p pending)
};

}  // namespace jfftb

struct jfftb_grid {
  jfftb::Geom geo;
  int device;
  cudaStream_t own_stream;
  cudaStream_t stream;
  // cuFFT plans: vector field (batch d) and doubled vector field (batch 2d)
  cufftHandle plan_fwd_d = 0, plan_inv_d = 0, plan_fwd_2d = 0;
  bool plans_ready = false;
  void* fft_work = nullptr;
  void* host_stage = nullptr;   // pinned staging ring for pageable host copies (hostio.cu)
  // one PCG iteration captured as a CUDA graph (api.cu jfftb_pcg), valid for
  // the key it was captured with
  static constexpr int kIterKey = 11;
  cudaGraphExec_t iter_graph = nullptr;
  const void* iter_key[kIterKey] = {};
  // constants baked into the kernels' arguments: op Lame, Green (pc, term) Lame
  double iter_lame[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  int iter_kind = -1;
  int iter_launches = 0;
  size_t fft_work_bytes = 0;
  // reduction scratch
  double* partials = nullptr;   // per-block partial sums
  int partials_cap = 0;
  double* dscal = nullptr;      // small device scalar scratch
  // fused spectral path (fused.cu): power-of-two grids, 16 <= n <= 2048
  bool fused = false;
  double2* twiddle = nullptr;   // exp(-2 pi i j / 4096)
  // cached PCG workspace (api.cu pcg_workspace) and the batched one
  void* ws = nullptr;
  size_t ws_bytes = 0;
  void* wsb = nullptr;
  size_t wsb_bytes = 0;
  jfftb::PcgState* wsb_host = nullptr;
  int wsb_L = 0;
  jfftb::PcgState* ws_host = nullptr;  // pinned mirror of the device state
  // stage profile (jfftb_profile_*)
  bool prof = false;
  std::vector<cudaEvent_t> ev_free;
  std::vector<cudaEvent_t> ev_cur;                  // events of the iteration being issued
  std::vector<std::vector<cudaEvent_t>> ev_pending;  // issued iterations, oldest first
  int64_t prof_seq = 0;       // iterations issued in the current solve
  int64_t prof_done_seq = 0;  // iterations of the current solve already collected
  double prof_ms[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  int64_t prof_iters = 0;
  // lifetime: operators and Green operators hold a reference; destroying the
  // grid first defers the release until the last of them is gone
  std::atomic<int> refs{0};
  std::atomic<bool> closed{false};
};

struct jfftb_op {
  jfftb_grid* grid;
  std::atomic<int> refs{0};  // Jacobi diagonals built from this operator
  std::atomic<bool> closed{false};
  double* rho;      // device, N
  double lambda0, mu0;
};

struct jfftb_green {
  jfftb_grid* grid;
  double lambda_ref, mu_ref;
  // Hermitian-packed blocks, planar: 2-D 4 planes (G00, G11, Re G01, Im G01);
  // 3-D 9 planes (G00, G11, G22, Re/Im G01, Re/Im G02, Re/Im G12), each nfreq
  double* blocks;
  int64_t nfreq = 0;  // frequencies per plane
};

struct jfftb_jacobi {
  jfftb_op* op;        // the operator it was probed from (null: given as an array)
  jfftb_grid* grid;
  double* inv_sqrt;  // device, d * N
};

namespace jfftb {

// ---------------------------------------------------------------------------
// P1 simplex tables (d-generic, see oracle/jfft_oracle.py edge_offsets)
// Simplex t = permutation t (lexicographic) of the axes; its path edge along
// axis a starts at voxel corner o(t,a) (bitmask: bit j = offset along axis j).
// ---------------------------------------------------------------------------
__host__ __device__ constexpr int perm_axis(int D, int t, int k) {
  // k-th axis visited by permutation t
  return D == 2 ? (t == 0 ? k : 1 - k)
                : (t == 0 ? k
                   : t == 1 ? (k == 0 ? 0 : k == 1 ? 2 : 1)
                   : t == 2 ? (k == 0 ? 1 : k == 1 ? 0 : 2)
                   : t == 3 ? (k == 0 ? 1 : k == 1 ? 2 : 0)
                   : t == 4 ? (k == 0 ? 2 : k == 1 ? 0 : 1)
                            : (k == 0 ? 2 : k == 1 ? 1 : 0));
}
__host__ __device__ constexpr int perm_pos(int D, int t, int ax) {
  return perm_axis(D, t, 0) == ax ? 0 : perm_axis(D, t, 1) == ax ? 1 : 2;
}
__host__ __device__ constexpr int edge_base(int D, int t, int a) {
  int m = 0;
  for (int j = 0; j < D; ++j) {
    if (j == a) continue;
    bool prec = perm_pos(D, t, j) < perm_pos(D, t, a);
    bool bit = (j == 0) ? !prec : prec;
    if (bit) m |= 1 << j;
  }
  return m;
}
__host__ __device__ constexpr int n_simplex(int D) { return D == 2 ? 2 : 6; }
__host__ __device__ constexpr int mandel_m(int D) { return D == 2 ? 3 : 6; }
// Mandel component of the symmetric pair (i, j)
__host__ __device__ constexpr int mandel_of(int D, int i, int j) {
  return i == j ? i
                : (D == 2 ? 2 : (i + j == 3 ? 3 : (i + j == 2 ? 4 : 5)));
}
__host__ __device__ constexpr int mandel_i(int D, int m) {
  return m < D ? m : (D == 2 ? 0 : (m == 3 ? 1 : 0));
}
__host__ __device__ constexpr int mandel_j(int D, int m) {
  return m < D ? m : (D == 2 ? 1 : (m == 3 ? 2 : (m == 4 ? 2 : 1)));
}

constexpr double kSqrt2 = 1.4142135623730951;
constexpr double kInvSqrt2 = 0.70710678118654752;

enum VoxMode { VOX_K = 0, VOX_RHS = 1, VOX_RES = 2 };

// Nodal forces of one voxel.  uc[c][i]: displacement component i at corner c
// (bit j of c = +1 along axis j).  G_t[i][a] = (diff along the path edge)*gs[a]
// (+ Ebar for VOX_RES; = Ebar for VOX_RHS).  Stress per simplex
// sigma = lam tr(G) I + mu (G + G^T) with lam/mu already scaled by rho*w (and,
// in ISO K mode, by 1/h^2 with gs = fs = 1).  Edge forces sigma[:,a]*fs[a] go
// + to the edge's high corner and - to its low corner; f[c][i] is the sum.
template <int D, int MODE, bool SCALE>
__device__ __forceinline__ void voxel_forces(const double (&uc)[1 << D][D],
                                             double lam, double mu,
                                             const double* gs, const double* fs,
                                             const double (*Ebar)[3],
                                             double (&f)[1 << D][D]) {
  constexpr int C = 1 << D;
  constexpr int T = n_simplex(D);
  double acc[D][C][D];
  bool init[D][C];
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int c = 0; c < C; ++c) init[a][c] = false;

#pragma unroll
  for (int t = 0; t < T; ++t) {
    double G[D][D];  // G[i][a] = d u_i / d x_a
#pragma unroll
    for (int a = 0; a < D; ++a) {
      const int o = edge_base(D, t, a);
#pragma unroll
      for (int i = 0; i < D; ++i) {
        double g = 0.0;
        if (MODE != VOX_RHS) {
          g = uc[o | (1 << a)][i] - uc[o][i];
          if (SCALE) g *= gs[a];
        }
        if (MODE == VOX_RHS) g = Ebar[i][a];
        if (MODE == VOX_RES) g += Ebar[i][a];
        G[i][a] = g;
      }
    }
    double tr = G[0][0];
#pragma unroll
    for (int a = 1; a < D; ++a) tr += G[a][a];
    const double lt = lam * tr;
    const double mu2 = 2.0 * mu;
    double S[D][D];
#pragma unroll
    for (int a = 0; a < D; ++a) {
      S[a][a] = fma(mu2, G[a][a], lt);
#pragma unroll
      for (int b = a + 1; b < D; ++b) {
        S[a][b] = mu * (G[a][b] + G[b][a]);
        S[b][a] = S[a][b];
      }
    }
#pragma unroll
    for (int a = 0; a < D; ++a) {
      const int o = edge_base(D, t, a);
#pragma unroll
      for (int i = 0; i < D; ++i) {
        if (init[a][o]) acc[a][o][i] += S[i][a];
        else acc[a][o][i] = S[i][a];
      }
      init[a][o] = true;
    }
  }
#pragma unroll
  for (int c = 0; c < C; ++c) {
#pragma unroll
    for (int i = 0; i < D; ++i) {
      double s = 0.0;
      bool first = true;
#pragma unroll
      for (int a = 0; a < D; ++a) {
        const bool high = (c >> a) & 1;
        const int o = high ? (c ^ (1 << a)) : c;
        if (!init[a][o]) continue;
        double e = acc[a][o][i];
        if (SCALE) e *= fs[a];
        if (first) { s = high ? e : -e; first = false; }
        else s = high ? s + e : s - e;
      }
      f[c][i] = s;
    }
  }
}

// ---------------------------------------------------------------------------
// launch helpers (defined in the .cu files)
// ---------------------------------------------------------------------------
enum StencilMode { ST_K = 0, ST_RHS = 1, ST_RES = 2 };

// out = K u (ST_K), -B^T W rho C E (ST_RHS), -B^T W sigma(E + B u) (ST_RES).
// rho == nullptr means rho = 1.  curv_partials (ST_K only, may be null):
// per-block <u, out> partials; returns number of blocks written.
// ext = 1 (3-D): u and rho are halo-extended slabs with n[1] + 2 rows along
// axis 1 (row i of out reads input rows i .. i + 2); no wrap along axis 1
int launch_stencil(const Geom& g, cudaStream_t s, int mode, const double* u,
                   const double* rho, double lam, double mu, const double* ebar_mandel,
                   double* out, double* curv_partials, int ext = 0);
int stencil_blocks(const Geom& g);
// 3-D tile rows of the stencil launch and output rows per tile row
int stencil_tile_rows(const Geom& g);
int stencil_tile_height(const Geom& g);
struct PcgState;
// K p on tile rows [ty0, ty1) (3-D), predicated on st->done; partial b keeps
// its full-launch index
void launch_stencil_rows(const Geom& g, cudaStream_t s, const double* u, const double* rho,
                         double lam, double mu, double* out, double* curv_partials,
                         const PcgState* st, int ty0, int ty1);
// K u for nb right-hand sides bstride doubles apart (one launch; returns the
// partials per right-hand side, rhs b's at curv_partials + b * that)
int launch_stencil_batch(const Geom& g, cudaStream_t s, const double* u, const double* rho,
                         double lam, double mu, double* out, double* curv_partials, int nb,
                         int64_t bstride);

void launch_total_strain(const Geom& g, cudaStream_t s, const double* u,
                         const double* ebar, double* out);
// per-block partials of sum_Q rho C0 (E + B u), M values per block
int launch_stress_sum(const Geom& g, cudaStream_t s, const double* u, const double* rho,
                      double lam, double mu, const double* ebar, double* partials);

// pass C transforms the last axis in place (DIF forward / DIT inverse), so
// the fused-layout Green planes are stored with the last axis in the
// transform's digit-reversed slot order (fft.cuh dif_pos); JFFTB_PASSC_DIF=0
// selects the Stockham pass C and natural order (read once per process)
bool fused_dif();

// host <-> device field copies (hostio.cu): pageable host memory is staged
// through a pinned ring by a team of host threads; d2h returns synchronised
void copy_h2d(jfftb_grid* g, void* dst, const void* src, size_t bytes, cudaStream_t s);
void copy_d2h(jfftb_grid* g, void* dst, const void* src, size_t bytes, cudaStream_t s);
void free_host_staging(jfftb_grid* g);

// Page-faults a pageable host output array on a few host threads while the
// device works (a fresh numpy array has no pages yet: the faults, not the
// memcpy, dominate its staged d2h).  Contents are preserved (each page is
// rewritten with its own first byte).  No-op for pinned or small arrays.
// wait() joins the team; the destructor waits too.
class HostPrefault {
 public:
  HostPrefault(void* p, size_t bytes);
  ~HostPrefault() { wait(); }
  void wait();
  HostPrefault(const HostPrefault&) = delete;
  HostPrefault& operator=(const HostPrefault&) = delete;

 private:
  std::vector<std::thread> team_;
};

// input generators (generators.cu)
void launch_binomial_filter(const Geom& g, cudaStream_t s, double* field, double* scratch,
                            int passes);
void launch_minmax(const Geom& g, cudaStream_t s, const double* field, double* partial,
                   double* out2);
void launch_rescale(const Geom& g, cudaStream_t s, double* field, const double* mm, double soft);
void launch_threshold(const Geom& g, cudaStream_t s, double* field, double soft);
void launch_simp(const Geom& g, cudaStream_t s, double* field, double* partial, double* mm,
                 double beta, double emin);
int gen_partials(const Geom& g);
void launch_fortran_to_c(const Geom& g, cudaStream_t s, const double* src, double* dst,
                         int planes, bool to_c);

// energy pairings of load-case solutions (loadcases.cu); returns K
int launch_load_pairings(const Geom& g, cudaStream_t s, int L, const double* u,
                         const double* rho, double lam, double mu, const double* ebar,
                         const double* wgt, double* field, double* partials);

// vector algebra
constexpr int kRedBlocks = 592;   // 4 x 148 SMs: fixed => deterministic
constexpr int kRedThreads = 256;
void launch_fill(cudaStream_t s, double* x, double v, int64_t n);
void launch_copy(cudaStream_t s, double* dst, const double* src, int64_t n);
void launch_mul(cudaStream_t s, double* out, const double* a, const double* b, int64_t n);
void launch_mul2(cudaStream_t s, double* out, const double* a, const double* b, int64_t n);
void launch_dot(cudaStream_t s, const double* a, const double* b, int64_t n, double* partials);
// sum `count` partials (stride `stride`, `m` interleaved values) -> out[m]
void launch_sum_partials(cudaStream_t s, const double* partials, int count, int m,
                         double* out);
// scratch: kRedBlocks * d + d doubles
void launch_sub_mean(const Geom& g, cudaStream_t s, double* x, double* scratch);

// spectral kernels
int green_planes(int d);
void launch_green_apply(const Geom& g, cudaStream_t s, const double* blocks,
                        const double2* in, double2* out, int ncomp_batches);
// resp: d x d x prod(m) impulse responses on the small grid m (packed m0|m1<<8|m2<<16)
// layout 0: numpy rfftn order (last axis halved), nfreq = Nh; layout 1:
// fused.cu order (axis 0 halved), nfreq = fused_spec_elems
// k0_off (layout 1): first axis-0 frequency of a k0-slab (distributed solves)
void launch_green_setup(const Geom& g, cudaStream_t s, const double* resp, int m,
                        double* blocks, int layout, int64_t nfreq, bool dif_last = false,
                        int k0_off = 0);

// PCG (pcg.cu)
struct PcgBuffers {
  double *x, *rs, *p, *kp;  // rs = [r ; s or z'] (2 d N)
  double2* spec;            // 2 d Nh
  PcgState* st;
  double* hist;
  double *kpart, *spart, *upart;
  int kcount;
  int hstride = 0;          // batched: history entries per right-hand side
  unsigned* bcbq = nullptr; // merged pass B/C/B' work queue (fused.cu passBCB)
};
// batched right-hand sides: L solves, vector fields vs doubles apart,
// spectra bss complex elements apart (L = 1: the plain solve)
struct Batch {
  int L = 1;
  int64_t vs = 0, bss = 0;
};
void pcg_dispatch(int kind, bool init, jfftb_op* op, jfftb_jacobi* jac, jfftb_green* gpc,
                  jfftb_green* gterm, const PcgBuffers& B);
void pcg_dispatch_batch(int kind, bool init, jfftb_op* op, jfftb_jacobi* jac, jfftb_green* gpc,
                        jfftb_green* gterm, const PcgBuffers& B, const Batch& bt);

// fused spectral path (fused.cu)
bool fused_supported(const Geom& g);
int64_t fused_spec_elems(const Geom& g);   // complex elements per spectral component
constexpr int kFusedMaxBlocks = 148 * 4 * 8;  // bound on pass-C partial pairs
// twiddle table: 4096 entries of exp(-2 pi i j / 4096), then per-stage tables
// (fft.cuh kTwN, tw_stage_off): 13 spans x 3 radices x 4096
constexpr int kTwiddleN = 4096 + 13 * 3 * 4096;
// complex elements per spectral component of whichever layout the grid uses
inline int64_t spec_elems(const jfftb_grid* g) {
  return g->fused ? fused_spec_elems(g->geo) : g->geo.Nh;
}
void launch_twiddles(cudaStream_t s, double2* tw);
void fused_precond_apply(const Geom& geo, cudaStream_t s, const jfftb_green* green,
                         const double* dinv, const double* r, double* out, double2* spec,
                         const double2* tw);
enum { FUSED_APPLY = 0, FUSED_INIT = 1, FUSED_ITER = 2 };
struct Batch;
void fused_stage_A(const Geom& geo, cudaStream_t s, int F, int mode, const PcgState* st,
                   double* r, const double* kp, const double* dinv, double2* spec,
                   const double2* tw, const Batch& bt);
void fused_stage_B(const Geom& geo, cudaStream_t s, bool inv, const PcgState* st,
                   double2* spec, int ncomp, const double2* tw, const Batch& bt);
int fused_stage_C(const Geom& geo, cudaStream_t s, int F, bool quad_only, const PcgState* st,
                  const jfftb_green* gpc, const jfftb_green* gterm, double2* spec,
                  double* partials, const double2* tw, const Batch& bt);
void fused_stage_I(const Geom& geo, cudaStream_t s, int mode, const PcgState* st,
                   const double2* zspec, const double* dinv, double* p, double* x,
                   const double2* tw, const Batch& bt);
// passes B, C, B' as one persistent kernel (3-D, n1 == n2, one solve)
bool fused_bcb_supported(const Geom& geo);
int64_t fused_bcb_partials(const Geom& geo);  // partial pairs it writes
int fused_stage_BCB(const Geom& geo, cudaStream_t s, int F, const PcgState* st,
                    const jfftb_green* gpc_h, const jfftb_green* gterm_h, double2* spec,
                    double* partials, const double2* tw, unsigned* q);

int64_t fused_component_stride(const Geom& geo);
// distributed solves (dist.cu): one rank's k0-slab of the spectral passes
struct SpecSlab {
  int k0lo, kcnt;  // axis-0 frequency rows [k0lo, k0lo + kcnt)
  int L1;          // axis-1 rows per source rank (segments of n1 / L1 ranks)
  int nf;          // fields held (2d green-jacobi, d green)
};
void fused_stage_B_slab(const Geom& geo, const SpecSlab& sl, cudaStream_t s, bool inv,
                        const PcgState* st, double2* recv, int comp0, int ncomp,
                        const double2* tw);
int fused_stage_C_slab(const Geom& geo, const SpecSlab& sl, cudaStream_t s, int F,
                       const PcgState* st, const double* green, double2* recv, double* partials,
                       const double2* tw);
// comp >= 0: that component only
void fused_stage_I_ext(const Geom& geo, cudaStream_t s, int mode, const PcgState* st,
                       const double2* zspec, const double* dinv, double* p_ext, double* x,
                       const double2* tw, int comp = -1);
void fused_stage_A_comp(const Geom& geo, cudaStream_t s, int F, int mode, const PcgState* st,
                        double* r, const double* kp, const double* dinv, double2* spec,
                        const double2* tw, int comp);
// PCG scalar kernels (pcg.cu) over `count` partials: alpha = rz / curvature,
// and the termination test / beta (solver.py:115-135)
// (partial j of block b at partials[b * stride + j])
void launch_alpha(cudaStream_t s, PcgState* st, const double* partials, int count, int stride);
void launch_finalize(int kind, bool init, cudaStream_t s, PcgState* st, const double* spart,
                     int scount, int sstride, double* hist);
void fused_debug_apply(const Geom& geo, cudaStream_t s, const jfftb_green* green,
                       const double* dinv, const double* r, double* out, double2* spec,
                       const double2* tw, int upto);

// stage profile hooks (api.cu); no-ops unless jfftb_profile_start was called
void prof_mark(jfftb_grid* g);         // event at a stage boundary
void prof_end_iter(jfftb_grid* g);     // close the iteration being issued
void prof_collect(jfftb_grid* g, int64_t real_iters, bool final);
void launch_pcg_spectral(const Geom& g, cudaStream_t s, int mode, const double* gpc,
                         const double* gterm, double2* spec, const PcgState* st,
                         double* partials);

}  // namespace jfftb
