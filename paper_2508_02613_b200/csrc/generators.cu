// Device input generators: the reference's microstructure
// post-processing (microstructures.py:73-115) on the device, so 512^3 /
// 1024^3 densities are smoothed, thresholded and rescaled where they are
// consumed instead of in a multi-minute NumPy pass.  All of them are
// HBM-streaming elementwise / 3-point kernels.
//
//  binomial filter   gaussian_filter, microstructures.py:73-82 (d-generic:
//                    one periodic [1 2 1]/4 pass per axis, axis 0 first);
//                    per axis v = (v + roll(v, 1) / 2 + roll(v, -1) / 2) / 2
//                    with NumPy's rounding order, so the result is
//                    bit-identical (halving is exact; a contracted
//                    v + a * 0.5 rounds exactly like v + a / 2)
//  rescale_contrast  microstructures.py:104-115, same operation order
//  threshold         microstructures.py:94-101
//  SIMP projection   BASELINE config 5: tanh(beta (v - 1/2)) -> min-max to
//                    [0, 1] -> emin + v^3 (v * v * v)
#include <cmath>
#include <limits>

#include "common.cuh"

namespace jfftb {

namespace {

constexpr int kGenThreads = 256;
constexpr int kGenBlocks = 148 * 8;

__global__ void binomial_axis_kernel(const double* __restrict__ v, double* __restrict__ out,
                                     int64_t N, int64_t stride, int n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)((i / stride) % n);
    const int64_t prev = c == 0 ? i + (int64_t)(n - 1) * stride : i - stride;
    const int64_t next = c == n - 1 ? i - (int64_t)(n - 1) * stride : i + stride;
    // (v + roll(v, 1) / 2 + roll(v, -1) / 2) / 2, left to right
    const double a = __dadd_rn(__ldg(v + i), __ldg(v + prev) * 0.5);
    out[i] = __dadd_rn(a, __ldg(v + next) * 0.5) * 0.5;
  }
}

__global__ void minmax_kernel(const double* __restrict__ v, int64_t N, double* partial) {
  __shared__ double lo_s[32], hi_s[32];
  double lo = std::numeric_limits<double>::infinity(), hi = -lo;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double x = __ldg(v + i);
    lo = fmin(lo, x);
    hi = fmax(hi, x);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    lo = fmin(lo, __shfl_down_sync(0xffffffffu, lo, o));
    hi = fmax(hi, __shfl_down_sync(0xffffffffu, hi, o));
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) { lo_s[wid] = lo; hi_s[wid] = hi; }
  __syncthreads();
  if (wid == 0) {
    const int nw = blockDim.x >> 5;
    lo = lane < nw ? lo_s[lane] : std::numeric_limits<double>::infinity();
    hi = lane < nw ? hi_s[lane] : -std::numeric_limits<double>::infinity();
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      lo = fmin(lo, __shfl_down_sync(0xffffffffu, lo, o));
      hi = fmax(hi, __shfl_down_sync(0xffffffffu, hi, o));
    }
    if (lane == 0) { partial[2 * blockIdx.x] = lo; partial[2 * blockIdx.x + 1] = hi; }
  }
}

__global__ void minmax_final(const double* partial, int count, double* out) {
  double lo = std::numeric_limits<double>::infinity(), hi = -lo;
  for (int i = threadIdx.x; i < count; i += blockDim.x) {
    lo = fmin(lo, partial[2 * i]);
    hi = fmax(hi, partial[2 * i + 1]);
  }
  __shared__ double lo_s[32], hi_s[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    lo = fmin(lo, __shfl_down_sync(0xffffffffu, lo, o));
    hi = fmax(hi, __shfl_down_sync(0xffffffffu, hi, o));
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) { lo_s[wid] = lo; hi_s[wid] = hi; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
      lo = fmin(lo, lo_s[w]);
      hi = fmax(hi, hi_s[w]);
    }
    out[0] = lo;
    out[1] = hi;
  }
}

// soft + (1 - soft) * (v - lo) / (hi - lo), evaluated left to right
__global__ void rescale_kernel(double* __restrict__ v, int64_t N, const double* __restrict__ mm,
                               double soft) {
  const double lo = mm[0], span = __dsub_rn(mm[1], mm[0]);
  const double a = __dsub_rn(1.0, soft);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N;
       i += (int64_t)gridDim.x * blockDim.x)
    v[i] = __dadd_rn(soft, __ddiv_rn(__dmul_rn(a, __dsub_rn(v[i], lo)), span));
}

__global__ void threshold_kernel(double* __restrict__ v, int64_t N, double soft) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N;
       i += (int64_t)gridDim.x * blockDim.x)
    v[i] = v[i] >= 0.5 ? 1.0 : soft;
}

__global__ void tanh_kernel(double* __restrict__ v, int64_t N, double beta) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N;
       i += (int64_t)gridDim.x * blockDim.x)
    v[i] = tanh(__dmul_rn(beta, __dsub_rn(v[i], 0.5)));
}

// (v - lo) / (hi - lo) -> emin + v * v * v
__global__ void simp_kernel(double* __restrict__ v, int64_t N, const double* __restrict__ mm,
                            double emin) {
  const double lo = mm[0], span = __dsub_rn(mm[1], mm[0]);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double x = __ddiv_rn(__dsub_rn(v[i], lo), span);
    v[i] = __dadd_rn(emin, __dmul_rn(__dmul_rn(x, x), x));
  }
}

int gen_blocks(int64_t N) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((N + kGenThreads - 1) / kGenThreads,
                                                     kGenBlocks));
}

}  // namespace

void launch_binomial_filter(const Geom& g, cudaStream_t s, double* field, double* scratch,
                            int passes) {
  // per axis: stride of axis a = product of the later extents
  double* src = field;
  double* dst = scratch;
  for (int p = 0; p < passes; ++p) {
    for (int a = 0; a < g.d; ++a) {
      int64_t stride = 1;
      for (int b = a + 1; b < g.d; ++b) stride *= g.n[b];
      binomial_axis_kernel<<<gen_blocks(g.N), kGenThreads, 0, s>>>(src, dst, g.N, stride,
                                                                    g.n[a]);
      JF_LAUNCHED();
      std::swap(src, dst);
    }
  }
  if (src != field) {
    JF_CUDA(cudaMemcpyAsync(field, src, sizeof(double) * g.N, cudaMemcpyDeviceToDevice, s));
  }
}

void launch_minmax(const Geom& g, cudaStream_t s, const double* field, double* partial,
                   double* out2) {
  const int blocks = gen_blocks(g.N);
  minmax_kernel<<<blocks, kGenThreads, 0, s>>>(field, g.N, partial);
  JF_LAUNCHED();
  minmax_final<<<1, 1024, 0, s>>>(partial, blocks, out2);
  JF_LAUNCHED();
}

void launch_rescale(const Geom& g, cudaStream_t s, double* field, const double* mm, double soft) {
  rescale_kernel<<<gen_blocks(g.N), kGenThreads, 0, s>>>(field, g.N, mm, soft);
  JF_LAUNCHED();
}

void launch_threshold(const Geom& g, cudaStream_t s, double* field, double soft) {
  threshold_kernel<<<gen_blocks(g.N), kGenThreads, 0, s>>>(field, g.N, soft);
  JF_LAUNCHED();
}

void launch_simp(const Geom& g, cudaStream_t s, double* field, double* partial, double* mm,
                 double beta, double emin) {
  tanh_kernel<<<gen_blocks(g.N), kGenThreads, 0, s>>>(field, g.N, beta);
  JF_LAUNCHED();
  launch_minmax(g, s, field, partial, mm);
  simp_kernel<<<gen_blocks(g.N), kGenThreads, 0, s>>>(field, g.N, mm, emin);
  JF_LAUNCHED();
}

int gen_partials(const Geom& g) { return 2 * gen_blocks(g.N) + 2; }

// ---------------------------------------------------------------------------
// field file layout (grid.py:225-295): every plane of the raw payload is
// "x1-fastest" (Fortran order of the n0 x ... x n_{d-1} array).  Converting
// between that and the C order of device fields swaps axes 0 and d-1 (the
// middle axis of a 3-D field keeps its stride): a 32 x 32 tiled transpose
// per (plane, middle index), coalesced on both sides.
// ---------------------------------------------------------------------------
namespace {
__global__ void swap_outer_axes_kernel(const double* __restrict__ src, double* __restrict__ dst,
                                       int na, int nm, int nb) {
  // src viewed as [q][b][m][a] (a fastest), dst as [q][a][m][b] (b fastest)
  __shared__ double tile[32][33];
  const int64_t q = blockIdx.z / nm;
  const int m = blockIdx.z % nm;
  const int64_t plane = (int64_t)na * nm * nb;
  const int a0 = blockIdx.x * 32, b0 = blockIdx.y * 32;
  const double* s = src + q * plane;
  double* o = dst + q * plane;
  for (int j = threadIdx.y; j < 32; j += blockDim.y) {
    const int a = a0 + threadIdx.x, b = b0 + j;
    if (a < na && b < nb) tile[j][threadIdx.x] = s[((int64_t)b * nm + m) * na + a];
  }
  __syncthreads();
  for (int j = threadIdx.y; j < 32; j += blockDim.y) {
    const int b = b0 + threadIdx.x, a = a0 + j;
    if (a < na && b < nb) o[((int64_t)a * nm + m) * nb + b] = tile[threadIdx.x][j];
  }
}
}  // namespace

// planes of x1-fastest (Fortran) order <-> C order; to_c selects the direction
void launch_fortran_to_c(const Geom& g, cudaStream_t s, const double* src, double* dst,
                         int planes, bool to_c) {
  const int n0 = g.n[0], nl = g.n[g.d - 1];
  const int nm = g.d == 3 ? g.n[1] : 1;
  // Fortran: axis 0 fastest -> viewed as [b = axis d-1][m][a = axis 0]
  const int na = to_c ? n0 : nl, nb = to_c ? nl : n0;
  dim3 grid((na + 31) / 32, (nb + 31) / 32, (unsigned)(planes * nm));
  swap_outer_axes_kernel<<<grid, dim3(32, 8), 0, s>>>(src, dst, na, nm, nb);
  JF_LAUNCHED();
}

}  // namespace jfftb
