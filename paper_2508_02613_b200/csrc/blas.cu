// Vector algebra and deterministic reductions (solver.py:60-61 `_dot`, the
// axpys of solver.py:119-136, the mean subtraction of solver.py:138).
//
// Every reduction runs a FIXED launch shape (kRedBlocks x kRedThreads) with a
// fixed per-thread stride and a fixed shuffle tree, writes one partial per
// block, and is finished by a single-block fixed-order sum: identical inputs
// give bitwise-identical results (test_solver.py:74-82).
#include "common.cuh"

namespace jfftb {

namespace {

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}

// sum over a 1-D block of blockDim.x (multiple of 32) threads; valid in thread 0
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

__global__ void fill_kernel(double* __restrict__ x, double v, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    x[i] = v;
}

__global__ void copy_kernel(double* __restrict__ d, const double* __restrict__ s, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    d[i] = s[i];
}

__global__ void mul_kernel(double* __restrict__ o, const double* __restrict__ a,
                           const double* __restrict__ b, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    o[i] = a[i] * b[i];
}

// o = a * (a * b)  (apply_jacobi, preconditioners.py:127-129, same order)
__global__ void mul2_kernel(double* __restrict__ o, const double* __restrict__ a,
                            const double* __restrict__ b, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    o[i] = a[i] * (a[i] * b[i]);
}

__global__ void dot_kernel(const double* __restrict__ a, const double* __restrict__ b,
                           int64_t n, double* __restrict__ partials) {
  __shared__ double red[32];
  double s = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    s = fma(a[i], b[i], s);
  s = block_sum1(s, red);
  if (threadIdx.x == 0) partials[blockIdx.x] = s;
}

// out[j] = sum_b partials[b * m + j], fixed order
__global__ void sum_partials_kernel(const double* __restrict__ partials, int count, int m,
                                    double* __restrict__ out) {
  __shared__ double red[32];
  for (int j = 0; j < m; ++j) {
    double s = 0.0;
    for (int b = threadIdx.x; b < count; b += blockDim.x) s += partials[(int64_t)b * m + j];
    s = block_sum1(s, red);
    if (threadIdx.x == 0) out[j] = s;
    __syncthreads();
  }
}

// per-component sums of x (d components of N) -> partials[block*d + comp]
__global__ void comp_sum_kernel(const double* __restrict__ x, int d, int64_t N,
                                double* __restrict__ partials) {
  __shared__ double red[32];
  for (int c = 0; c < d; ++c) {
    double s = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N;
         i += (int64_t)gridDim.x * blockDim.x)
      s += x[c * N + i];
    s = block_sum1(s, red);
    if (threadIdx.x == 0) partials[blockIdx.x * d + c] = s;
    __syncthreads();
  }
}

__global__ void sub_mean_kernel(double* __restrict__ x, int d, int64_t N,
                                const double* __restrict__ sums) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < d * N;
       i += (int64_t)gridDim.x * blockDim.x)
    x[i] -= sums[i / N] / (double)N;
}

int grid_blocks(int64_t n) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 16));
}

}  // namespace

void launch_fill(cudaStream_t s, double* x, double v, int64_t n) {
  fill_kernel<<<grid_blocks(n), 256, 0, s>>>(x, v, n);
  JF_LAUNCHED();
}
void launch_copy(cudaStream_t s, double* dst, const double* src, int64_t n) {
  copy_kernel<<<grid_blocks(n), 256, 0, s>>>(dst, src, n);
  JF_LAUNCHED();
}
void launch_mul(cudaStream_t s, double* out, const double* a, const double* b, int64_t n) {
  mul_kernel<<<grid_blocks(n), 256, 0, s>>>(out, a, b, n);
  JF_LAUNCHED();
}
void launch_mul2(cudaStream_t s, double* out, const double* a, const double* b, int64_t n) {
  mul2_kernel<<<grid_blocks(n), 256, 0, s>>>(out, a, b, n);
  JF_LAUNCHED();
}
void launch_dot(cudaStream_t s, const double* a, const double* b, int64_t n, double* partials) {
  dot_kernel<<<kRedBlocks, kRedThreads, 0, s>>>(a, b, n, partials);
  JF_LAUNCHED();
}
void launch_sum_partials(cudaStream_t s, const double* partials, int count, int m, double* out) {
  sum_partials_kernel<<<1, 1024, 0, s>>>(partials, count, m, out);
  JF_LAUNCHED();
}
void launch_sub_mean(const Geom& g, cudaStream_t s, double* x, double* part) {
  comp_sum_kernel<<<kRedBlocks, kRedThreads, 0, s>>>(x, g.d, g.N, part);
  JF_LAUNCHED();
  double* sums = part + kRedBlocks * g.d;
  sum_partials_kernel<<<1, 1024, 0, s>>>(part, kRedBlocks, g.d, sums);
  JF_LAUNCHED();
  sub_mean_kernel<<<grid_blocks(g.d * g.N), 256, 0, s>>>(x, g.d, g.N, sums);
  JF_LAUNCHED();
}

}  // namespace jfftb
