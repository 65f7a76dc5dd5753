// Device FFT building blocks for the fused spectral passes (fused.cu).
//
// cta_fft<L, NSEQ, NT, INV> transforms NSEQ sequences of length L (power of
// two, 2..2048) held in shared memory, element k of sequence q at
// buf[q * qs + k * ks], with a Stockham autosort radix-8 (+ one radix-2/4)
// schedule.  Every stage reads all its butterfly inputs into registers,
// barriers, and writes in place, so no ping-pong buffer is needed; NT threads
// share the NSEQ * L / R butterflies of a stage.  Twiddles come from
// per-stage tables copied out of one 4096-entry table of exp(-2 pi i j / 4096)
// (fp64, built once per grid), laid out so a warp's reads are contiguous.
// Forward = numpy's unnormalised exp(-i...) convention; INV = exp(+i...)
// without the 1/L factor (folded into the spectral multiply).
#pragma once

#include "common.cuh"

namespace jfftb {

constexpr int kTwN = 4096;

// Per-stage twiddle tables follow the 4096-entry table: the stage of span
// P = NS * R (radix R) reads w_P^(j t) for j < NS, t = 1..R-1 at
// [(t - 1) * NS + j], so the threads of a warp (consecutive j) read
// consecutive entries -- a strided walk through the 4096 table would touch
// one cache line per thread in the late stages.  Same values, bit for bit.
__host__ __device__ constexpr int ilog2c(int x) { return x <= 1 ? 0 : 1 + ilog2c(x / 2); }
__host__ __device__ constexpr int tw_ridx(int R) { return R == 8 ? 0 : (R == 4 ? 1 : 2); }
__host__ __device__ constexpr int tw_stage_off(int P, int R) {
  return 4096 + (ilog2c(P) * 3 + tw_ridx(R)) * 4096;
}

// Ampere+ asynchronous global -> shared copies (LDGSTS), used to prefetch the
// next tile while the current one is transformed
__device__ __forceinline__ void cpa16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cpa8(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cpa_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// Bulk (TMA engine) global -> shared copies completing on an mbarrier: one
// thread moves a whole contiguous block without per-thread LDGSTS issue
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "JF_WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra JF_WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// order this thread's earlier generic-proxy shared accesses (after a CTA
// barrier: everyone's) before subsequent async-proxy (bulk copy) writes
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// L2 prefetches: one 128-byte line / a contiguous block (bulk, TMA engine)
__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];\n" ::"l"(p));
}
__device__ __forceinline__ void bulk_prefetch_l2(const void* p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(p), "r"(bytes) : "memory");
}

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cmulc(double2 a, double2 b) {  // a * conj(b)
  return make_double2(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y);
}
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
// multiply by -i (forward) or +i (inverse)
template <bool INV>
__device__ __forceinline__ double2 mul_mi(double2 a) {
  return INV ? make_double2(-a.y, a.x) : make_double2(a.y, -a.x);
}

template <bool INV>
__device__ __forceinline__ void dft2(double2& a, double2& b) {
  const double2 t = a;
  a = cadd(t, b);
  b = csub(t, b);
}

template <bool INV>
__device__ __forceinline__ void dft4(double2& v0, double2& v1, double2& v2, double2& v3) {
  const double2 t0 = cadd(v0, v2), t1 = csub(v0, v2);
  const double2 t2 = cadd(v1, v3), t3 = mul_mi<INV>(csub(v1, v3));
  v0 = cadd(t0, t2);
  v2 = csub(t0, t2);
  v1 = cadd(t1, t3);
  v3 = csub(t1, t3);
}

template <bool INV>
__device__ __forceinline__ void dft8(double2 (&v)[8]) {
  constexpr double h = 0.70710678118654752440;
  double2 e0 = v[0], e1 = v[2], e2 = v[4], e3 = v[6];
  double2 o0 = v[1], o1 = v[3], o2 = v[5], o3 = v[7];
  dft4<INV>(e0, e1, e2, e3);
  dft4<INV>(o0, o1, o2, o3);
  // W8^1 = h(1 -+ i), W8^2 = -+i, W8^3 = h(-1 -+ i)
  const double2 w1o1 = INV ? make_double2(h * (o1.x - o1.y), h * (o1.x + o1.y))
                           : make_double2(h * (o1.x + o1.y), h * (o1.y - o1.x));
  const double2 w2o2 = mul_mi<INV>(o2);
  const double2 w3o3 = INV ? make_double2(-h * (o3.x + o3.y), h * (o3.x - o3.y))
                           : make_double2(h * (o3.y - o3.x), -h * (o3.x + o3.y));
  v[0] = cadd(e0, o0);
  v[4] = csub(e0, o0);
  v[1] = cadd(e1, w1o1);
  v[5] = csub(e1, w1o1);
  v[2] = cadd(e2, w2o2);
  v[6] = csub(e2, w2o2);
  v[3] = cadd(e3, w3o3);
  v[7] = csub(e3, w3o3);
}

// radix of stage s for length L: radix-8 stages first, one trailing 2 or 4
__host__ __device__ constexpr int fft_nstages(int L) {
  int s = 0;
  while (L >= 8) { L /= 8; ++s; }
  return s + (L > 1 ? 1 : 0);
}
__host__ __device__ constexpr int fft_radix(int L, int s) {
  int full = 0, r = L;
  while (r >= 8) { r /= 8; ++full; }
  return s < full ? 8 : r;
}

template <int R, bool INV>
__device__ __forceinline__ void dftR(double2 (&v)[8]) {
  if (R == 8) dft8<INV>(v);
  else if (R == 4) dft4<INV>(v[0], v[1], v[2], v[3]);
  else if (R == 2) dft2<INV>(v[0], v[1]);
}

// element k of a sequence sits at pidx(k) * ks: PAD inserts one slot every 8
// elements so that the radix-8 stride patterns of contiguous (ks = 1) rows
// stay free of shared-memory bank conflicts
template <int PAD>
__device__ __forceinline__ int pidx(int k) {
  if constexpr (PAD > 0) return k + k / PAD;
  else return k;
}
template <int PAD>
__host__ __device__ constexpr int padded_len(int L) {
  if constexpr (PAD > 0) return L + L / PAD;
  else return L;
}

// QFAST: consecutive threads take consecutive sequences (layouts with qs = 1,
// sequences interleaved); otherwise consecutive butterflies of one sequence
// WARP: the calling warp alone transforms its sequences (NT = 32, lane-indexed,
// __syncwarp between stages) -- no block-wide barrier
// GIN: the first stage reads its inputs from global memory (sequence q
// contiguous at gin + q * gqs; L2 loads, never through L1: the merged pass
// B/C/B' reads rows other SMs wrote during the same launch) instead of buf; GOUT: the last stage writes
// its outputs to gout + q * gqs (no trailing barrier -- buf is only read).
template <int L, int NSEQ, int NT, bool INV, bool QFAST, int PAD, int S, int NS, bool WARP = false,
          bool GIN = false, bool GOUT = false, bool SEG = false>
__device__ __forceinline__ void cta_fft_stage(double2* buf, int ks, int qs,
                                              const double2* __restrict__ tw,
                                              const double2* gin = nullptr,
                                              double2* gout = nullptr, int64_t gqs = 0,
                                              int64_t gks = 1, int gsh = 0, int64_t gss = 0) {
  // global element k of a sequence: k gks, or with SEG the segmented
  // (k >> gsh) gss + (k & (2^gsh - 1)) gks
  auto gix = [&](int k) -> int64_t {
    if constexpr (SEG) return (int64_t)(k >> gsh) * gss + (int64_t)(k & ((1 << gsh) - 1)) * gks;
    else return (int64_t)k * gks;
  };
  if constexpr (S < fft_nstages(L)) {
    constexpr bool FROM_G = GIN && S == 0;
    constexpr bool TO_G = GOUT && S + 1 == fft_nstages(L);
    constexpr int R = fft_radix(L, S);
    constexpr int NB = L / R;            // butterflies per sequence
    constexpr int B = NSEQ * NB;         // butterflies per stage
    constexpr int PER = (B + NT - 1) / NT;
    static_assert(!WARP || NT == 32, "warp FFT runs on 32 lanes");
    const int tid = WARP ? (int)(threadIdx.x & 31) : (int)threadIdx.x;
    // SHARE: every butterfly of this thread has the same index j within its
    // sequence (NT a multiple of NB), so the twiddles are fetched once
    constexpr bool SHARE = !QFAST && PER > 1 && NT % NB == 0 && B % NT == 0;
    double2 v[PER][8];
    int qq[PER], jj[PER];
    double2 ws[SHARE ? 8 : 1];
    const double2* __restrict__ tws = tw + tw_stage_off(NS * R, R);
    if constexpr (SHARE) {
      if (NS > 1) {
        const int jb = (tid % NB) % NS;
#pragma unroll
        for (int t = 1; t < R; ++t) ws[SHARE ? t : 0] = __ldg(tws + (t - 1) * NS + jb);
      }
    }
#pragma unroll
    for (int m = 0; m < PER; ++m) {
      const int b = tid + m * NT;
      qq[m] = QFAST ? b % NSEQ : (SHARE ? tid / NB + m * (NT / NB) : b / NB);
      jj[m] = QFAST ? b / NSEQ : (SHARE ? tid % NB : b % NB);
      if (B % NT == 0 || b < B) {
        if constexpr (FROM_G) {
          const double2* src = gin + qq[m] * gqs;
#pragma unroll
          for (int t = 0; t < R; ++t) v[m][t] = __ldcg(src + gix(jj[m] + t * NB));
        } else {
          const double2* src = buf + qq[m] * qs;
#pragma unroll
          for (int t = 0; t < R; ++t) v[m][t] = src[pidx<PAD>(jj[m] + t * NB) * ks];
        }
        if (NS > 1) {
          const int jb = jj[m] % NS;
#pragma unroll
          for (int t = 1; t < R; ++t) {
            const double2 w = SHARE ? ws[SHARE ? t : 0] : __ldg(tws + (t - 1) * NS + jb);
            v[m][t] = INV ? cmulc(v[m][t], w) : cmul(v[m][t], w);
          }
        }
        dftR<R, INV>(v[m]);
      }
    }
    if constexpr (!FROM_G) {
      if (WARP) __syncwarp(); else __syncthreads();
    }
#pragma unroll
    for (int m = 0; m < PER; ++m) {
      const int b = tid + m * NT;
      if (B % NT == 0 || b < B) {
        const int j = jj[m];
        const int o = (j / NS) * NS * R + (j % NS);
        if constexpr (TO_G) {
          double2* dst = gout + qq[m] * gqs;
#pragma unroll
          for (int t = 0; t < R; ++t) dst[gix(o + t * NS)] = v[m][t];
        } else {
          double2* dst = buf + qq[m] * qs;
#pragma unroll
          for (int t = 0; t < R; ++t) dst[pidx<PAD>(o + t * NS) * ks] = v[m][t];
        }
      }
    }
    if constexpr (!TO_G) {
      if (WARP) __syncwarp(); else __syncthreads();
    }
    cta_fft_stage<L, NSEQ, NT, INV, QFAST, PAD, S + 1, NS * R, WARP, GIN, GOUT, SEG>(
        buf, ks, qs, tw, gin, gout, gqs, gks, gsh, gss);
  }
}

// Transform NSEQ sequences in smem in place.  Caller must __syncthreads()
// before (data written) -- this routine ends with a barrier.
template <int L, int NSEQ, int NT, bool INV, bool QFAST = true, int PAD = 0>
__device__ __forceinline__ void cta_fft(double2* buf, int ks, int qs,
                                        const double2* __restrict__ tw) {
  cta_fft_stage<L, NSEQ, NT, INV, QFAST, PAD, 0, 1>(buf, ks, qs, tw);
}
// Sequences transformed on the way between global and shared memory: GIN
// reads the first stage's inputs from gin + q * gqs + k * gks (no prior smem
// staging; the caller barriers before, as buf is written by the first
// stage), GOUT writes the last stage's outputs to gout + q * gqs + k * gks.
template <int L, int NSEQ, int NT, bool INV, bool QFAST, int PAD, bool GIN, bool GOUT,
          bool SEG = false>
__device__ __forceinline__ void cta_fft_io(double2* buf, int ks, int qs,
                                           const double2* __restrict__ tw, const double2* gin,
                                           double2* gout, int64_t gqs, int64_t gks, int gsh = 0,
                                           int64_t gss = 0) {
  cta_fft_stage<L, NSEQ, NT, INV, QFAST, PAD, 0, 1, false, GIN, GOUT, SEG>(
      buf, ks, qs, tw, gin, gout, gqs, gks, gsh, gss);
}

// ---------------------------------------------------------------------------
// In-place mixed-radix transforms (radix-8 stages, one trailing 2 or 4):
// forward decimation in frequency (natural order in, digit-reversed out),
// inverse decimation in time (digit-reversed in, natural out).  Every thread
// reads and writes the same R elements of a stage, so a stage needs one
// barrier (after its writes) instead of the Stockham schedule's two.  Stage s
// of length-L sequences works on blocks of P_s = L / (R_0 ... R_{s-1})
// elements; butterfly (block, j < Q = P_s / R_s) takes elements
// block P_s + j + Q t.  Forward: DFT_R, then output t times w_P^(j t);
// inverse: input t times conj(w_P^(j t)), then the inverse DFT_R (no 1/L).
// Frequency k of the forward transform sits at slot dif_pos(L, k).
// ---------------------------------------------------------------------------
__host__ __device__ constexpr int fft_span(int L, int s) {
  int p = L;
  for (int i = 0; i < s; ++i) p /= fft_radix(L, i);
  return p;
}
__host__ __device__ constexpr int dif_pos(int L, int k) {
  int pos = 0, block = L;
  for (int s = 0; s < fft_nstages(L); ++s) {
    const int R = fft_radix(L, s);
    block /= R;
    pos += (k % R) * block;
    k /= R;
  }
  return pos;
}
__host__ __device__ constexpr int dif_freq(int L, int p) {
  int k = 0, mult = 1, block = L;
  for (int s = 0; s < fft_nstages(L); ++s) {
    const int R = fft_radix(L, s);
    block /= R;
    k += (p / block) * mult;
    p %= block;
    mult *= R;
  }
  return k;
}

// one in-place stage; sequences are contiguous rows at buf + q * qs (element
// e at pidx<PAD>(e)); GIN: forward stage 0 reads gin + q * gqs + e; GOUT:
// inverse stage 0 writes gout + q * gqs + e instead of buf
// QF: interleaved sequences (element e of sequence q at buf[e * ks + q],
// consecutive threads take consecutive sequences); otherwise rows at
// buf + q * qs with consecutive threads on consecutive butterflies
template <int L, int NSEQ, int NT, bool INV, int PAD, int S, bool GIN, bool GOUT, bool QF = false>
__device__ __forceinline__ void cta_fft_ip_stage(double2* buf, int qs,
                                                 const double2* __restrict__ tw,
                                                 const double2* gin, double2* gout,
                                                 int64_t gqs, int ks = 1) {
  constexpr int R = fft_radix(L, S);
  constexpr int P = fft_span(L, S);
  constexpr int Q = P / R;
  constexpr int NB = L / R;          // butterflies per sequence
  constexpr int B = NSEQ * NB;
  constexpr int PER = (B + NT - 1) / NT;
  constexpr bool FROM_G = GIN && !INV && S == 0;
  constexpr bool TO_G = GOUT && INV && S == 0;
  const double2* __restrict__ tws = tw + tw_stage_off(P, R);
#pragma unroll
  for (int m = 0; m < PER; ++m) {
    const int b = threadIdx.x + m * NT;
    if (B % NT == 0 || b < B) {
      const int q = QF ? b % NSEQ : b / NB, bb = QF ? b / NSEQ : b % NB;
      const int j = bb % Q;
      const int base = (bb / Q) * P + j;
      double2 v[8];
      if constexpr (FROM_G) {
        const double2* src = gin + q * gqs;
#pragma unroll
        for (int t = 0; t < R; ++t) v[t] = __ldcg(src + base + Q * t);
      } else if constexpr (QF) {
#pragma unroll
        for (int t = 0; t < R; ++t) v[t] = buf[(base + Q * t) * ks + q];
      } else {
        const double2* src = buf + q * qs;
#pragma unroll
        for (int t = 0; t < R; ++t) v[t] = src[pidx<PAD>(base + Q * t)];
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
      if constexpr (TO_G) {
        double2* dst = gout + q * gqs;
#pragma unroll
        for (int t = 0; t < R; ++t) dst[base + Q * t] = v[t];
      } else if constexpr (QF) {
#pragma unroll
        for (int t = 0; t < R; ++t) buf[(base + Q * t) * ks + q] = v[t];
      } else {
        double2* dst = buf + q * qs;
#pragma unroll
        for (int t = 0; t < R; ++t) dst[pidx<PAD>(base + Q * t)] = v[t];
      }
    }
  }
  if constexpr (!TO_G) __syncthreads();
}

// stages S .. END-1 (END < nstages leaves the last stages to the caller)
template <int L, int NSEQ, int NT, int PAD, bool GIN, int S = 0, int END = fft_nstages(L)>
__device__ __forceinline__ void cta_fft_dif(double2* buf, int qs, const double2* __restrict__ tw,
                                            const double2* gin, int64_t gqs) {
  if constexpr (S < END) {
    cta_fft_ip_stage<L, NSEQ, NT, false, PAD, S, GIN, false>(buf, qs, tw, gin, nullptr, gqs);
    cta_fft_dif<L, NSEQ, NT, PAD, GIN, S + 1, END>(buf, qs, tw, gin, gqs);
  }
}
// forward in-place DIF of interleaved sequences, stages S.. (S0 = 1 when the
// caller did stage 0 in registers)
template <int L, int NSEQ, int NT, int S>
__device__ __forceinline__ void cta_fft_dif_qf(double2* buf, int ks, const double2* __restrict__ tw) {
  if constexpr (S < fft_nstages(L)) {
    cta_fft_ip_stage<L, NSEQ, NT, false, 0, S, false, false, true>(buf, 0, tw, nullptr, nullptr, 0,
                                                                   ks);
    cta_fft_dif_qf<L, NSEQ, NT, S + 1>(buf, ks, tw);
  }
}

// stages S .. END-1 of cta_fft_dif_qf (the caller fuses the rest)
template <int L, int NSEQ, int NT, int S, int END>
__device__ __forceinline__ void cta_fft_dif_qf_until(double2* buf, int ks,
                                                     const double2* __restrict__ tw) {
  if constexpr (S < END) {
    cta_fft_ip_stage<L, NSEQ, NT, false, 0, S, false, false, true>(buf, 0, tw, nullptr, nullptr, 0,
                                                                   ks);
    cta_fft_dif_qf_until<L, NSEQ, NT, S + 1, END>(buf, ks, tw);
  }
}

template <int L, int NSEQ, int NT, int PAD, bool GOUT, int S = fft_nstages(L) - 1>
__device__ __forceinline__ void cta_fft_dit_inv(double2* buf, int qs,
                                                const double2* __restrict__ tw, double2* gout,
                                                int64_t gqs) {
  if constexpr (S >= 0) {
    cta_fft_ip_stage<L, NSEQ, NT, true, PAD, S, false, GOUT>(buf, qs, tw, nullptr, gout, gqs);
    cta_fft_dit_inv<L, NSEQ, NT, PAD, GOUT, S - 1>(buf, qs, tw, gout, gqs);
  }
}

// exp(-2 pi i j / 4096), j < 4096
void launch_twiddles(cudaStream_t s, double2* tw);

}  // namespace jfftb
