// Host <-> device copies of whole fields for the host-pointer entry points
// (where == JFFTB_HOST: the reference's NumPy arrays cross the boundary here).
//
// Pinned host memory goes straight through the copy engine.  Pageable memory
// (a fresh numpy array, the common case) would be staged by the driver
// through one CPU thread, page faults included -- measured at ~8 GB/s for a
// 3 GiB solution.  Here it goes through a ring of two pinned staging chunks
// instead: the copy engine moves chunk i+1 while a team of host threads
// copies chunk i between the staging buffer and the user's array, so the
// page faults and memcpy run on several cores in parallel with the DMA.
#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <system_error>
#include <thread>
#include <vector>

#include "common.cuh"

namespace jfftb {

namespace {

constexpr size_t kChunk = size_t(32) << 20;       // staging chunk (bytes)
constexpr size_t kDirectBytes = size_t(8) << 20;  // below this: plain cudaMemcpy

int copy_threads() {
  static const int n = [] {
    if (const char* e = std::getenv("JFFTB_COPY_THREADS")) return std::max(1, std::atoi(e));
    const unsigned hc = std::thread::hardware_concurrency();
    return (int)std::min(16u, std::max(1u, hc / 2));
  }();
  return n;
}

bool is_pinned(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();  // clear: unregistered pointers may report an error
    return false;
  }
  return a.type == cudaMemoryTypeHost || a.type == cudaMemoryTypeManaged;
}

struct Staging {
  void* buf[2] = {nullptr, nullptr};
  cudaEvent_t ev[2] = {nullptr, nullptr};
};

Staging& staging(jfftb_grid* g) {
  if (!g->host_stage) {
    auto* st = new Staging;
    for (int b = 0; b < 2; ++b) {
      JF_CUDA(cudaHostAlloc(&st->buf[b], kChunk, cudaHostAllocDefault));
      JF_CUDA(cudaEventCreateWithFlags(&st->ev[b], cudaEventDisableTiming));
    }
    g->host_stage = st;
  }
  return *static_cast<Staging*>(g->host_stage);
}

// Split [0, len) of chunk i among `nt` threads: slice t.
inline void slice(size_t len, int t, int nt, size_t& lo, size_t& hi) {
  const size_t per = (len / nt + 63) & ~size_t(63);
  lo = std::min(len, per * t);
  hi = std::min(len, lo + per);
}

// D2H (to_host) or H2D through the staging ring; returns when the data has
// arrived (D2H: in host memory; H2D: on the device, the stream synchronised).
void staged_copy(jfftb_grid* g, char* host, char* dev, size_t bytes, cudaStream_t s, bool to_host) {
  Staging& st = staging(g);
  const size_t nchunks = (bytes + kChunk - 1) / kChunk;
  const int nt = (int)std::min<size_t>(copy_threads(), std::max<size_t>(1, kChunk >> 20));
  std::vector<std::atomic<int>> arrived(nchunks), gate(nchunks);
  for (size_t i = 0; i < nchunks; ++i) { arrived[i].store(0); gate[i].store(0); }
  std::atomic<int> err{cudaSuccess};
  auto clen = [&](size_t i) { return std::min(kChunk, bytes - i * kChunk); };
  auto issue = [&](size_t i) {  // D2H: device chunk i -> staging; H2D: staging -> device
    const int b = (int)(i & 1);
    cudaError_t e = to_host
        ? cudaMemcpyAsync(st.buf[b], dev + i * kChunk, clen(i), cudaMemcpyDeviceToHost, s)
        : cudaMemcpyAsync(dev + i * kChunk, st.buf[b], clen(i), cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = cudaEventRecord(st.ev[b], s);
    if (e != cudaSuccess) err.store(e);
  };
  if (to_host) {
    issue(0);
    if (nchunks > 1) issue(1);
  }
  auto worker = [&](int t) {
    if (t > 0) cudaSetDevice(g->device);
    for (size_t i = 0; i < nchunks && err.load() == cudaSuccess; ++i) {
      const int b = (int)(i & 1);
      // D2H: chunk i landed in buf[b]; H2D: the DMA out of buf[b] (chunk i-2) is done
      if (to_host || i >= 2) {
        const cudaError_t e = cudaEventSynchronize(st.ev[b]);
        if (e != cudaSuccess) { err.store(e); return; }
      }
      size_t lo, hi;
      slice(clen(i), t, nt, lo, hi);
      if (hi > lo) {
        char* stg = static_cast<char*>(st.buf[b]);
        if (to_host) std::memcpy(host + i * kChunk + lo, stg + lo, hi - lo);
        else std::memcpy(stg + lo, host + i * kChunk + lo, hi - lo);
      }
      if (arrived[i].fetch_add(1) + 1 == nt) {
        // last thread out of chunk i: buf[b] is free (D2H) / filled (H2D)
        if (to_host) { if (i + 2 < nchunks) issue(i + 2); }
        else issue(i);
        gate[i].store(1);
      } else {
        // nobody touches buf[b] again (chunk i+2) before that copy was issued
        while (!gate[i].load() && err.load() == cudaSuccess) std::this_thread::yield();
      }
    }
  };
  std::vector<std::thread> team;
  team.reserve(nt - 1);
  try {
    for (int t = 1; t < nt; ++t) team.emplace_back(worker, t);
  } catch (const std::system_error&) {
    // the started workers would wait for the missing ones: stop them
    err.store(cudaErrorMemoryAllocation);
    for (auto& th : team) th.join();
    JF_CUDA(cudaStreamSynchronize(s));
    throw Error(JFFTB_ECUDA, "staged host copy: cannot start the copy threads");
  }
  worker(0);
  for (auto& th : team) th.join();
  if (err.load() != cudaSuccess)
    throw Error(JFFTB_ECUDA, std::string("staged host copy: ") +
                                 cudaGetErrorString((cudaError_t)err.load()));
  JF_CUDA(cudaStreamSynchronize(s));
}

}  // namespace

void copy_h2d(jfftb_grid* g, void* dst, const void* src, size_t bytes, cudaStream_t s) {
  if (bytes < kDirectBytes || is_pinned(src)) {
    JF_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
    return;
  }
  staged_copy(g, static_cast<char*>(const_cast<void*>(src)), static_cast<char*>(dst), bytes, s,
              false);
}

void copy_d2h(jfftb_grid* g, void* dst, const void* src, size_t bytes, cudaStream_t s) {
  if (bytes < kDirectBytes || is_pinned(dst)) {
    JF_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s));
    JF_CUDA(cudaStreamSynchronize(s));
    return;
  }
  staged_copy(g, static_cast<char*>(dst), static_cast<char*>(const_cast<void*>(src)), bytes, s,
              true);
}

HostPrefault::HostPrefault(void* p, size_t bytes) {
  if (!p || bytes < kChunk || is_pinned(p)) return;
  // a quarter of the copy team: the faults finish well inside any solve long
  // enough for them to matter, and the polling host thread keeps a core
  const int nt = std::max(1, copy_threads() / 4);
  constexpr size_t kPage = 4096;
  char* base = static_cast<char*>(p);
  auto touch = [=](int t) {
    size_t lo, hi;
    slice(bytes, t, nt, lo, hi);
    for (size_t o = (lo + kPage - 1) & ~(kPage - 1); o < hi; o += kPage) {
      volatile char* q = base + o;
      *q = *q;  // write fault, contents unchanged
    }
  };
  // the prefault is an optimisation: if a thread cannot be started, the
  // slices already handed out still run and the rest are left to the copy
  try {
    for (int t = 0; t < nt; ++t) team_.emplace_back(touch, t);
  } catch (const std::system_error&) {
  }
}

void HostPrefault::wait() {
  for (auto& th : team_) th.join();
  team_.clear();
}

void free_host_staging(jfftb_grid* g) {
  if (!g->host_stage) return;
  auto* st = static_cast<Staging*>(g->host_stage);
  for (int b = 0; b < 2; ++b) {
    if (st->buf[b]) cudaFreeHost(st->buf[b]);
    if (st->ev[b]) cudaEventDestroy(st->ev[b]);
  }
  delete st;
  g->host_stage = nullptr;
}

}  // namespace jfftb
