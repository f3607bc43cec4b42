// common.cuh -- error handling, device buffers, launch accounting and the
// deterministic reduction / scan building blocks shared by every kernel file.
//
// Determinism: every reduction is a fixed two-pass tree (per-block partials in
// a fixed partition of the index range, then one block per result summing the
// partials in a fixed order).  No floating-point atomics anywhere, so results
// are bitwise reproducible run to run.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <string>
#include <stdexcept>
#include <vector>
#include <algorithm>
#include "../../include/bbot.h"

namespace bbot {

struct Error : public std::runtime_error {
  bbot_status status;
  Error(bbot_status s, const std::string& m) : std::runtime_error(m), status(s) {}
};

#define BB_CUDA(call)                                                                  \
  do {                                                                                 \
    cudaError_t e_ = (call);                                                           \
    if (e_ != cudaSuccess)                                                             \
      throw ::bbot::Error(e_ == cudaErrorMemoryAllocation ? BBOT_E_NOMEM : BBOT_E_CUDA, \
                          std::string(#call) + ": " + cudaGetErrorString(e_) + " @" +  \
                          __FILE__ + ":" + std::to_string(__LINE__));                  \
  } while (0)

#define BB_REQUIRE(cond, status, msg)                                   \
  do {                                                                  \
    if (!(cond)) throw ::bbot::Error(status, std::string(msg));         \
  } while (0)

// Per-context device handle: stream + launch counter + optional per-launch
// event profiler (bbot_prof_start/stop: CUDA events around every launch on the
// launching stream; used by bench.py for the live per-kernel roofline).
struct ProfRec {
  const void* fn;
  cudaEvent_t a, b;
};
struct Dev {
  cudaStream_t stream = nullptr;
  long long launches = 0;
  int num_sms = 148;
  bool prof = false;
  std::vector<ProfRec> recs;
  std::vector<cudaEvent_t> pool;
  cudaEvent_t get_event() {
    if (pool.empty()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      return e;
    }
    cudaEvent_t e = pool.back();
    pool.pop_back();
    return e;
  }
  ~Dev() {
    for (auto& r : recs) { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
    for (auto e : pool) cudaEventDestroy(e);
  }
};

template <class K, class... Args>
inline void launch(Dev& d, K kernel, dim3 grid, dim3 block, size_t smem, Args... args) {
  if (grid.x == 0 || grid.y == 0 || grid.z == 0) return;
  if (d.prof) {
    ProfRec r{(const void*)kernel, d.get_event(), d.get_event()};
    cudaEventRecord(r.a, d.stream);
    kernel<<<grid, block, smem, d.stream>>>(args...);
    cudaEventRecord(r.b, d.stream);
    d.recs.push_back(r);
  } else {
    kernel<<<grid, block, smem, d.stream>>>(args...);
  }
  d.launches++;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess)
    throw Error(BBOT_E_CUDA, std::string("kernel launch: ") + cudaGetErrorString(e));
}

inline unsigned nblocks(long long n, int bs, long long cap = 1LL << 30) {
  long long b = (n + bs - 1) / bs;
  if (b < 1) b = 1;
  if (b > cap) b = cap;
  return (unsigned)b;
}

// Stream-ordered device buffer.
template <class T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  cudaStream_t s = nullptr;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept { p = o.p; n = o.n; s = o.s; o.p = nullptr; o.n = 0; }
  DBuf& operator=(DBuf&& o) noexcept {
    if (this != &o) { release(); p = o.p; n = o.n; s = o.s; o.p = nullptr; o.n = 0; }
    return *this;
  }
  ~DBuf() { release(); }
  void release() {
    if (p) cudaFreeAsync(p, s);
    p = nullptr; n = 0;
  }
  void alloc(size_t count, cudaStream_t st) {
    if (count == n && p && st == s) return;
    release();
    s = st; n = count;
    if (count == 0) return;
    BB_CUDA(cudaMallocAsync((void**)&p, count * sizeof(T), st));
  }
  void zero() { if (n) BB_CUDA(cudaMemsetAsync(p, 0, n * sizeof(T), s)); }
  void upload(const T* h, size_t count) {
    alloc(count, s);
    if (count) BB_CUDA(cudaMemcpyAsync(p, h, count * sizeof(T), cudaMemcpyHostToDevice, s));
  }
  void upload(const std::vector<T>& h, cudaStream_t st) { s = st; upload(h.data(), h.size()); }
  std::vector<T> download() const {
    std::vector<T> h(n);
    if (n) {
      BB_CUDA(cudaMemcpyAsync(h.data(), p, n * sizeof(T), cudaMemcpyDeviceToHost, s));
      BB_CUDA(cudaStreamSynchronize(s));
    }
    return h;
  }
  T* get() const { return p; }
  operator T*() const { return p; }
};

// ---------------------------------------------------------------------------
// block reduction helpers
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_min(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_down_sync(0xffffffffu, v, o));
  return v;
}
// Sum over the block (blockDim.x multiple of 32, <= 1024); result valid in thread 0.
__device__ __forceinline__ double block_sum(double v) {
  __shared__ double sh[32];
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) sh[w] = v;
  __syncthreads();
  int nw = blockDim.x >> 5;
  v = (threadIdx.x < nw) ? sh[threadIdx.x] : 0.0;
  if (w == 0) v = warp_sum(v);
  return v;
}
__device__ __forceinline__ double block_min(double v) {
  __shared__ double shm[32];
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  v = warp_min(v);
  __syncthreads();
  if (lane == 0) shm[w] = v;
  __syncthreads();
  int nw = blockDim.x >> 5;
  v = (threadIdx.x < nw) ? shm[threadIdx.x] : 1e300;
  if (w == 0) v = warp_min(v);
  return v;
}

// Sliced reduction: out[k] = sum_{i < len} f(k, i) for k < nslices.
// Phase 1: grid (parts, nslices), each block sums a fixed contiguous chunk.
template <class F>
__global__ void k_slice_partial(F f, long long len, int parts, double* partial) {
  int k = blockIdx.y;
  long long chunk = (len + parts - 1) / parts;
  long long beg = (long long)blockIdx.x * chunk;
  long long end = beg + chunk < len ? beg + chunk : len;
  double acc = 0.0;
  for (long long i = beg + threadIdx.x; i < end; i += blockDim.x) acc += f(k, i);
  acc = block_sum(acc);
  if (threadIdx.x == 0) partial[(size_t)k * parts + blockIdx.x] = acc;
}
// Phase 2: one block per slice, fixed-order tree over the partials.
__global__ void k_slice_final(const double* partial, int parts, double* out, int op_sqrt);

template <class F>
__global__ void k_slice_partial_min(F f, long long len, int parts, double* partial) {
  int k = blockIdx.y;
  long long chunk = (len + parts - 1) / parts;
  long long beg = (long long)blockIdx.x * chunk;
  long long end = beg + chunk < len ? beg + chunk : len;
  double acc = 1e300;
  for (long long i = beg + threadIdx.x; i < end; i += blockDim.x) acc = fmin(acc, f(k, i));
  acc = block_min(acc);
  if (threadIdx.x == 0) partial[(size_t)k * parts + blockIdx.x] = acc;
}
__global__ void k_slice_final_min(const double* partial, int parts, double* out);

// Workspace for reductions (partials), owned by the context.
struct Reducer {
  Dev* dev = nullptr;
  DBuf<double> partial;
  int parts_for(long long len, int nslices) const {
    long long p = (len + 2047) / 2048;
    long long cap = std::max(1LL, (long long)(4 * dev->num_sms) / std::max(1, nslices));
    if (cap < 1) cap = 1;
    p = std::min(p, std::max(1LL, cap));
    p = std::min(p, 1024LL);
    return (int)std::max(1LL, p);
  }
  void ensure(size_t n) { if (partial.n < n) partial.alloc(std::max(n, (size_t)4096), dev->stream); }

  template <class F>
  void slice_sum(F f, long long len, int nslices, double* out, bool take_sqrt = false) {
    int parts = parts_for(len, nslices);
    ensure((size_t)parts * nslices);
    launch(*dev, k_slice_partial<F>, dim3(parts, nslices), dim3(256), 0, f, len, parts, partial.p);
    launch(*dev, k_slice_final, dim3(nslices), dim3(256), 0, (const double*)partial.p, parts, out,
           (int)take_sqrt);
  }
  template <class F>
  void slice_min(F f, long long len, int nslices, double* out) {
    int parts = parts_for(len, nslices);
    ensure((size_t)parts * nslices);
    launch(*dev, k_slice_partial_min<F>, dim3(parts, nslices), dim3(256), 0, f, len, parts, partial.p);
    launch(*dev, k_slice_final_min, dim3(nslices), dim3(256), 0, (const double*)partial.p, parts, out);
  }
};

// Exclusive scan of int64 (len n) -> out (len n+1, out[n] = total).  In-place safe.
void exclusive_scan(Dev& d, const long long* in, long long* out, long long n, DBuf<long long>& ws);
void exclusive_scan_i32(Dev& d, const int* in, long long* out, long long n, DBuf<long long>& ws);

// Host helpers
inline void sync(Dev& d) { BB_CUDA(cudaStreamSynchronize(d.stream)); }
template <class T>
inline T read_scalar(Dev& d, const T* dptr) {
  T v;
  BB_CUDA(cudaMemcpyAsync(&v, dptr, sizeof(T), cudaMemcpyDeviceToHost, d.stream));
  BB_CUDA(cudaStreamSynchronize(d.stream));
  return v;
}

}  // namespace bbot
