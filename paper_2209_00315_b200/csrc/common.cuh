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

// resident CTAs per SM requested by the fused level-0 A_k kernels (k_pcg_pq, k_up_dot):
// 8 x 256 threads caps them at 32 registers (full occupancy; the gathers are latency-bound)
#ifndef BBOT_LAP_MINB
#define BBOT_LAP_MINB 8
#endif
// residual-based post sweeps of AMG(A) (amg.cu: k_up_dot_res, k_up_res): defaults of the
// BBOT_LAP_RES (level 0), BBOT_SELL_RES (SELL levels) and BBOT_LAP_RDINV (level 0: 1/diag
// recomputed from the row's slots instead of read) knobs
#ifndef BBOT_LAP_RES_DEFAULT
#define BBOT_LAP_RES_DEFAULT 1
#endif
#ifndef BBOT_LAP_RDINV_DEFAULT
#define BBOT_LAP_RDINV_DEFAULT 1
#endif
#ifndef BBOT_SELL_RES_DEFAULT
#define BBOT_SELL_RES_DEFAULT 1
#endif

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
  long long grid;     // CTAs of the launch (tells the levels of a multigrid kernel apart)
};
struct Dev {
  cudaStream_t stream = nullptr;
  long long launches = 0;
  int num_sms = 148;
  bool prof = false;
  bool capturing = false;      // kernels are being captured into a CUDA graph
  bool sync_check = false;     // BBOT_SYNC_CHECK=1: synchronise after every eager launch (debug)
  int depth = 0;               // nesting depth of device loops being captured
  std::vector<cudaStream_t> cap_streams;
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
    for (auto st : cap_streams) cudaStreamDestroy(st);
    for (auto& r : recs) { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
    for (auto e : pool) cudaEventDestroy(e);
  }
};

template <class K, class... Args>
inline void launch(Dev& d, K kernel, dim3 grid, dim3 block, size_t smem, Args... args) {
  if (grid.x == 0 || grid.y == 0 || grid.z == 0) return;
  if (d.prof && !d.capturing) {
    ProfRec r{(const void*)kernel, d.get_event(), d.get_event(), (long long)grid.x * grid.y * grid.z};
    cudaEventRecord(r.a, d.stream);
    kernel<<<grid, block, smem, d.stream>>>(args...);
    cudaEventRecord(r.b, d.stream);
    d.recs.push_back(r);
  } else {
    kernel<<<grid, block, smem, d.stream>>>(args...);
  }
  if (!d.capturing) d.launches++;
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess && d.sync_check && !d.capturing) e = cudaStreamSynchronize(d.stream);
  if (e != cudaSuccess) {
    const char* nm = nullptr;
    cudaFuncGetName(&nm, (const void*)kernel);
    throw Error(BBOT_E_CUDA, std::string("kernel ") + (nm ? nm : "?") + ": " + cudaGetErrorString(e));
  }
}

// launch with a thread-block cluster of `cl` CTAs along x (grid.x multiple of cl)
template <class K, class... Args>
inline void launch_cluster(Dev& d, K kernel, dim3 grid, dim3 block, size_t smem, int cl, Args... args) {
  if (grid.x == 0) return;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = d.stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cl;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  ProfRec r{(const void*)kernel, nullptr, nullptr, (long long)grid.x * grid.y * grid.z};
  bool prof = d.prof && !d.capturing;
  if (prof) {
    r.a = d.get_event();
    r.b = d.get_event();
    cudaEventRecord(r.a, d.stream);
  }
  cudaError_t e = cudaLaunchKernelEx(&cfg, kernel, args...);
  if (prof) {
    cudaEventRecord(r.b, d.stream);
    d.recs.push_back(r);
  }
  if (!d.capturing) d.launches++;
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e == cudaSuccess && d.sync_check && !d.capturing) e = cudaStreamSynchronize(d.stream);
  if (e != cudaSuccess) throw Error(BBOT_E_CUDA, std::string("cluster kernel launch: ") + cudaGetErrorString(e));
}

inline unsigned nblocks(long long n, int bs, long long cap = 1LL << 30) {
  long long b = (n + bs - 1) / bs;
  if (b < 1) b = 1;
  if (b > cap) b = cap;
  return (unsigned)b;
}

// The library's private stream-ordered memory pool on the current device (created on
// first use, release threshold raised so the AMG hierarchies rebuilt every Newton step
// do not unmap/remap pages at each sync).  The device default pool -- shared with the
// host framework -- is left untouched.
cudaMemPool_t device_pool();

// Stream-ordered device buffer (allocated from device_pool()).
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
    BB_CUDA(cudaMallocFromPoolAsync((void**)&p, count * sizeof(T), device_pool(), st));
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
// The reconstruction of rho-bar on a fine edge: arithmetic (A3) or the weighted
// harmonic mean (NEXT f4, A39) of the two lifted values a (left), b (right):
//   f = 1 / (lam/a + (1-lam)/b),  df/da = lam f^2/a^2,  df/db = (1-lam) f^2/b^2,
//   d2f/da2 = 2 lam f^2 a^-3 (lam f/a - 1),  d2f/dadb = 2 lam (1-lam) f^3 a^-2 b^-2,
//   d2f/db2 = 2 (1-lam) f^2 b^-3 ((1-lam) f/b - 1)   (oracle/ops.py recon_*).
struct Recon {
  double f, ja, jb;
  __device__ __forceinline__ static Recon eval(int harm, double lam, double a, double b) {
    Recon r;
    if (!harm) {
      r.f = lam * a + (1.0 - lam) * b;
      r.ja = lam;
      r.jb = 1.0 - lam;
    } else {
      r.f = 1.0 / (lam / a + (1.0 - lam) / b);
      double f2 = r.f * r.f;
      r.ja = lam * f2 / (a * a);
      r.jb = (1.0 - lam) * f2 / (b * b);
    }
    return r;
  }
  // (haa, hab, hbb) of the harmonic mean
  __device__ __forceinline__ static void hess(double lam, double a, double b, double& haa, double& hab,
                                              double& hbb) {
    double f = 1.0 / (lam / a + (1.0 - lam) / b);
    haa = 2.0 * lam * f * f / (a * a * a) * (lam * f / a - 1.0);
    hbb = 2.0 * (1.0 - lam) * f * f / (b * b * b) * ((1.0 - lam) * f / b - 1.0);
    hab = 2.0 * lam * (1.0 - lam) * f * f * f / (a * a * b * b);
  }
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
// partial[k * parts + blockIdx.x] = block sum of acc[k] for k < cnt (<= NR): per value the
// same butterfly order as block_sum (bitwise-identical partials), one barrier in total
// instead of two per value.  Writers fence before red_last_block's counter increment.
template <int NR>
__device__ __forceinline__ void block_sum_many(const double (&acc)[NR], int cnt, double* partial, int parts) {
  __shared__ double shn[NR][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int k = 0; k < NR; k++)
    if (k < cnt) {
      double v = warp_sum(acc[k]);
      if (lane == 0) shn[k][w] = v;
    }
  __syncthreads();
  for (int k = w; k < cnt; k += nw) {
    double v = lane < nw ? shn[k][lane] : 0.0;
    v = warp_sum(v);
    if (lane == 0) {
      partial[(size_t)k * parts + blockIdx.x] = v;
      __threadfence();
    }
  }
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

// ---------------------------------------------------------------------------
// Deterministic single-launch reductions ("last block finishes").
//
// Grid (parts, ns): block (p, k) reduces a fixed contiguous chunk of slice k and
// writes its partial to partial[k*parts + p]; the block that arrives last at the
// counter sums every slice's partials in a fixed order (warp per slice, lanes
// strided, shuffle tree) into out[k] and then runs the caller's epilogue.  The
// result depends only on (len, ns, parts), never on block scheduling, so it is
// bitwise reproducible, and the scalar logic that consumes it (Givens rotations,
// PCG alpha/beta, loop conditions) runs in the same launch.  One counter per
// Reducer: launches on one stream are serialised, and the last block re-arms it.
struct RedArgs {
  double* partial;
  unsigned* counter;
  double* out;       // per-slice results of the launched slices (out[0] = slice k0)
  int parts;
  int k0;            // first slice of the launch (time slabs: a rank launches its own slices)
};

// Called by all threads of every block after the block's partial(s) are written
// by thread 0.  Returns true in all threads of the last block.
__device__ __forceinline__ bool red_last_block(unsigned* counter) {
  __shared__ int s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    unsigned total = gridDim.x * gridDim.y;
    unsigned t = atomicAdd(counter, 1u);
    s_last = (t == total - 1) ? 1 : 0;
    if (s_last) {
      __threadfence();
      *counter = 0u;
    }
  }
  __syncthreads();
  return s_last != 0;
}

// Last block only: out[s] = sum_p partial[s*parts + p], s < ns.  Ends with a barrier.
__device__ __forceinline__ void red_finish(const double* partial, int parts, int ns, double* out) {
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int s = w; s < ns; s += nw) {
    double v = 0.0;
    for (int p = lane; p < parts; p += 32) v += __ldcg(partial + (size_t)s * parts + p);
    v = warp_sum(v);
    if (lane == 0) out[s] = v;
  }
  __syncthreads();
}

// Block (p, k) of a (parts, ns) grid: reduce acc and commit; last block finishes.
// (A two-level variant -- the last block of each slice summing that slice -- measured 12 %
// slower on the C4 PCG kernels: the per-slice counters share a few contended L2 lines.)
__device__ __forceinline__ bool red_commit(double acc, const RedArgs& R) {
  acc = block_sum(acc);
  if (threadIdx.x == 0) R.partial[(size_t)blockIdx.y * R.parts + blockIdx.x] = acc;
  if (!red_last_block(R.counter)) return false;
  red_finish(R.partial, R.parts, gridDim.y, R.out);
  return true;
}

// chunk of slice-local indices owned by block p
__device__ __forceinline__ void red_chunk(long long len, int parts, long long& beg, long long& end) {
  long long chunk = (len + parts - 1) / parts;
  beg = (long long)blockIdx.x * chunk;
  end = beg + chunk < len ? beg + chunk : len;
}

struct NoFin {
  __device__ void operator()(const double*) const {}
};
struct SqrtFin {   // out[k] = sqrt(out[k])
  double* out;
  int ns;
  __device__ void operator()(const double*) const {
    for (int k = threadIdx.x; k < ns; k += blockDim.x) out[k] = sqrt(out[k]);
  }
};

// out[k] = sum_{i < len} f(k, i); then fin(out) in the last block (all threads).
template <class F, class Fin>
__global__ void k_slice_reduce(F f, long long len, RedArgs R, Fin fin) {
  int k = R.k0 + blockIdx.y;
  long long beg, end;
  red_chunk(len, R.parts, beg, end);
  double acc = 0.0;
  for (long long i = beg + threadIdx.x; i < end; i += blockDim.x) acc += f(k, i);
  if (red_commit(acc, R)) fin(R.out);
}

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

// Reduction workspace, owned by the context.  Sized once at creation (nothing is
// allocated while a CUDA graph is being captured).
struct Reducer {
  Dev* dev = nullptr;
  DBuf<double> partial;
  DBuf<unsigned> counter;
  size_t cap = 0;
  static constexpr int BS = 256;
  void init(Dev* d, int max_slices) {
    dev = d;
    // (parts <= 1024) x (<= 33 CGS2 dots) covers every multi-result reduction
    cap = std::max((size_t)std::max(64, blocks_per_sm()) * d->num_sms + 2 * (size_t)max_slices + 4096,
                   (size_t)4096 * 33);
    partial.alloc(cap, d->stream);
    counter.alloc(1 + (size_t)std::max(max_slices, 64), d->stream);
    counter.zero();
  }
  // blocks per slice: ~512 elements per block (2 per thread), <= blocks_per_sm blocks per
  // SM in total (several waves: enough independent loads in flight for HBM)
  static int blocks_per_sm() {
    static const int v = [] { const char* e = getenv("BBOT_RED_BLOCKS_PER_SM"); return e ? atoi(e) : 64; }();
    return v;
  }
  int parts_for(long long len, int nslices) const {
    long long p = (len + 511) / 512;
    long long cap_b = std::max(1LL, (long long)(blocks_per_sm() * dev->num_sms) / std::max(1, nslices));
    p = std::min(p, cap_b);
    p = std::min(p, 4096LL);
    return (int)std::max(1LL, p);
  }
  RedArgs args(int parts, int nslices, double* out, int k0 = 0) {
    if ((size_t)parts * nslices > cap) throw Error(BBOT_E_INTERNAL, "reduction workspace too small");
    return RedArgs{partial.p, counter.p, out, parts, k0};
  }
  template <class F, class Fin>
  void reduce(F f, long long len, int nslices, double* out, Fin fin) {
    int parts = parts_for(len, nslices);
    launch(*dev, k_slice_reduce<F, Fin>, dim3(parts, nslices), dim3(BS), 0, f, len, args(parts, nslices, out), fin);
  }
  template <class F>
  void slice_sum(F f, long long len, int nslices, double* out, bool take_sqrt = false) {
    if (take_sqrt) reduce(f, len, nslices, out, SqrtFin{out, nslices});
    else reduce(f, len, nslices, out, NoFin{});
  }
  // per-slice sums of the slices [k_lo, k_hi) of an ns_total-slice vector into out[k] (global
  // index); the partition into blocks depends on (len, ns_total) only, so a slab's results are
  // bitwise those of the full launch (time slabs)
  template <class F>
  void slice_sum_range(F f, long long len, int k_lo, int k_hi, int ns_total, double* out) {
    if (k_hi <= k_lo) return;
    int parts = parts_for(len, ns_total);
    launch(*dev, k_slice_reduce<F, NoFin>, dim3(parts, k_hi - k_lo), dim3(BS), 0, f, len,
           args(parts, k_hi - k_lo, out + k_lo, k_lo), NoFin{});
  }
  template <class F>
  void slice_min(F f, long long len, int nslices, double* out) {
    int parts = parts_for(len, nslices);
    args(parts, nslices, out);
    launch(*dev, k_slice_partial_min<F>, dim3(parts, nslices), dim3(BS), 0, f, len, parts, partial.p);
    launch(*dev, k_slice_final_min, dim3(nslices), dim3(BS), 0, (const double*)partial.p, parts, out);
  }
};

// ---------------------------------------------------------------------------
// Device-controlled loops.  The loop condition lives in device memory (`flag`)
// and is written by the body's last control kernel.  Under graph capture a loop
// becomes a conditional WHILE node whose handle the control kernel also sets
// (cudaGraphSetConditional), so a whole Krylov solve -- nested loops included --
// is one graph launch with no host round trip.  Eagerly (profiling, debugging,
// single calls) the same body runs on the stream and the host reads the flag.
struct LoopCtl {
  cudaGraphConditionalHandle h;
  int* flag;
  int graph;
  __device__ __forceinline__ void set(int v) const {
    *flag = v;
    if (graph) cudaGraphSetConditional(h, v ? 1u : 0u);
  }
};

__global__ void k_cond_from_flag(LoopCtl L);

cudaStream_t capture_stream(Dev& d, int depth);

template <class Body>
void dev_while(Dev& d, int* flag, Body&& body) {
  if (!d.capturing) {
    LoopCtl L{0, flag, 0};
    d.launches++;            // the graph's k_cond_from_flag, so eager and graph counts agree
    while (true) {
      int f = 0;
      BB_CUDA(cudaMemcpyAsync(&f, flag, sizeof(int), cudaMemcpyDeviceToHost, d.stream));
      BB_CUDA(cudaStreamSynchronize(d.stream));
      if (!f) break;
      body(L);
    }
    return;
  }
  cudaStreamCaptureStatus st;
  cudaGraph_t g;
  const cudaGraphNode_t* deps = nullptr;
  size_t nd = 0;
  BB_CUDA(cudaStreamGetCaptureInfo(d.stream, &st, nullptr, &g, &deps, &nd));
  cudaGraphConditionalHandle h;
  BB_CUDA(cudaGraphConditionalHandleCreate(&h, g, 0, 0));
  LoopCtl L{h, flag, 1};
  launch(d, k_cond_from_flag, dim3(1), dim3(1), 0, L);
  BB_CUDA(cudaStreamGetCaptureInfo(d.stream, &st, nullptr, &g, &deps, &nd));
  cudaGraphNodeParams p = {};
  p.type = cudaGraphNodeTypeConditional;
  p.conditional.handle = h;
  p.conditional.type = cudaGraphCondTypeWhile;
  p.conditional.size = 1;
  cudaGraphNode_t node;
  BB_CUDA(cudaGraphAddNode(&node, g, deps, nd, &p));
  cudaGraph_t body_g = p.conditional.phGraph_out[0];
  BB_CUDA(cudaStreamUpdateCaptureDependencies(d.stream, &node, 1, cudaStreamSetCaptureDependencies));
  cudaStream_t outer = d.stream;
  cudaStream_t inner = capture_stream(d, ++d.depth);
  BB_CUDA(cudaStreamBeginCaptureToGraph(inner, body_g, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  d.stream = inner;
  try {
    body(L);
  } catch (...) {
    d.stream = outer;
    d.depth--;
    cudaGraph_t junk;
    cudaStreamEndCapture(inner, &junk);
    throw;
  }
  d.stream = outer;
  d.depth--;
  BB_CUDA(cudaStreamEndCapture(inner, nullptr));
}

// Exclusive scan of int64 (len n) -> out (len n+1, out[n] = total).  In-place safe.
void exclusive_scan(Dev& d, const long long* in, long long* out, long long n, DBuf<long long>& ws);
void exclusive_scan_i32(Dev& d, const int* in, long long* out, long long n, DBuf<long long>& ws);

// address of a member of a device-resident struct (no dereference on the host)
template <class S, class T>
inline T* dev_field(S* base, T S::*m) {
  static const S probe{};
  size_t off = (size_t)(reinterpret_cast<const char*>(&(probe.*m)) - reinterpret_cast<const char*>(&probe));
  return reinterpret_cast<T*>(reinterpret_cast<char*>(base) + off);
}

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
