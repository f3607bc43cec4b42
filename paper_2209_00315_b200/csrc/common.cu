// common.cu -- deterministic reduction finalisers and the device-wide scan.
#include "common.cuh"
#include <map>
#include <mutex>

namespace bbot {

cudaMemPool_t device_pool() {
  static std::mutex mu;
  static std::map<int, cudaMemPool_t> pools;
  int dev = 0;
  BB_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  auto it = pools.find(dev);
  if (it != pools.end()) return it->second;
  cudaMemPoolProps props = {};
  props.allocType = cudaMemAllocationTypePinned;
  props.location.type = cudaMemLocationTypeDevice;
  props.location.id = dev;
  cudaMemPool_t pool;
  BB_CUDA(cudaMemPoolCreate(&pool, &props));
  unsigned long long thr = ~0ULL;
  BB_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
  pools[dev] = pool;
  return pool;
}

__global__ void k_cond_from_flag(LoopCtl L) { cudaGraphSetConditional(L.h, *L.flag ? 1u : 0u); }

cudaStream_t capture_stream(Dev& d, int depth) {
  while ((int)d.cap_streams.size() <= depth) {
    cudaStream_t st;
    BB_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    d.cap_streams.push_back(st);
  }
  return d.cap_streams[depth];
}

__global__ void k_slice_final_min(const double* partial, int parts, double* out) {
  int k = blockIdx.x;
  double acc = 1e300;
  for (int i = threadIdx.x; i < parts; i += blockDim.x) acc = fmin(acc, partial[(size_t)k * parts + i]);
  acc = block_min(acc);
  if (threadIdx.x == 0) out[k] = acc;
}

// ---------------------------------------------------------------- scan
// tile = 1024 threads x 4 items
constexpr int SCAN_BS = 1024;
constexpr int SCAN_ITEMS = 4;
constexpr long long SCAN_TILE = SCAN_BS * SCAN_ITEMS;

template <class T>
__global__ void k_scan_tile_sums(const T* in, long long n, long long* tile_sums) {
  long long base = (long long)blockIdx.x * SCAN_TILE;
  long long acc = 0;
  for (int j = 0; j < SCAN_ITEMS; j++) {
    long long i = base + (long long)j * SCAN_BS + threadIdx.x;
    if (i < n) acc += (long long)in[i];
  }
  // block reduce (integer)
  __shared__ long long sh[32];
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    acc = sh[threadIdx.x];
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
    if (threadIdx.x == 0) tile_sums[blockIdx.x] = acc;
  }
}

// single block: exclusive scan of tile sums in place (any length)
__global__ void k_scan_small(long long* a, long long n) {
  __shared__ long long sh[SCAN_BS];
  __shared__ long long carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (long long base = 0; base < n; base += SCAN_BS) {
    long long i = base + threadIdx.x;
    long long v = i < n ? a[i] : 0;
    sh[threadIdx.x] = v;
    __syncthreads();
    for (int o = 1; o < SCAN_BS; o <<= 1) {
      long long t = threadIdx.x >= o ? sh[threadIdx.x - o] : 0;
      __syncthreads();
      sh[threadIdx.x] += t;
      __syncthreads();
    }
    long long incl = sh[threadIdx.x];
    if (i < n) a[i] = carry + incl - v;
    __syncthreads();
    if (threadIdx.x == SCAN_BS - 1) carry += incl;
    __syncthreads();
  }
}

template <class T>
__global__ void k_scan_tiles(const T* in, long long* out, long long n, const long long* tile_off) {
  __shared__ long long sh[SCAN_BS];
  long long base = (long long)blockIdx.x * SCAN_TILE;
  // each thread owns SCAN_ITEMS consecutive items
  long long v[SCAN_ITEMS];
  long long loc = 0;
  for (int j = 0; j < SCAN_ITEMS; j++) {
    long long i = base + (long long)threadIdx.x * SCAN_ITEMS + j;
    v[j] = i < n ? (long long)in[i] : 0;
    loc += v[j];
  }
  sh[threadIdx.x] = loc;
  __syncthreads();
  for (int o = 1; o < SCAN_BS; o <<= 1) {
    long long t = threadIdx.x >= o ? sh[threadIdx.x - o] : 0;
    __syncthreads();
    sh[threadIdx.x] += t;
    __syncthreads();
  }
  long long run = tile_off[blockIdx.x] + sh[threadIdx.x] - loc;
  __syncthreads();
  for (int j = 0; j < SCAN_ITEMS; j++) {
    long long i = base + (long long)threadIdx.x * SCAN_ITEMS + j;
    if (i < n) out[i] = run;
    run += v[j];
  }
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x == SCAN_BS - 1) out[n] = run;
}

template <class T>
static void scan_impl(Dev& d, const T* in, long long* out, long long n, DBuf<long long>& ws) {
  long long tiles = (n + SCAN_TILE - 1) / SCAN_TILE;
  if (tiles < 1) tiles = 1;
  if ((long long)ws.n < tiles + 1) ws.alloc(tiles + 1, d.stream);
  launch(d, k_scan_tile_sums<T>, dim3((unsigned)tiles), dim3(SCAN_BS), 0, in, n, ws.p);
  launch(d, k_scan_small, dim3(1), dim3(SCAN_BS), 0, ws.p, tiles);
  launch(d, k_scan_tiles<T>, dim3((unsigned)tiles), dim3(SCAN_BS), 0, in, out, n, (const long long*)ws.p);
}

void exclusive_scan(Dev& d, const long long* in, long long* out, long long n, DBuf<long long>& ws) {
  scan_impl<long long>(d, in, out, n, ws);
}
void exclusive_scan_i32(Dev& d, const int* in, long long* out, long long n, DBuf<long long>& ws) {
  scan_impl<int>(d, in, out, n, ws);
}

}  // namespace bbot
