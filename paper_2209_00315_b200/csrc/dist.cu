// dist.cu -- multi-GPU time slabs, round-1 scope.
//
// One process per GPU; rank r owns a contiguous slab [a_r, b_r) of the K+1
// potential slices.  The per-slice A_k solves of every BB apply (4.20) -- the
// dominant cost (~60 % of a C4 solve) and independent per time slice (P:1469,
// P:1814 "well suited for parallelization") -- run on the owned slices only;
// the results are then exchanged with NCCL (one grouped broadcast per rank's
// slab over NVLink/NVSwitch, inside the apply).  Every other step (assembly, AMG
// setup, T-solve, J_P, FGMRES, recovery, update) is computed redundantly and
// deterministically on every rank, so all ranks hold the same iterate, bitwise
// equal to the single-GPU run (the A_k solves never couple slices, and the
// skipped slices are exact no-ops).  Halos for a full slab decomposition of J_P /
// T (memory per GPU / P) are the next step.
//
// NCCL is loaded with dlopen on first use (libnccl.so.2: the copy torch already
// loaded, or the system one), so libbbot.so has no link-time NCCL dependency.
#include "ops.cuh"
#include <dlfcn.h>
#include <nccl.h>
#include <cstring>

namespace bbot {

namespace {
struct NcclApi {
  bool ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  static bool tried = false;
  if (tried) return api;
  tried = true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return api;
  api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(h, "ncclGetUniqueId");
  api.CommInitRank = (decltype(api.CommInitRank))dlsym(h, "ncclCommInitRank");
  api.CommDestroy = (decltype(api.CommDestroy))dlsym(h, "ncclCommDestroy");
  api.Broadcast = (decltype(api.Broadcast))dlsym(h, "ncclBroadcast");
  api.GroupStart = (decltype(api.GroupStart))dlsym(h, "ncclGroupStart");
  api.GroupEnd = (decltype(api.GroupEnd))dlsym(h, "ncclGroupEnd");
  api.GetErrorString = (decltype(api.GetErrorString))dlsym(h, "ncclGetErrorString");
  api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.Broadcast && api.GroupStart &&
           api.GroupEnd && api.GetErrorString;
  return api;
}

void check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw Error(BBOT_E_NCCL, std::string(what) + ": " + (nccl().GetErrorString ? nccl().GetErrorString(r) : "?"));
}
}  // namespace

int slab_begin(int nslices, int rank, int nranks) {
  return (int)(((long long)rank * nslices) / nranks);
}

void nccl_unique_id(unsigned char out[128]) {
  NcclApi& a = nccl();
  BB_REQUIRE(a.ok, BBOT_E_NCCL, "libnccl.so.2 not loadable");
  ncclUniqueId id;
  check(a.GetUniqueId(&id), "ncclGetUniqueId");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  memcpy(out, &id, 128);
}

void set_dist(bbot_ctx* c, int rank, int nranks, const unsigned char* uid) {
  BB_REQUIRE(nranks >= 1 && rank >= 0 && rank < nranks, BBOT_E_INPUT, "bad rank / nranks");
  BB_REQUIRE(nranks <= c->g.K + 1, BBOT_E_INPUT, "more ranks than time slices");
  drop_dist(c);
  drop_solve_graph(c);
  c->rank = rank;
  c->nranks = nranks;
  c->own_begin = slab_begin(c->g.K + 1, rank, nranks);
  c->own_end = slab_begin(c->g.K + 1, rank + 1, nranks);
  c->virt = (uid == nullptr);
  if (nranks > 1 && uid) {
    NcclApi& a = nccl();
    BB_REQUIRE(a.ok, BBOT_E_NCCL, "libnccl.so.2 not loadable");
    ncclUniqueId id;
    memcpy(&id, uid, 128);
    ncclComm_t comm;
    check(a.CommInitRank(&comm, nranks, id, rank), "ncclCommInitRank");
    c->comm = (void*)comm;
  }
}

void drop_dist(bbot_ctx* c) {
  if (c->comm) {
    nccl().CommDestroy((ncclComm_t)c->comm);
    c->comm = nullptr;
  }
}

// every rank's slab of the K+1 potential slices (N values each) to every rank
void exchange_slabs(bbot_ctx* c, double* x) {
  if (c->nranks <= 1 || !c->comm) return;
  NcclApi& a = nccl();
  const long long N = c->g.N;
  check(a.GroupStart(), "ncclGroupStart");
  for (int q = 0; q < c->nranks; q++) {
    long long b0 = slab_begin(c->g.K + 1, q, c->nranks), b1 = slab_begin(c->g.K + 1, q + 1, c->nranks);
    double* p = x + b0 * N;
    check(a.Broadcast(p, p, (size_t)((b1 - b0) * N), ncclDouble, q, (ncclComm_t)c->comm, c->dev.stream),
          "ncclBroadcast");
  }
  check(a.GroupEnd(), "ncclGroupEnd");
}

}  // namespace bbot
