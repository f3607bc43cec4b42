// dist.cu -- multi-GPU time slabs: the exchange layer
// (comm.cuh) with its NCCL and virtual backends, and the rank setup of a context.
//
// NCCL is loaded with dlopen on first use (libnccl.so.2: the copy torch already loaded,
// or the system one), so libbbot.so has no link-time NCCL dependency.
#include "ops.cuh"
#include <chrono>
#include <condition_variable>
#include <dlfcn.h>
#include <map>
#include <mutex>
#include <nccl.h>
#include <cstring>

namespace bbot {

int slab_begin(int Kp1, int rank, int nranks) {
  if (rank >= nranks) return Kp1;
  const int K = Kp1 - 1;
  return time_block_size(K) * (int)(((long long)rank * time_blocks(K)) / nranks);
}

// ------------------------------------------------------------------ NCCL backend
namespace {
struct NcclApi {
  bool ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(h, "ncclGetUniqueId");
    api.CommInitRank = (decltype(api.CommInitRank))dlsym(h, "ncclCommInitRank");
    api.CommDestroy = (decltype(api.CommDestroy))dlsym(h, "ncclCommDestroy");
    api.Broadcast = (decltype(api.Broadcast))dlsym(h, "ncclBroadcast");
    api.Send = (decltype(api.Send))dlsym(h, "ncclSend");
    api.Recv = (decltype(api.Recv))dlsym(h, "ncclRecv");
    api.GroupStart = (decltype(api.GroupStart))dlsym(h, "ncclGroupStart");
    api.GroupEnd = (decltype(api.GroupEnd))dlsym(h, "ncclGroupEnd");
    api.GetErrorString = (decltype(api.GetErrorString))dlsym(h, "ncclGetErrorString");
    api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.Broadcast && api.Send && api.Recv &&
             api.GroupStart && api.GroupEnd && api.GetErrorString;
  });
  return api;
}

void check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw Error(BBOT_E_NCCL, std::string(what) + ": " + (nccl().GetErrorString ? nccl().GetErrorString(r) : "?"));
}

class NcclComm : public Comm {
 public:
  ncclComm_t comm = nullptr;
  ~NcclComm() override {
    if (comm) nccl().CommDestroy(comm);
  }
  // one grouped send/recv pair per neighbour (slice lo-1 <- left, slice hi <- right)
  void halo(Dev& d, const Layout& L, double* base) override {
    NcclApi& a = nccl();
    const int S = L.S();
    int lo, hi;
    owned(L, rank, lo, hi);
    check(a.GroupStart(), "ncclGroupStart");
    if (rank > 0 && lo > 0 && hi > lo) {
      check(a.Send(base + L.off[lo], (size_t)(L.off[lo + 1] - L.off[lo]), ncclDouble, rank - 1, comm, d.stream),
            "ncclSend");
      check(a.Recv(base + L.off[lo - 1], (size_t)(L.off[lo] - L.off[lo - 1]), ncclDouble, rank - 1, comm, d.stream),
            "ncclRecv");
    }
    int nlo, nhi;
    owned(L, rank + 1, nlo, nhi);
    if (rank + 1 < nranks && hi < S && nhi > nlo) {
      check(a.Send(base + L.off[hi - 1], (size_t)(L.off[hi] - L.off[hi - 1]), ncclDouble, rank + 1, comm, d.stream),
            "ncclSend");
      check(a.Recv(base + L.off[hi], (size_t)(L.off[hi + 1] - L.off[hi]), ncclDouble, rank + 1, comm, d.stream),
            "ncclRecv");
    }
    check(a.GroupEnd(), "ncclGroupEnd");
  }
  // in place: one broadcast per rank of its owned contiguous range
  void allgather(Dev& d, const Layout& L, double* base) override {
    NcclApi& a = nccl();
    check(a.GroupStart(), "ncclGroupStart");
    for (int q = 0; q < nranks; q++) {
      int lo, hi;
      owned(L, q, lo, hi);
      if (hi <= lo) continue;
      double* p = base + L.off[lo];
      check(a.Broadcast(p, p, (size_t)(L.off[hi] - L.off[lo]), ncclDouble, q, comm, d.stream), "ncclBroadcast");
    }
    check(a.GroupEnd(), "ncclGroupEnd");
  }
  void barrier(Dev&) override {}
};

// ------------------------------------------------------------------ virtual backend
// P contexts in one process (one host thread each), on one or several devices of the
// process: the posted buffer pointers are exchanged through a shared group; every phase
// is fenced by host barriers after the posting stream has been synchronised.
struct VirtGroup {
  int P;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  long long gen = 0;
  std::vector<double*> ptr;
  explicit VirtGroup(int p) : P(p), ptr(p, nullptr) {}
  // a rank that never arrives (ranks issuing different exchange sequences, or one rank
  // failing) surfaces as an error after a timeout instead of a hang
  void barrier() {
    static const int tmo = [] { const char* e = getenv("BBOT_VIRT_TIMEOUT_S"); return e ? atoi(e) : 120; }();
    std::unique_lock<std::mutex> lk(mu);
    long long g = gen;
    if (++arrived == P) {
      arrived = 0;
      gen++;
      cv.notify_all();
    } else if (!cv.wait_for(lk, std::chrono::seconds(tmo), [&] { return gen != g; })) {
      throw Error(BBOT_E_INTERNAL, "virtual ranks: exchange barrier timed out (ranks diverged or one failed)");
    }
  }
};

std::mutex g_reg_mu;
std::map<long long, std::weak_ptr<VirtGroup>> g_reg;

class VirtComm : public Comm {
 public:
  std::shared_ptr<VirtGroup> grp;
  long long nops = 0;
  void trace(const char* what, const Layout& L) {
    static const bool on = getenv("BBOT_COMM_TRACE") != nullptr;
    if (on) fprintf(stderr, "[comm r%d #%lld] %s S=%d len=%lld\n", rank, nops, what, L.S(), L.off.back());
    nops++;
  }
  void post(Dev& d, double* base) {
    BB_CUDA(cudaStreamSynchronize(d.stream));    // my data is complete before anyone reads it
    grp->ptr[rank] = base;
    grp->barrier();
  }
  void done(Dev& d) {
    BB_CUDA(cudaStreamSynchronize(d.stream));    // my copies are complete before anyone moves on
    grp->barrier();
  }
  void copy(Dev& d, double* dst, const double* src, long long n) {
    if (n > 0) BB_CUDA(cudaMemcpyAsync(dst, src, n * sizeof(double), cudaMemcpyDeviceToDevice, d.stream));
  }
  void halo(Dev& d, const Layout& L, double* base) override {
    trace("halo", L);
    post(d, base);
    const int S = L.S();
    int lo, hi;
    owned(L, rank, lo, hi);
    if (rank > 0 && lo > 0 && hi > lo) copy(d, base + L.off[lo - 1], grp->ptr[rank - 1] + L.off[lo - 1], L.off[lo] - L.off[lo - 1]);
    int nlo, nhi;
    owned(L, rank + 1, nlo, nhi);
    if (rank + 1 < nranks && hi < S && nhi > nlo)
      copy(d, base + L.off[hi], grp->ptr[rank + 1] + L.off[hi], L.off[hi + 1] - L.off[hi]);
    done(d);
  }
  void allgather(Dev& d, const Layout& L, double* base) override {
    trace("allgather", L);
    post(d, base);
    for (int q = 0; q < nranks; q++) {
      if (q == rank) continue;
      int lo, hi;
      owned(L, q, lo, hi);
      if (hi > lo) copy(d, base + L.off[lo], grp->ptr[q] + L.off[lo], L.off[hi] - L.off[lo]);
    }
    done(d);
  }
  void barrier(Dev& d) override {
    BB_CUDA(cudaStreamSynchronize(d.stream));
    grp->barrier();
  }
};
}  // namespace

std::unique_ptr<Comm> make_nccl_comm(int rank, int nranks, int Kp1, const unsigned char* uid) {
  NcclApi& a = nccl();
  BB_REQUIRE(a.ok, BBOT_E_NCCL, "libnccl.so.2 not loadable");
  std::unique_ptr<NcclComm> c(new NcclComm());
  c->rank = rank;
  c->nranks = nranks;
  c->Kp1 = Kp1;
  ncclUniqueId id;
  memcpy(&id, uid, 128);
  check(a.CommInitRank(&c->comm, nranks, id, rank), "ncclCommInitRank");
  return c;
}

std::unique_ptr<Comm> make_virtual_comm(int rank, int nranks, int Kp1, long long group) {
  std::unique_ptr<VirtComm> c(new VirtComm());
  c->rank = rank;
  c->nranks = nranks;
  c->Kp1 = Kp1;
  std::lock_guard<std::mutex> lk(g_reg_mu);
  auto sp = g_reg[group].lock();
  if (!sp || sp->P != nranks) {
    sp = std::make_shared<VirtGroup>(nranks);
    g_reg[group] = sp;
  }
  c->grp = sp;
  return c;
}

void nccl_unique_id(unsigned char out[128]) {
  NcclApi& a = nccl();
  BB_REQUIRE(a.ok, BBOT_E_NCCL, "libnccl.so.2 not loadable");
  ncclUniqueId id;
  check(a.GetUniqueId(&id), "ncclGetUniqueId");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  memcpy(out, &id, 128);
}

// uid != NULL: NCCL (one process per GPU); uid == NULL: virtual ranks of group `group`
void set_dist(bbot_ctx* c, int rank, int nranks, const unsigned char* uid, long long group) {
  BB_REQUIRE(nranks >= 1 && rank >= 0 && rank < nranks, BBOT_E_INPUT, "bad rank / nranks");
  BB_REQUIRE(nranks == 1 || nranks <= time_blocks(c->g.K), BBOT_E_INPUT,
             "time slabs: every rank needs >= 1 AMG(T) time block (P <= nb, bbot_time_blocks)");
  drop_dist(c);
  drop_solve_graph(c);
  c->rank = rank;
  c->nranks = nranks;
  c->own_begin = slab_begin(c->g.K + 1, rank, nranks);
  c->own_end = slab_begin(c->g.K + 1, rank + 1, nranks);
  if (nranks > 1) {
    c->comm = uid ? make_nccl_comm(rank, nranks, c->g.K + 1, uid)
                  : make_virtual_comm(rank, nranks, c->g.K + 1, group);
  }
}

void drop_dist(bbot_ctx* c) {
  c->comm.reset();
  c->rank = 0;
  c->nranks = 1;
  c->own_begin = 0;
  c->own_end = 1 << 30;
}

}  // namespace bbot
