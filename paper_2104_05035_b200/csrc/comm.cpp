// comm.cpp — run-time-loaded NCCL (see comm.h).  Types come from nccl.h; the
// functions are resolved with dlsym from the libnccl.so.2 already mapped into
// the process by torch (RTLD_NOLOAD first), else from the loader path.
#include "comm.h"

#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <condition_variable>
#include <cstring>
#include <deque>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "error.h"

namespace rn {

// ---------------------------------------------------------------------------
// In-process transport (test vehicle for the multi-rank executor on ONE GPU):
// ranks are plans of this process, each driven by its own host thread, sharing
// one device.  send/recv = a rendezvous in host memory + a device-to-device
// copy on the receiver's stream (the sender's stream then waits for that copy:
// NCCL's completion semantics); all-reduce = every member's buffer summed in
// rank order into member 0's buffer and copied back; broadcast = copies from
// the root.  Selected by an id whose first 8 bytes are "RNLOCAL" + NUL.
// ---------------------------------------------------------------------------
struct LocalMsg {
  const void *ptr = nullptr;
  size_t bytes = 0;
  cudaEvent_t ready = nullptr, done = nullptr;
  bool copied = false;
};

struct LocalGroup {
  int size = 0;
  std::mutex mu;
  std::condition_variable cv;
  std::map<std::pair<int, int>, std::deque<std::shared_ptr<LocalMsg>>> q;  // (src, dst)
  // collectives (all-reduce / broadcast): one round at a time
  long gen = 0;
  int arrived = 0;
  std::vector<void *> bufs;
  std::vector<cudaEvent_t> evs;
  std::map<long, cudaEvent_t> done;  // round -> completion event
  // splits: round -> (rank -> (color, key))
  long split_gen = 0;
  int split_arrived = 0;
  std::map<long, std::vector<std::pair<int, int>>> split_ck;  // round -> rank -> (color, key)
  std::map<std::pair<long, int>, std::shared_ptr<LocalGroup>> subs;  // (round, color) -> subgroup
  std::vector<cudaEvent_t> owned;                                     // destroyed with the group
  ~LocalGroup() {
    for (auto e : owned) cudaEventDestroy(e);
  }
};

namespace {
std::mutex g_local_mu;
std::map<std::string, std::shared_ptr<LocalGroup>> g_local;  // id -> world group

bool is_local_id(const uint8_t id[128]) { return memcmp(id, "RNLOCAL", 8) == 0; }

cudaEvent_t new_event(LocalGroup &g) {  // caller holds g.mu
  cudaEvent_t e = nullptr;
  CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  g.owned.push_back(e);
  return e;
}

__global__ void add_f32_k(float *__restrict__ dst, const float *__restrict__ src, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    dst[i] += src[i];
}
}  // namespace

struct NcclComm {
  ncclComm_t c;
  int size;
  std::shared_ptr<LocalGroup> lg;  // in-process transport when set
  int lrank = 0;
};

namespace {
struct Api {
  void *h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId *);
  ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int);
  ncclResult_t (*CommSplit)(ncclComm_t, int, int, ncclComm_t *, ncclConfig_t *);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  ncclResult_t (*CommCount)(const ncclComm_t, int *);
  ncclResult_t (*GroupStart)();
  ncclResult_t (*GroupEnd)();
  ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t);
  ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*Broadcast)(const void *, void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  const char *(*GetErrorString)(ncclResult_t);
};
Api g_api;
std::mutex g_mu;

template <typename F>
void sym(F &f, const char *name) {
  f = reinterpret_cast<F>(dlsym(g_api.h, name));
  if (!f) throw Error(RN_ERR_NCCL, std::string("libnccl: missing symbol ") + name);
}

void check(ncclResult_t r, const char *what) {
  if (r != ncclSuccess) {
    std::string m = std::string(what) + " failed: ";
    m += g_api.GetErrorString ? g_api.GetErrorString(r) : "error";
    throw Error(RN_ERR_NCCL, m);
  }
}
}  // namespace

void nccl_load() {
  std::lock_guard<std::mutex> lk(g_mu);
  if (g_api.h) return;
  void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) throw Error(RN_ERR_NCCL, std::string("cannot load libnccl.so.2: ") + dlerror());
  g_api.h = h;
  sym(g_api.GetUniqueId, "ncclGetUniqueId");
  sym(g_api.CommInitRank, "ncclCommInitRank");
  sym(g_api.CommSplit, "ncclCommSplit");
  sym(g_api.CommDestroy, "ncclCommDestroy");
  sym(g_api.CommCount, "ncclCommCount");
  sym(g_api.GroupStart, "ncclGroupStart");
  sym(g_api.GroupEnd, "ncclGroupEnd");
  sym(g_api.AllReduce, "ncclAllReduce");
  sym(g_api.Send, "ncclSend");
  sym(g_api.Recv, "ncclRecv");
  sym(g_api.Broadcast, "ncclBroadcast");
  sym(g_api.GetErrorString, "ncclGetErrorString");
}

void nccl_unique_id(uint8_t out[128]) {
  nccl_load();
  ncclUniqueId id;
  check(g_api.GetUniqueId(&id), "ncclGetUniqueId");
  memcpy(out, id.internal, 128);
}

NcclComm *nccl_init(const uint8_t idb[128], int nranks, int rank) {
  if (is_local_id(idb)) {
    std::lock_guard<std::mutex> lk(g_local_mu);
    auto &g = g_local[std::string((const char *)idb, 128)];
    if (!g) {
      g = std::make_shared<LocalGroup>();
      g->size = nranks;
    }
    if (g->size != nranks) throw Error(RN_ERR_ARG, "local transport: world size mismatch");
    NcclComm *c = new NcclComm{nullptr, nranks, g, rank};
    return c;
  }
  nccl_load();
  ncclUniqueId id;
  memcpy(id.internal, idb, 128);
  NcclComm *c = new NcclComm{nullptr, nranks};
  check(g_api.CommInitRank(&c->c, nranks, id, rank), "ncclCommInitRank");
  return c;
}

NcclComm *nccl_split(NcclComm *parent, int color, int key) {
  if (parent->lg) {
    LocalGroup &g = *parent->lg;
    std::unique_lock<std::mutex> lk(g.mu);
    const long round = g.split_gen;
    auto &ck = g.split_ck[round];
    if (ck.empty()) ck.assign(g.size, {0, 0});
    ck[parent->lrank] = {color, key};
    if (++g.split_arrived == g.size) {
      // every member posted: build the subgroups of this round
      std::map<int, std::vector<std::tuple<int, int, int>>> by_color;  // color -> (key, rank)
      for (int r = 0; r < g.size; ++r) by_color[ck[r].first].push_back({ck[r].second, r, 0});
      for (auto &kv : by_color) {
        auto sub = std::make_shared<LocalGroup>();
        sub->size = (int)kv.second.size();
        g.subs[{round, kv.first}] = sub;
      }
      g.split_arrived = 0;
      ++g.split_gen;
      g.cv.notify_all();
    } else {
      g.cv.wait(lk, [&] { return g.split_gen != round; });
    }
    // my rank within the color: order by (key, parent rank)
    std::vector<std::pair<int, int>> mem;
    const auto &ckr = g.split_ck[round];
    for (int r = 0; r < g.size; ++r)
      if (ckr[r].first == color) mem.push_back({ckr[r].second, r});
    std::sort(mem.begin(), mem.end());
    int lr = 0;
    for (size_t i = 0; i < mem.size(); ++i)
      if (mem[i].second == parent->lrank) lr = (int)i;
    auto sub = g.subs[{round, color}];
    return new NcclComm{nullptr, sub->size, sub, lr};
  }
  NcclComm *c = new NcclComm{nullptr, 0};
  check(g_api.CommSplit(parent->c, color, key, &c->c, nullptr), "ncclCommSplit");
  int n = 0;
  if (g_api.CommCount) check(g_api.CommCount(c->c, &n), "ncclCommCount");
  c->size = n;
  return c;
}

void nccl_destroy(NcclComm *c) {
  if (!c) return;
  if (c->c && g_api.CommDestroy) g_api.CommDestroy(c->c);
  if (c->lg && c->size >= 0) {
    // drop the world group from the registry once its last member is gone
    std::lock_guard<std::mutex> lk(g_local_mu);
    for (auto it = g_local.begin(); it != g_local.end(); ++it)
      if (it->second == c->lg && c->lg.use_count() <= 2) {
        g_local.erase(it);
        break;
      }
  }
  delete c;
}

int nccl_size(NcclComm *c) { return c->size; }
bool nccl_is_local(NcclComm *c) { return c && c->lg; }

void nccl_group_start(NcclComm *c) {
  if (c && !c->lg) check(g_api.GroupStart(), "ncclGroupStart");
}
void nccl_group_end(NcclComm *c) {
  if (c && !c->lg) check(g_api.GroupEnd(), "ncclGroupEnd");
}

// all-reduce (sum) / broadcast over the in-process transport: the last member to
// arrive enqueues the reduction (rank order, into member 0's buffer) and the
// copies back on its own stream; every member's stream then waits for it
static void local_collective(NcclComm *c, void *buf, size_t bytes, int root, bool reduce, cudaStream_t st) {
  LocalGroup &g = *c->lg;
  std::unique_lock<std::mutex> lk(g.mu);
  const long round = g.gen;
  if (g.bufs.empty()) {
    g.bufs.assign(g.size, nullptr);
    g.evs.assign(g.size, nullptr);
  }
  cudaEvent_t ready = new_event(g);
  CUDA_CHECK(cudaEventRecord(ready, st));
  g.bufs[c->lrank] = buf;
  g.evs[c->lrank] = ready;
  if (++g.arrived == g.size) {
    for (int r = 0; r < g.size; ++r) CUDA_CHECK(cudaStreamWaitEvent(st, g.evs[r], 0));
    const int src = reduce ? 0 : root;
    if (reduce) {
      const size_t n = bytes / 4;
      const unsigned blocks = (unsigned)std::min<size_t>((n + 255) / 256, 148 * 8);
      for (int r = 1; r < g.size; ++r) {
        add_f32_k<<<blocks ? blocks : 1, 256, 0, st>>>((float *)g.bufs[0], (const float *)g.bufs[r], n);
        CUDA_CHECK(cudaGetLastError());
      }
    }
    for (int r = 0; r < g.size; ++r)
      if (r != src) CUDA_CHECK(cudaMemcpyAsync(g.bufs[r], g.bufs[src], bytes, cudaMemcpyDeviceToDevice, st));
    cudaEvent_t done = new_event(g);
    CUDA_CHECK(cudaEventRecord(done, st));
    g.done[round] = done;
    g.arrived = 0;
    ++g.gen;
    g.cv.notify_all();
  } else {
    g.cv.wait(lk, [&] { return g.gen != round; });
    CUDA_CHECK(cudaStreamWaitEvent(st, g.done[round], 0));
  }
}

void nccl_allreduce_sum_f32(NcclComm *c, float *buf, size_t count, cudaStream_t st) {
  if (c->lg) {
    if (c->size > 1) local_collective(c, buf, count * sizeof(float), 0, true, st);
    return;
  }
  check(g_api.AllReduce(buf, buf, count, ncclFloat32, ncclSum, c->c, st), "ncclAllReduce");
}

void nccl_send_bytes(NcclComm *c, const void *buf, size_t bytes, int peer, cudaStream_t st) {
  if (c->lg) {
    LocalGroup &g = *c->lg;
    std::unique_lock<std::mutex> lk(g.mu);
    auto m = std::make_shared<LocalMsg>();
    m->ptr = buf;
    m->bytes = bytes;
    m->ready = new_event(g);
    CUDA_CHECK(cudaEventRecord(m->ready, st));
    g.q[{c->lrank, peer}].push_back(m);
    g.cv.notify_all();
    g.cv.wait(lk, [&] { return m->copied; });  // rendezvous: the receiver enqueued its copy
    CUDA_CHECK(cudaStreamWaitEvent(st, m->done, 0));
    return;
  }
  check(g_api.Send(buf, bytes, ncclUint8, peer, c->c, st), "ncclSend");
}

void nccl_recv_bytes(NcclComm *c, void *buf, size_t bytes, int peer, cudaStream_t st) {
  if (c->lg) {
    LocalGroup &g = *c->lg;
    std::unique_lock<std::mutex> lk(g.mu);
    auto &dq = g.q[{peer, c->lrank}];
    g.cv.wait(lk, [&] { return !dq.empty(); });
    auto m = dq.front();
    dq.pop_front();
    if (m->bytes != bytes) throw Error(RN_ERR_NCCL, "local transport: send/recv size mismatch");
    CUDA_CHECK(cudaStreamWaitEvent(st, m->ready, 0));
    CUDA_CHECK(cudaMemcpyAsync(buf, m->ptr, bytes, cudaMemcpyDeviceToDevice, st));
    m->done = new_event(g);
    CUDA_CHECK(cudaEventRecord(m->done, st));
    m->copied = true;
    g.cv.notify_all();
    return;
  }
  check(g_api.Recv(buf, bytes, ncclUint8, peer, c->c, st), "ncclRecv");
}

void nccl_bcast_f32(NcclComm *c, float *buf, size_t count, int root, cudaStream_t st) {
  if (c->lg) {
    if (c->size > 1) local_collective(c, buf, count * sizeof(float), root, false, st);
    return;
  }
  check(g_api.Broadcast(buf, buf, count, ncclFloat32, root, c->c, st), "ncclBroadcast");
}

}  // namespace rn
