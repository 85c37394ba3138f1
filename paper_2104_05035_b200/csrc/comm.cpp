// comm.cpp — run-time-loaded NCCL (see comm.h).  Types come from nccl.h; the
// functions are resolved with dlsym from the libnccl.so.2 already mapped into
// the process by torch (RTLD_NOLOAD first), else from the loader path.
#include "comm.h"

#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <string>

#include "error.h"

namespace rn {

struct NcclComm {
  ncclComm_t c;
  int size;
};

namespace {
struct Api {
  void *h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId *);
  ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int);
  ncclResult_t (*CommSplit)(ncclComm_t, int, int, ncclComm_t *, ncclConfig_t *);
  ncclResult_t (*CommDestroy)(ncclComm_t);
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
  nccl_load();
  ncclUniqueId id;
  memcpy(id.internal, idb, 128);
  NcclComm *c = new NcclComm{nullptr, nranks};
  check(g_api.CommInitRank(&c->c, nranks, id, rank), "ncclCommInitRank");
  return c;
}

NcclComm *nccl_split(NcclComm *parent, int color, int key) {
  NcclComm *c = new NcclComm{nullptr, 0};
  check(g_api.CommSplit(parent->c, color, key, &c->c, nullptr), "ncclCommSplit");
  // size = number of ranks with the same color; computed by the caller
  return c;
}

void nccl_destroy(NcclComm *c) {
  if (!c) return;
  if (c->c && g_api.CommDestroy) g_api.CommDestroy(c->c);
  delete c;
}

int nccl_size(NcclComm *c) { return c->size; }

void nccl_allreduce_sum_f32(NcclComm *c, float *buf, size_t count, cudaStream_t st) {
  check(g_api.AllReduce(buf, buf, count, ncclFloat32, ncclSum, c->c, st), "ncclAllReduce");
}

void nccl_send_bytes(NcclComm *c, const void *buf, size_t bytes, int peer, cudaStream_t st) {
  check(g_api.Send(buf, bytes, ncclUint8, peer, c->c, st), "ncclSend");
}

void nccl_recv_bytes(NcclComm *c, void *buf, size_t bytes, int peer, cudaStream_t st) {
  check(g_api.Recv(buf, bytes, ncclUint8, peer, c->c, st), "ncclRecv");
}

void nccl_bcast_f32(NcclComm *c, float *buf, size_t count, int root, cudaStream_t st) {
  check(g_api.Broadcast(buf, buf, count, ncclFloat32, root, c->c, st), "ncclBroadcast");
}

}  // namespace rn
