// comm.h — NCCL over NVLink/NVSwitch for the two exchange steps of the hybrid
// scheme: partition-boundary send/recv (activation a^t to
// partition i+1, gradient g^t to partition i-1) and the data-parallel ring
// all-reduce of gradients (§3.2, Eqs. 9-11).  libnccl.so.2 is loaded at
// run time (the copy torch already loaded, so one NCCL per process).
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace rn {

struct NcclComm;  // opaque

// Load libnccl (idempotent).  Throws Error(RN_ERR_NCCL) on failure.
void nccl_load();
void nccl_unique_id(uint8_t out[128]);
NcclComm *nccl_init(const uint8_t id[128], int nranks, int rank);
NcclComm *nccl_split(NcclComm *parent, int color, int key);
void nccl_destroy(NcclComm *c);
int nccl_size(NcclComm *c);
// in-process transport (ranks = plans of this process on one device; id prefix "RNLOCAL\0")
bool nccl_is_local(NcclComm *c);
// ncclGroupStart/End (no-ops on the in-process transport)
void nccl_group_start(NcclComm *c);
void nccl_group_end(NcclComm *c);
void nccl_allreduce_sum_f32(NcclComm *c, float *buf, size_t count, cudaStream_t st);
void nccl_send_bytes(NcclComm *c, const void *buf, size_t bytes, int peer, cudaStream_t st);
void nccl_recv_bytes(NcclComm *c, void *buf, size_t bytes, int peer, cudaStream_t st);
void nccl_bcast_f32(NcclComm *c, float *buf, size_t count, int root, cudaStream_t st);

}  // namespace rn
