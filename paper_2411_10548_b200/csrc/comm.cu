// Data-parallel collectives of the train step (SURVEY.md §8b "Comms": comm_init(ncclUniqueId, rank, world),
// allreduce_bucket(ptr, count, dtype, stream)), NCCL over NVLink 5 / NVSwitch.
//
// NCCL is resolved at run time (dlopen "libnccl.so.2", preferring the copy the process already loaded -- the
// one torch.distributed uses -- so there is a single NCCL in the process); the library itself has no link-time
// NCCL dependency.  One communicator per rank, owned by the caller through an opaque handle (the only mutable
// state the C ABI keeps).  Every collective is enqueued on the caller's stream, so it can be captured in a CUDA
// graph together with the backward kernels that produce the gradients.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>

#include "common.cuh"

namespace esm {
namespace {

struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*ReduceScatter)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                                cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GetVersion)(int*) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  bool ok = false;
};

NcclApi& api() {
  static NcclApi a;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // the NCCL already in the process (torch's)
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    a.GetUniqueId = (decltype(a.GetUniqueId))dlsym(h, "ncclGetUniqueId");
    a.CommInitRank = (decltype(a.CommInitRank))dlsym(h, "ncclCommInitRank");
    a.CommDestroy = (decltype(a.CommDestroy))dlsym(h, "ncclCommDestroy");
    a.AllReduce = (decltype(a.AllReduce))dlsym(h, "ncclAllReduce");
    a.ReduceScatter = (decltype(a.ReduceScatter))dlsym(h, "ncclReduceScatter");
    a.AllGather = (decltype(a.AllGather))dlsym(h, "ncclAllGather");
    a.GetVersion = (decltype(a.GetVersion))dlsym(h, "ncclGetVersion");
    a.GetErrorString = (decltype(a.GetErrorString))dlsym(h, "ncclGetErrorString");
    a.ok = a.GetUniqueId && a.CommInitRank && a.CommDestroy && a.AllReduce && a.ReduceScatter && a.AllGather &&
           a.GetVersion && a.GetErrorString;
  });
  return a;
}

int nccl_rc(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return 0;
  set_last_error("%s: %s", what, api().GetErrorString ? api().GetErrorString(r) : "nccl error");
  return ESM_ENCCL_BASE + (int)r;
}

bool nccl_type(int dtype, ncclDataType_t& t) {
  switch (dtype) {
    case ESM_F32: t = ncclFloat32; return true;
    case ESM_BF16: t = ncclBfloat16; return true;
    case ESM_I32: t = ncclInt32; return true;
    default: return false;
  }
}

}  // namespace
}  // namespace esm

using namespace esm;

struct esm_comm {
  ncclComm_t comm;
  int rank, world;
};

extern "C" {

int esm_comm_version(void) {
  if (!api().ok) return 0;
  int v = 0;
  api().GetVersion(&v);
  return v;
}

int esm_comm_unique_id(uint8_t* out) {
  ESM_CHECK_ARG(out != nullptr, "esm_comm_unique_id: null");
  if (!api().ok) {
    set_last_error("libnccl.so.2 not loadable");
    return ESM_ENOTSUP;
  }
  ncclUniqueId id;
  const int rc = nccl_rc(api().GetUniqueId(&id), "ncclGetUniqueId");
  if (rc) return rc;
  static_assert(sizeof(id.internal) == ESM_COMM_ID_BYTES, "NCCL unique id size");
  memcpy(out, id.internal, ESM_COMM_ID_BYTES);
  return 0;
}

int esm_comm_init(const uint8_t* id, int rank, int world, esm_comm_t* out) {
  ESM_CHECK_ARG(id && out && world > 0 && rank >= 0 && rank < world, "esm_comm_init: bad args");
  if (!api().ok) {
    set_last_error("libnccl.so.2 not loadable");
    return ESM_ENOTSUP;
  }
  ncclUniqueId uid;
  memcpy(uid.internal, id, ESM_COMM_ID_BYTES);
  ncclComm_t c;
  const int rc = nccl_rc(api().CommInitRank(&c, world, uid, rank), "ncclCommInitRank");
  if (rc) return rc;
  *out = new esm_comm{c, rank, world};
  return 0;
}

int esm_comm_destroy(esm_comm_t c) {
  if (!c) return 0;
  const int rc = api().ok ? nccl_rc(api().CommDestroy(c->comm), "ncclCommDestroy") : 0;
  delete c;
  return rc;
}

int esm_comm_allreduce(esm_comm_t c, void* buf, int64_t count, int dtype, esm_stream_t stream) {
  ncclDataType_t t;
  ESM_CHECK_ARG(c && buf && count >= 0 && nccl_type(dtype, t), "esm_comm_allreduce: bad args");
  return nccl_rc(api().AllReduce(buf, buf, (size_t)count, t, ncclSum, c->comm, (cudaStream_t)stream),
                 "ncclAllReduce");
}

int esm_comm_reduce_scatter(esm_comm_t c, void* buf, int64_t count, int dtype, esm_stream_t stream) {
  ncclDataType_t t;
  ESM_CHECK_ARG(c && buf && count >= 0 && count % c->world == 0 && nccl_type(dtype, t),
                "esm_comm_reduce_scatter: count must be a multiple of the world size");
  const size_t per = (size_t)count / c->world;
  const size_t esz = dtype == ESM_BF16 ? 2 : 4;
  void* recv = static_cast<char*>(buf) + (size_t)c->rank * per * esz;  // in place: this rank's slice
  return nccl_rc(api().ReduceScatter(buf, recv, per, t, ncclSum, c->comm, (cudaStream_t)stream),
                 "ncclReduceScatter");
}

int esm_comm_allgather(esm_comm_t c, void* buf, int64_t count, int dtype, esm_stream_t stream) {
  ncclDataType_t t;
  ESM_CHECK_ARG(c && buf && count >= 0 && count % c->world == 0 && nccl_type(dtype, t),
                "esm_comm_allgather: count must be a multiple of the world size");
  const size_t per = (size_t)count / c->world;
  const size_t esz = dtype == ESM_BF16 ? 2 : 4;
  const void* send = static_cast<const char*>(buf) + (size_t)c->rank * per * esz;  // in place
  return nccl_rc(api().AllGather(send, buf, per, t, c->comm, (cudaStream_t)stream), "ncclAllGather");
}

}  // extern "C"
