// Multi-GPU scale-gradient exchange through NCCL.
//
// The only data exchanged by the scale-only QAT step is the per-channel
// scale-gradient vector (1,494 fp64 per frame set). Frames are sharded over
// GPUs; each rank's backward leaves one gradient row per local frame, and
//   qfb_gather_fold_scale_grads: ncclAllGather of the rows + a row-order
//     fold (qfb_fold_rows) -> bit-identical to the single-GPU trainer's
//     frame-order accumulation (frontend.hpp:222-228, distill.hpp:249-250)
//     at every GPU count;
//   qfb_allreduce_scale_grads: ncclAllReduce(sum), the cheaper exchange
//     whose bits depend on the GPU count (NCCL's reduction order).
// NCCL is loaded with dlopen (the copy already in the process, e.g. torch's,
// else libnccl.so.2 from the loader path) so libqfb has no link-time NCCL
// dependency; a missing NCCL is QFB_ERR_NCCL at the call, never a fallback.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <string>

#include "../../include/qfb.h"
#include "qfb_kernels.h"

namespace {

struct Nccl {
  void* h = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*init_all)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*get_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*count)(const ncclComm_t, int*) = nullptr;
  const char* (*err_str)(ncclResult_t) = nullptr;
  std::string why;
};

const Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* env = getenv("QFB_NCCL_LIB");
    const char* names[] = {env, "libnccl.so.2", "libnccl.so"};
    for (const char* nm : names) {
      if (!nm) continue;
      n.h = dlopen(nm, RTLD_NOW | RTLD_NOLOAD);  // prefer the copy already loaded (torch's)
      if (!n.h) n.h = dlopen(nm, RTLD_NOW | RTLD_LOCAL);
      if (n.h) break;
    }
    if (!n.h) {
      n.why = "NCCL not found (libnccl.so.2; set QFB_NCCL_LIB)";
      return;
    }
    n.all_gather = reinterpret_cast<decltype(n.all_gather)>(dlsym(n.h, "ncclAllGather"));
    n.all_reduce = reinterpret_cast<decltype(n.all_reduce)>(dlsym(n.h, "ncclAllReduce"));
    n.init_all = reinterpret_cast<decltype(n.init_all)>(dlsym(n.h, "ncclCommInitAll"));
    n.destroy = reinterpret_cast<decltype(n.destroy)>(dlsym(n.h, "ncclCommDestroy"));
    n.get_id = reinterpret_cast<decltype(n.get_id)>(dlsym(n.h, "ncclGetUniqueId"));
    n.init_rank = reinterpret_cast<decltype(n.init_rank)>(dlsym(n.h, "ncclCommInitRank"));
    n.count = reinterpret_cast<decltype(n.count)>(dlsym(n.h, "ncclCommCount"));
    n.err_str = reinterpret_cast<decltype(n.err_str)>(dlsym(n.h, "ncclGetErrorString"));
    if (!n.all_gather || !n.all_reduce || !n.init_all || !n.destroy || !n.count || !n.err_str || !n.get_id ||
        !n.init_rank)
      n.why = "NCCL library lacks a required symbol";
  });
  return n;
}

qfb_status nccl_ready() {
  const Nccl& n = nccl();
  if (!n.why.empty()) return qfb::set_error(QFB_ERR_NCCL, n.why.c_str());
  return QFB_OK;
}

qfb_status nccl_fail(ncclResult_t r, const char* what) {
  std::string m = std::string(what) + ": " + nccl().err_str(r);
  return qfb::set_error(QFB_ERR_NCCL, m.c_str());
}

}  // namespace

extern "C" {

qfb_status qfb_nccl_available(void) { return nccl_ready(); }

qfb_status qfb_nccl_comm_init_all(int ndev, const int* devices, void** comms) {
  if (ndev < 1 || !comms) return qfb::set_error(QFB_ERR_VALUE, "nccl_comm_init_all: bad arguments");
  if (qfb_status s = nccl_ready()) return s;
  ncclResult_t r = nccl().init_all(reinterpret_cast<ncclComm_t*>(comms), ndev, devices);
  if (r != ncclSuccess) return nccl_fail(r, "ncclCommInitAll");
  return QFB_OK;
}

static_assert(sizeof(ncclUniqueId) == QFB_NCCL_UNIQUE_ID_BYTES, "ncclUniqueId size");

qfb_status qfb_nccl_get_unique_id(void* id) {
  if (!id) return qfb::set_error(QFB_ERR_VALUE, "nccl_get_unique_id: null buffer");
  if (qfb_status s = nccl_ready()) return s;
  ncclResult_t r = nccl().get_id(static_cast<ncclUniqueId*>(id));
  if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
  return QFB_OK;
}

qfb_status qfb_nccl_comm_init_rank(void** comm, int nranks, const void* id, int rank, int device) {
  if (!comm || !id || nranks < 1 || rank < 0 || rank >= nranks)
    return qfb::set_error(QFB_ERR_VALUE, "nccl_comm_init_rank: bad arguments");
  if (qfb_status s = nccl_ready()) return s;
  int prev = -1;
  cudaGetDevice(&prev);
  if (cudaSetDevice(device) != cudaSuccess) return qfb::set_error(QFB_ERR_CUDA, "nccl_comm_init_rank: bad device");
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof uid);
  ncclResult_t r = nccl().init_rank(reinterpret_cast<ncclComm_t*>(comm), nranks, uid, rank);
  if (prev >= 0) cudaSetDevice(prev);
  if (r != ncclSuccess) return nccl_fail(r, "ncclCommInitRank");
  return QFB_OK;
}

qfb_status qfb_nccl_comm_destroy(void* comm) {
  if (!comm) return QFB_OK;
  if (qfb_status s = nccl_ready()) return s;
  ncclResult_t r = nccl().destroy(static_cast<ncclComm_t>(comm));
  if (r != ncclSuccess) return nccl_fail(r, "ncclCommDestroy");
  return QFB_OK;
}

qfb_status qfb_allreduce_scale_grads(qfb_ctx* ctx, void* comm, double* grads, int64_t n) {
  if (!ctx || !comm || !grads || n < 0) return qfb::set_error(QFB_ERR_VALUE, "allreduce_scale_grads: bad arguments");
  if (n == 0) return QFB_OK;
  if (qfb_status s = nccl_ready()) return s;
  ncclResult_t r = nccl().all_reduce(grads, grads, (size_t)n, ncclFloat64, ncclSum,
                                     static_cast<ncclComm_t>(comm), qfb::ctx_stream(ctx));
  if (r != ncclSuccess) return nccl_fail(r, "ncclAllReduce");
  return QFB_OK;
}

qfb_status qfb_gather_fold_scale_grads(qfb_ctx* ctx, void* comm, const double* rows, int64_t rows_per_rank,
                                       int64_t n, double* gathered, const double* into, double* out) {
  if (!ctx || !comm || !rows || !gathered || !out || rows_per_rank < 1 || n < 0)
    return qfb::set_error(QFB_ERR_VALUE, "gather_fold_scale_grads: bad arguments");
  if (n == 0) return QFB_OK;
  if (qfb_status s = nccl_ready()) return s;
  int nranks = 0;
  ncclResult_t r = nccl().count(static_cast<ncclComm_t>(comm), &nranks);
  if (r != ncclSuccess) return nccl_fail(r, "ncclCommCount");
  // rank k's rows land at gathered[k * rows_per_rank * n ...]: global row
  // order = rank-major = frame order when rank k holds frames
  // [k * rows_per_rank, (k + 1) * rows_per_rank)
  r = nccl().all_gather(rows, gathered, (size_t)(rows_per_rank * n), ncclFloat64,
                        static_cast<ncclComm_t>(comm), qfb::ctx_stream(ctx));
  if (r != ncclSuccess) return nccl_fail(r, "ncclAllGather");
  return qfb_fold_rows(ctx, gathered, (int64_t)nranks * rows_per_rank, n, into, out);
}

}  // extern "C"
