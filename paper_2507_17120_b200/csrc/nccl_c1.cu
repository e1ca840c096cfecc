// nccl_c1.cu — C1, the one exchange step of a sharded window, over NCCL owned by the
// library: the sum of the ranks' per-(class, length) histograms.
//
// The reference has no distributed code (NVLink appears only as a cost formula,
// pd_sim.py:93-96); what must hold is that every rank runs K2 on the same global
// histogram, so the edges are identical everywhere and equal to the single-window
// edges of the whole trace.  The all-reduce is issued on the window's own stream
// between K1 and K2 inside bs_window_schedule, so with a communicator attached the
// whole window — K1, C1, K2..K6 — is one stream sequence that a CUDA graph captures
// (NCCL collectives are capturable), instead of K1 / host all-reduce / graph replay.
//
// libnccl is resolved at run time (dlopen): the instance the process already loaded
// (PyTorch's, by soname) is reused, so a communicator made here and torch's NCCL
// process group live in the same library.  No NCCL type crosses bucketserve.h: the
// unique id is 128 opaque bytes, a caller-owned communicator is a void*.
#include <dlfcn.h>

#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include "ctx.cuh"

namespace {

// the NCCL ABI pieces used here (nccl.h; stable since NCCL 2.0)
typedef struct { char internal[BS_NCCL_ID_BYTES]; } NcclUid;
typedef int (*fn_get_uid)(NcclUid*);
typedef int (*fn_init_rank)(void** comm, int nranks, NcclUid id, int rank);
typedef int (*fn_all_reduce)(const void*, void*, size_t, int dtype, int op, void* comm,
                             cudaStream_t);
typedef int (*fn_destroy)(void*);
typedef const char* (*fn_err)(int);
constexpr int kNcclUint32 = 3, kNcclSum = 0;

struct NcclApi {
  fn_get_uid get_uid = nullptr;
  fn_init_rank init_rank = nullptr;
  fn_all_reduce all_reduce = nullptr;
  fn_destroy destroy = nullptr;
  fn_err err = nullptr;
  std::string why;
};

NcclApi load_nccl() {
  NcclApi a;
  void* h = nullptr;
  if (const char* p = getenv("BS_NCCL_LIB")) h = dlopen(p, RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // the process's NCCL (torch)
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) {
    const char* e = dlerror();
    a.why = std::string("libnccl.so.2 not found: ") + (e ? e : "?");
    return a;
  }
  a.get_uid = reinterpret_cast<fn_get_uid>(dlsym(h, "ncclGetUniqueId"));
  a.init_rank = reinterpret_cast<fn_init_rank>(dlsym(h, "ncclCommInitRank"));
  a.all_reduce = reinterpret_cast<fn_all_reduce>(dlsym(h, "ncclAllReduce"));
  a.destroy = reinterpret_cast<fn_destroy>(dlsym(h, "ncclCommDestroy"));
  a.err = reinterpret_cast<fn_err>(dlsym(h, "ncclGetErrorString"));
  if (!a.get_uid || !a.init_rank || !a.all_reduce || !a.destroy || !a.err)
    a.why = "libnccl lacks a required symbol";
  return a;
}

const NcclApi& nccl() {
  static NcclApi api = load_nccl();  // thread-safe one-time init
  return api;
}

std::string nccl_msg(const char* what, int r) {
  return std::string(what) + ": " + (nccl().err ? nccl().err(r) : "nccl error") + " (" +
         std::to_string(r) + ")";
}

}  // namespace

namespace bsk {

int nccl_status(std::string* why) {
  const NcclApi& a = nccl();
  if (!a.why.empty()) {
    if (why) *why = a.why;
    return -1;
  }
  return 0;
}

int nccl_unique_id(void* id_out, std::string* why) {
  if (nccl_status(why)) return -1;
  NcclUid u;
  const int r = nccl().get_uid(&u);
  if (r) {
    *why = nccl_msg("ncclGetUniqueId", r);
    return -1;
  }
  memcpy(id_out, &u, sizeof u);
  return 0;
}

int nccl_comm_init(void** comm, int world, const void* id, int rank, std::string* why) {
  if (nccl_status(why)) return -1;
  NcclUid u;
  memcpy(&u, id, sizeof u);
  const int r = nccl().init_rank(comm, world, u, rank);
  if (r) {
    *why = nccl_msg("ncclCommInitRank", r);
    return -1;
  }
  return 0;
}

void nccl_comm_destroy(void* comm) {
  if (comm && nccl().destroy) nccl().destroy(comm);
}

// C1: hist_global = sum over ranks of hist_local (C * L uint32 counts), on `st`
int nccl_allreduce_hist(bs_ctx* ctx, const uint32_t* hist_local, uint32_t* hist_global,
                        size_t count, cudaStream_t st, std::string* why) {
  const int r = nccl().all_reduce(hist_local, hist_global, count, kNcclUint32, kNcclSum,
                                  ctx->nccl_comm, st);
  if (r) {
    *why = nccl_msg("ncclAllReduce", r);
    return -1;
  }
  return 0;
}

}  // namespace bsk
