// comm.cu — the slab-decomposed grid's exchange over NVLink (SURVEY 8e config 5,
// 2a C1): an NCCL communicator owned by the library, the tile all-to-all as
// grouped ncclSend / ncclRecv (NCCL has no native all-to-all; nccl.h:439-503),
// and one frame of the slab surface with the exchange pipelined per packed
// pair against the row and column passes.
//
// NCCL is resolved at run time (dlopen of libnccl.so.2, reusing the copy a
// host framework already loaded), so the library has no link-time NCCL
// dependency and shares one NCCL with e.g. torch.distributed in a process.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <memory>

#include "objects.cuh"

struct ocn_comm {
  ocn_ctx* ctx = nullptr;
  ncclComm_t comm = nullptr;
  int nranks = 1, rank = 0;
  cudaStream_t xs = nullptr;      // exchange stream (overlaps the passes on ctx->stream)
  cudaEvent_t rows_done[4]{}, xchg_done[4]{};
};

namespace ocn {

// slab.cu: the passes restricted to packed pairs [p0, p0 + np)
void slab_rows_pairs(ocn_slab* sl, double t, double choppiness, void* dev_send, int p0, int np,
                     bool evolve);
void slab_cols_pairs(ocn_slab* sl, void* dev_recv, int p0, int np);
void slab_geometry(const ocn_slab* sl, ocn_ctx** ctx, int* n, int* ranks, int* rank, int* rows);

namespace {

struct NcclApi {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*group_start)() = nullptr;
  ncclResult_t (*group_end)() = nullptr;
  ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  std::string why;
  bool ok() const { return send != nullptr; }
};

NcclApi load_nccl() {
  NcclApi a;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // already in the process?
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) {
    a.why = dlerror() ? dlerror() : "libnccl.so.2 not found";
    return a;
  }
  auto sym = [&](const char* name) { return dlsym(h, name); };
  a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(sym("ncclGetUniqueId"));
  a.comm_init_rank = reinterpret_cast<decltype(a.comm_init_rank)>(sym("ncclCommInitRank"));
  a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(sym("ncclCommDestroy"));
  a.group_start = reinterpret_cast<decltype(a.group_start)>(sym("ncclGroupStart"));
  a.group_end = reinterpret_cast<decltype(a.group_end)>(sym("ncclGroupEnd"));
  a.send = reinterpret_cast<decltype(a.send)>(sym("ncclSend"));
  a.recv = reinterpret_cast<decltype(a.recv)>(sym("ncclRecv"));
  a.error_string = reinterpret_cast<decltype(a.error_string)>(sym("ncclGetErrorString"));
  if (!a.get_unique_id || !a.comm_init_rank || !a.comm_destroy || !a.group_start ||
      !a.group_end || !a.send || !a.recv) {
    a.send = nullptr;
    a.why = "libnccl.so.2 lacks the point-to-point API";
  }
  return a;
}

NcclApi& nccl() {
  static NcclApi api = load_nccl();
  if (!api.ok()) fail(OCN_ERR_CUDA, "NCCL unavailable: %s", api.why.c_str());
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    fail(OCN_ERR_CUDA, "%s: %s", what, nccl().error_string ? nccl().error_string(r) : "NCCL error");
}

// The tile blocks of packed pairs [p0, p0 + np): send layout [dest][4][R][R],
// receive layout [src][4][R][R] complex64; block (peer, p) goes to / comes
// from rank `peer`. The rank's own block is a device copy.
void exchange_pairs(ocn_comm* cm, int rows, void* send, void* recv, int p0, int np,
                    cudaStream_t st) {
  const size_t blk = (size_t)rows * rows;  // complex elements per (peer, pair) block
  auto at = [&](void* base, int peer, int p) {
    return static_cast<char*>(base) + ((size_t)peer * 4 + p) * blk * sizeof(float2);
  };
  for (int p = p0; p < p0 + np; ++p)
    if (send != recv)
      OCN_CUDA(cudaMemcpyAsync(at(recv, cm->rank, p), at(send, cm->rank, p), blk * sizeof(float2),
                               cudaMemcpyDeviceToDevice, st));
  if (cm->nranks == 1) return;
  NcclApi& N = nccl();
  nccl_check(N.group_start(), "ncclGroupStart");
  for (int k = 1; k < cm->nranks; ++k) {
    // pair peers in rank-rotated order so every link is busy from the start
    const int to = (cm->rank + k) % cm->nranks, from = (cm->rank - k + cm->nranks) % cm->nranks;
    for (int p = p0; p < p0 + np; ++p) {
      nccl_check(N.send(at(send, to, p), 2 * blk, ncclFloat, to, cm->comm, st), "ncclSend");
      nccl_check(N.recv(at(recv, from, p), 2 * blk, ncclFloat, from, cm->comm, st), "ncclRecv");
    }
  }
  nccl_check(N.group_end(), "ncclGroupEnd");
}

}  // namespace
}  // namespace ocn

using namespace ocn;

extern "C" {

int ocn_comm_unique_id(char* host_id) {
  return api_call(nullptr, [&] {
    OCN_REQUIRE(host_id, "null argument");
    ncclUniqueId id;
    nccl_check(nccl().get_unique_id(&id), "ncclGetUniqueId");
    std::memcpy(host_id, id.internal, NCCL_UNIQUE_ID_BYTES);
  });
}

int ocn_comm_create(ocn_ctx* ctx, const char* host_id, int nranks, int rank, ocn_comm** out) {
  return api_call(ctx, [&] {
    OCN_REQUIRE(ctx && host_id && out, "null argument");
    OCN_REQUIRE(nranks >= 1 && rank >= 0 && rank < nranks, "bad rank %d of %d", rank, nranks);
    DeviceScope ds(ctx);
    auto cm = std::make_unique<ocn_comm>();
    cm->ctx = ctx;
    cm->nranks = nranks;
    cm->rank = rank;
    if (nranks > 1) {
      ncclUniqueId id;
      std::memcpy(id.internal, host_id, NCCL_UNIQUE_ID_BYTES);
      nccl_check(nccl().comm_init_rank(&cm->comm, nranks, id, rank), "ncclCommInitRank");
    }
    int lo = 0, hi = 0;
    OCN_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    OCN_CUDA(cudaStreamCreateWithPriority(&cm->xs, cudaStreamNonBlocking, hi));
    for (int p = 0; p < 4; ++p) {
      OCN_CUDA(cudaEventCreateWithFlags(&cm->rows_done[p], cudaEventDisableTiming));
      OCN_CUDA(cudaEventCreateWithFlags(&cm->xchg_done[p], cudaEventDisableTiming));
    }
    ctx_retain(ctx);
    *out = cm.release();
  });
}

int ocn_comm_destroy(ocn_comm* cm) {
  if (!cm) return OCN_OK;
  ocn_ctx* ctx = cm->ctx;
  {
    DeviceScope ds(ctx);
    cudaStreamSynchronize(cm->xs);
    for (int p = 0; p < 4; ++p) {
      cudaEventDestroy(cm->rows_done[p]);
      cudaEventDestroy(cm->xchg_done[p]);
    }
    cudaStreamDestroy(cm->xs);
    if (cm->comm) {
      try {
        nccl().comm_destroy(cm->comm);
      } catch (...) {
      }
    }
    delete cm;
  }
  ctx_release(ctx);
  return OCN_OK;
}

int ocn_comm_info(const ocn_comm* cm, int* nranks, int* rank) {
  if (!cm) return OCN_ERR_ARG;
  if (nranks) *nranks = cm->nranks;
  if (rank) *rank = cm->rank;
  return OCN_OK;
}

int ocn_slab_exchange(ocn_slab* sl, ocn_comm* cm, int pair, void* dev_send, void* dev_recv) {
  NvtxRange nv("slab.exchange");
  ocn_ctx* ctx = nullptr;
  int n = 0, ranks = 0, rank = 0, rows = 0;
  if (sl) slab_geometry(sl, &ctx, &n, &ranks, &rank, &rows);
  return api_call(ctx, [&] {
    OCN_REQUIRE(sl && cm && dev_send && dev_recv, "null argument");
    OCN_REQUIRE(cm->nranks == ranks && cm->rank == rank,
                "communicator rank %d of %d does not match the slab's %d of %d", cm->rank,
                cm->nranks, rank, ranks);
    OCN_REQUIRE(pair >= -1 && pair < 4, "pair %d out of range", pair);
    DeviceScope ds(ctx);
    exchange_pairs(cm, rows, dev_send, dev_recv, pair < 0 ? 0 : pair, pair < 0 ? 4 : 1,
                   ctx->stream);
  });
}

int ocn_slab_frame(ocn_slab* sl, ocn_comm* cm, double t, double choppiness, void* dev_send,
                   void* dev_recv) {
  ocn_ctx* ctx = nullptr;
  int n = 0, ranks = 0, rank = 0, rows = 0;
  if (sl) slab_geometry(sl, &ctx, &n, &ranks, &rank, &rows);
  return api_call(ctx, [&] {
    OCN_REQUIRE(sl && dev_send && dev_recv, "null argument");
    OCN_REQUIRE(cm || ranks == 1, "a %d-rank slab needs a communicator", ranks);
    OCN_REQUIRE(!cm || (cm->nranks == ranks && cm->rank == rank),
                "communicator does not match the slab decomposition");
    DeviceScope ds(ctx);
    if (!cm || ranks == 1) {  // no exchange: the column pass reads the row pass's layout
      if (dev_send != dev_recv) {
        slab_rows_pairs(sl, t, choppiness, dev_send, 0, 4, true);
        OCN_CUDA(cudaMemcpyAsync(dev_recv, dev_send, (size_t)4 * rows * n * sizeof(float2),
                                 cudaMemcpyDeviceToDevice, ctx->stream));
      } else {
        slab_rows_pairs(sl, t, choppiness, dev_send, 0, 4, true);
      }
      slab_cols_pairs(sl, dev_recv, 0, 4);
      return;
    }
    // rows(p) -> exchange(p) on the exchange stream -> cols(p): the NVLink
    // transfer of pair p overlaps the row pass of p + 1 and the column pass of p - 1
    cudaStream_t st = ctx->stream;
    for (int p = 0; p < 4; ++p) {
      slab_rows_pairs(sl, t, choppiness, dev_send, p, 1, p == 0);
      OCN_CUDA(cudaEventRecord(cm->rows_done[p], st));
      OCN_CUDA(cudaStreamWaitEvent(cm->xs, cm->rows_done[p], 0));
      exchange_pairs(cm, rows, dev_send, dev_recv, p, 1, cm->xs);
      OCN_CUDA(cudaEventRecord(cm->xchg_done[p], cm->xs));
    }
    for (int p = 0; p < 4; ++p) {
      OCN_CUDA(cudaStreamWaitEvent(st, cm->xchg_done[p], 0));
      slab_cols_pairs(sl, dev_recv, p, 1);
    }
  });
}

}  // extern "C"
