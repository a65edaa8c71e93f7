// exchange.cu -- the cross-rank exchanges of the sharded step (P:79 S2.2 "learners"; SURVEY S8(b),
// S8(e)): the NCCL communicator the library owns (edkm_comm_*), the collectives on it, and the
// kernels of the page-compact count exchange.
//
// The sharded step has two real exchanges: the int32 pattern counts after F1 (exact, order
// independent) and the fp64 gamma_T partials after B1 ("weights are identical in each
// learner", so C_T and dC_0 must come out bit-identical on every rank -- NCCL's all-reduce returns
// the same bits on every rank).  Optional: the table phase split by tensor block, whose results
// are all-gathered (edkm_comm_allgather).
//
// NCCL is loaded at run time (dlopen of libnccl.so.2; in a PyTorch process that is the copy torch
// already loaded, found by its soname), so libedkm.so loads on machines without NCCL and only the
// comm calls fail (EDKM_E_NCCL) there.
#include <dlfcn.h>
#include <nccl.h>
#include <stdio.h>
#include <string.h>

#include "../../include/edkm.h"
#include "common.cuh"
#include "launch.h"

using namespace edkm;

struct edkm_comm {
  ncclComm_t c;
  int rank, nranks, device;
};

namespace {

struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*);
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t);
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t);
  const char* (*GetErrorString)(ncclResult_t);
  ncclResult_t (*GetVersion)(int*);
  bool ok;
  char why[256];
};

NcclApi load_nccl() {
  NcclApi a;
  memset(&a, 0, sizeof(a));
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // the process's NCCL (torch's), if loaded
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);   // else the system's, kept private
  if (!h) {
    snprintf(a.why, sizeof(a.why), "cannot load libnccl.so.2: %s", dlerror());
    return a;
  }
#define EDKM_SYM(field, name)                                                   \
  a.field = reinterpret_cast<decltype(a.field)>(dlsym(h, name));                \
  if (!a.field) {                                                               \
    snprintf(a.why, sizeof(a.why), "libnccl.so.2 has no symbol %s", name);      \
    return a;                                                                   \
  }
  EDKM_SYM(GetUniqueId, "ncclGetUniqueId")
  EDKM_SYM(CommInitRank, "ncclCommInitRank")
  EDKM_SYM(CommDestroy, "ncclCommDestroy")
  EDKM_SYM(AllReduce, "ncclAllReduce")
  EDKM_SYM(AllGather, "ncclAllGather")
  EDKM_SYM(GetErrorString, "ncclGetErrorString")
  EDKM_SYM(GetVersion, "ncclGetVersion")
#undef EDKM_SYM
  a.ok = true;
  return a;
}

const NcclApi& nccl() {
  static const NcclApi a = load_nccl();
  return a;
}

edkm_status nccl_fail(ncclResult_t r, const char* where) {
  char buf[384];
  snprintf(buf, sizeof(buf), "%s: %s", where, nccl().GetErrorString ? nccl().GetErrorString(r) : "NCCL error");
  return set_error(EDKM_E_NCCL, buf);
}

edkm_status need_nccl() {
  if (!nccl().ok) return set_error(EDKM_E_NCCL, nccl().why);
  return EDKM_OK;
}

// ---------------------------------------------------------------------------- page-compact kernels
// Page p of tensor t = patterns [p*256, p*256+256) of its [65536] counts row (global page id
// t*256 + p).  Counts live in few pages (bf16 N(0, 0.02^2): ~30 of 256), so ranks
// exchange only the pages some rank populated: an all-reduce (MAX) of one byte per page, then a
// sum all-reduce of the packed pages (~7 MB instead of 59 MB for CFG3).

// mask[g] = 1 if page g has a nonzero count: one warp per page, 8 counts per lane (two int4),
// grid-stride over the pages
__global__ void count_pages_kernel(const int32_t* __restrict__ counts, int64_t npages, uint8_t* __restrict__ mask) {
  const int64_t wpb = blockDim.x >> 5;
  const int lane = threadIdx.x & 31;
  for (int64_t g = (int64_t)blockIdx.x * wpb + (threadIdx.x >> 5); g < npages; g += (int64_t)gridDim.x * wpb) {
    const int4* p = reinterpret_cast<const int4*>(counts + g * 256) + lane * 2;
    const int4 a = __ldg(p), b = __ldg(p + 1);
    const int any = (a.x | a.y | a.z | a.w | b.x | b.y | b.z | b.w) != 0;
    const unsigned m = __ballot_sync(0xffffffffu, any);
    if (lane == 0) mask[g] = m != 0;
  }
}

// DIR 0: compact[i] = page pages[i] of the table; DIR 1: page pages[i] of the table = compact[i].
// A page is 256 entries of `esize` bytes (q16 = 16 * esize int4 words).  One 64-thread group per
// page, grid-stride over the page list; a page id outside [0, npages_table) is skipped.
template <int DIR>
__global__ void page_copy_kernel(int4* __restrict__ table, const int32_t* __restrict__ pages, int npages,
                                 int4* __restrict__ compact, int64_t npages_table, int q16) {
  const int per = blockDim.x >> 6;
  for (int i = blockIdx.x * per + (threadIdx.x >> 6); i < npages; i += gridDim.x * per) {
    const int32_t pg = __ldg(pages + i);
    if (pg < 0 || pg >= npages_table) continue;
    int4* c = table + (int64_t)pg * q16;
    int4* k = compact + (int64_t)i * q16;
    for (int q = threadIdx.x & 63; q < q16; q += 64) {
      if (DIR == 0) k[q] = c[q];
      else c[q] = k[q];
    }
  }
}

int grid_pages(int64_t npages, int per_block) {
  int64_t g = (npages + per_block - 1) / per_block;
  if (g > 148 * 16) g = 148 * 16;
  return g < 1 ? 1 : (int)g;
}

}  // namespace

namespace edkm {
// F1's all-reduce of the counts, and B1's all-reduce of gamma_T, on the caller's stream (api.cu)
edkm_status comm_allreduce_sum(edkm_comm* comm, void* buf, size_t count, int fp64, cudaStream_t s) {
  if (!comm || count == 0) return EDKM_OK;
  EDKM_NVTX(fp64 ? "edkm allreduce gamma" : "edkm allreduce counts");
  const ncclResult_t r = nccl().AllReduce(buf, buf, count, fp64 ? ncclFloat64 : ncclInt32, ncclSum, comm->c, s);
  return r == ncclSuccess ? EDKM_OK : nccl_fail(r, fp64 ? "ncclAllReduce(gamma)" : "ncclAllReduce(counts)");
}
}  // namespace edkm

extern "C" {

edkm_status edkm_comm_unique_id(void* id_out) {
  edkm_status st = need_nccl();
  if (st != EDKM_OK) return st;
  if (!id_out) return set_error(EDKM_E_ARG, "id_out is NULL");
  ncclUniqueId id;
  const ncclResult_t r = nccl().GetUniqueId(&id);
  if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
  memcpy(id_out, &id, sizeof(id));
  return EDKM_OK;
}

edkm_status edkm_comm_init(edkm_comm** out, const void* id, int rank, int nranks) {
  if (!out || !id) return set_error(EDKM_E_ARG, "out or id is NULL");
  *out = nullptr;
  if (nranks < 1 || rank < 0 || rank >= nranks) return set_error(EDKM_E_ARG, "rank must be in [0, nranks), nranks >= 1");
  edkm_status st = need_nccl();
  if (st != EDKM_OK) return st;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return set_error(EDKM_E_CUDA, cudaGetErrorString(e));
  ncclUniqueId uid;
  memcpy(&uid, id, sizeof(uid));
  ncclComm_t c = nullptr;
  const ncclResult_t r = nccl().CommInitRank(&c, nranks, uid, rank);
  if (r != ncclSuccess) return nccl_fail(r, "ncclCommInitRank");
  *out = new edkm_comm{c, rank, nranks, dev};
  return EDKM_OK;
}

edkm_status edkm_comm_destroy(edkm_comm* comm) {
  if (!comm) return EDKM_OK;
  const ncclResult_t r = nccl().CommDestroy(comm->c);
  delete comm;
  return r == ncclSuccess ? EDKM_OK : nccl_fail(r, "ncclCommDestroy");
}

edkm_status edkm_comm_info(const edkm_comm* comm, int* rank, int* nranks, int* nccl_version) {
  if (!comm) return set_error(EDKM_E_ARG, "comm is NULL");
  if (rank) *rank = comm->rank;
  if (nranks) *nranks = comm->nranks;
  if (nccl_version) {
    *nccl_version = 0;
    if (nccl().GetVersion) nccl().GetVersion(nccl_version);
  }
  return EDKM_OK;
}

edkm_status edkm_comm_allreduce(edkm_comm* comm, void* buf, size_t count, int dtype, int op, void* stream) {
  if (!comm) return set_error(EDKM_E_ARG, "comm is NULL");
  if (count > 0 && !buf) return set_error(EDKM_E_ARG, "buf is NULL");
  ncclDataType_t t;
  switch (dtype) {
    case EDKM_I32: t = ncclInt32; break;
    case EDKM_FP64: t = ncclFloat64; break;
    case EDKM_FP32: t = ncclFloat32; break;
    case EDKM_U8: t = ncclUint8; break;
    default: return set_error(EDKM_E_DTYPE, "allreduce dtype must be I32, FP64, FP32 or U8");
  }
  if (op != EDKM_SUM && op != EDKM_MAX) return set_error(EDKM_E_ARG, "op must be EDKM_SUM or EDKM_MAX");
  if (count == 0) return EDKM_OK;
  EDKM_NVTX("edkm comm allreduce");
  const ncclResult_t r = nccl().AllReduce(buf, buf, count, t, op == EDKM_SUM ? ncclSum : ncclMax, comm->c,
                                          (cudaStream_t)stream);
  return r == ncclSuccess ? EDKM_OK : nccl_fail(r, "ncclAllReduce");
}

edkm_status edkm_comm_allgather(edkm_comm* comm, const void* send, void* recv, size_t bytes_per_rank, void* stream) {
  if (!comm) return set_error(EDKM_E_ARG, "comm is NULL");
  if (bytes_per_rank > 0 && (!send || !recv)) return set_error(EDKM_E_ARG, "send or recv is NULL");
  if (bytes_per_rank == 0) return EDKM_OK;
  EDKM_NVTX("edkm comm allgather");
  cudaStream_t s = (cudaStream_t)stream;
  const ncclResult_t r = nccl().AllGather(send, recv, bytes_per_rank, ncclUint8, comm->c, s);
  return r == ncclSuccess ? EDKM_OK : nccl_fail(r, "ncclAllGather");
}

edkm_status edkm_count_pages(const int32_t* counts, int nt, uint8_t* mask, void* stream) {
  reset_launches();
  if (nt < 0) return set_error(EDKM_E_ARG, "nt < 0");
  if (nt == 0) return EDKM_OK;
  if (!counts || !mask) return set_error(EDKM_E_ARG, "NULL buffer");
  const int64_t np = (int64_t)nt * 256;
  count_pages_kernel<<<grid_pages(np, 8), 256, 0, (cudaStream_t)stream>>>(counts, np, mask);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(EDKM_E_CUDA, cudaGetErrorString(e));
  add_launches(1);
  return EDKM_OK;
}

static edkm_status page_copy(int dir, void* table, int esize, int nt, const int32_t* pages, int npages, void* compact,
                             void* stream) {
  reset_launches();
  if (esize != 1 && esize != 2 && esize != 4 && esize != 8) return set_error(EDKM_E_ARG, "esize must be 1, 2, 4 or 8");
  if (nt < 0 || npages < 0 || (int64_t)npages > (int64_t)nt * 256) return set_error(EDKM_E_ARG, "need 0 <= npages <= 256 nt");
  if (npages == 0) return EDKM_OK;
  if (!table || !pages || !compact) return set_error(EDKM_E_ARG, "NULL buffer");
  if (((uintptr_t)table | (uintptr_t)compact) & 15u) return set_error(EDKM_E_ARG, "buffers must be 16-byte aligned");
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t ncp = (int64_t)nt * 256;
  const int q16 = 16 * esize;
  int4* t4 = reinterpret_cast<int4*>(table);
  int4* c4 = reinterpret_cast<int4*>(compact);
  if (dir == 0) page_copy_kernel<0><<<grid_pages(npages, 4), 256, 0, s>>>(t4, pages, npages, c4, ncp, q16);
  else page_copy_kernel<1><<<grid_pages(npages, 4), 256, 0, s>>>(t4, pages, npages, c4, ncp, q16);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(EDKM_E_CUDA, cudaGetErrorString(e));
  add_launches(1);
  return EDKM_OK;
}

edkm_status edkm_counts_pack(const int32_t* counts, int nt, const int32_t* pages, int npages, int32_t* compact,
                             void* stream) {
  return page_copy(0, const_cast<int32_t*>(counts), 4, nt, pages, npages, compact, stream);
}

edkm_status edkm_counts_unpack(const int32_t* compact, const int32_t* pages, int npages, int nt, int32_t* counts,
                               void* stream) {
  return page_copy(1, counts, 4, nt, pages, npages, const_cast<int32_t*>(compact), stream);
}

edkm_status edkm_pages_pack(const void* table, int esize, int nt, const int32_t* pages, int npages, void* compact,
                            void* stream) {
  return page_copy(0, const_cast<void*>(table), esize, nt, pages, npages, compact, stream);
}

edkm_status edkm_pages_unpack(const void* compact, int esize, const int32_t* pages, int npages, int nt, void* table,
                              void* stream) {
  return page_copy(1, table, esize, nt, pages, npages, const_cast<void*>(compact), stream);
}

}  // extern "C"
