// Interface halo sum and scalar allreduce over NCCL for the z-slab
// decomposition (SURVEY.md 8(b) `fpb_halo_sum`, 8(e)): the compiled
// multi-GPU entry points, so a C-ABI caller can run the decomposed step
// without Python's torch.distributed.
//
// NCCL is resolved at run time (dlopen of libnccl.so.2, preferring the copy
// torch already loaded), so libfempack_b200.so itself has no link-time NCCL
// dependency and single-GPU users never load it.
//
// fpb_halo_exchange: every segment (peer, send offset, receive offset,
// count) of x is sent to `peer` and the peer's matching segment received,
// all in one NCCL group (sends and receives to one peer pair up in call
// order — both sides list their segments in the same order); summing mode
// receives into scratch and one kernel adds it into x (fpb_halo_sum: the
// interface-row sums), copy mode receives in place (ghost-plane refresh).
// Stream-ordered and capturable in a CUDA graph (NCCL P2P and allreduce are
// graph-capturable).  a + b == b + a bit for bit, so both
// copies of an interface row end up with the same value.
#include <dlfcn.h>
#include <nccl.h>

#include "common.cuh"

namespace fpb {

struct NcclApi {
  bool ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*);
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*GroupStart)();
  ncclResult_t (*GroupEnd)();
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t);
  const char* (*GetErrorString)(ncclResult_t);
};

static NcclApi g_nccl;

static bool nccl_load() {
  if (g_nccl.ok) return true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) {
    set_error("libnccl.so.2 not loadable: %s", dlerror());
    return false;
  }
#define FPB_SYM(f, name)                                                   \
  g_nccl.f = reinterpret_cast<decltype(g_nccl.f)>(dlsym(h, name));          \
  if (!g_nccl.f) {                                                         \
    set_error("libnccl.so.2 lacks %s", name);                              \
    return false;                                                          \
  }
  FPB_SYM(GetUniqueId, "ncclGetUniqueId")
  FPB_SYM(CommInitRank, "ncclCommInitRank")
  FPB_SYM(CommDestroy, "ncclCommDestroy")
  FPB_SYM(Send, "ncclSend")
  FPB_SYM(Recv, "ncclRecv")
  FPB_SYM(GroupStart, "ncclGroupStart")
  FPB_SYM(GroupEnd, "ncclGroupEnd")
  FPB_SYM(AllReduce, "ncclAllReduce")
  FPB_SYM(GetErrorString, "ncclGetErrorString")
#undef FPB_SYM
  g_nccl.ok = true;
  return true;
}

#define FPB_NCCL(call)                                                                  \
  do {                                                                                  \
    ncclResult_t r_ = (call);                                                           \
    if (r_ != ncclSuccess) {                                                            \
      ::fpb::set_error("%s:%d %s: %s", __FILE__, __LINE__, #call, g_nccl.GetErrorString(r_)); \
      return FPB_ECUDA;                                                                 \
    }                                                                                   \
  } while (0)

constexpr int kHaloMaxSeg = 16;

struct HaloSegs {
  int n;
  int64_t off[kHaloMaxSeg];   // segment start in x
  int64_t cnt[kHaloMaxSeg];   // length
  int64_t soff[kHaloMaxSeg];  // start in scratch (exclusive prefix of cnt)
};

__global__ void k_halo_add(HaloSegs s, int64_t total, const double* __restrict__ scratch, double* __restrict__ x) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    int i = 0;
#pragma unroll 1
    while (i + 1 < s.n && t >= s.soff[i + 1]) ++i;
    x[s.off[i] + (t - s.soff[i])] += scratch[t];
  }
}

}  // namespace fpb

using namespace fpb;

extern "C" {

int fpb_nccl_unique_id(unsigned char* id128) {
  if (!nccl_load()) return FPB_ECONFIG;
  ncclUniqueId id;
  FPB_NCCL(g_nccl.GetUniqueId(&id));
  memcpy(id128, id.internal, sizeof(id.internal));
  return FPB_OK;
}

int fpb_nccl_comm_init(int nranks, int rank, const unsigned char* id128, int device, void** comm) {
  FPB_REQUIRE(nranks >= 1 && rank >= 0 && rank < nranks, "bad rank %d of %d", rank, nranks);
  if (!nccl_load()) return FPB_ECONFIG;
  FPB_CUDA(cudaSetDevice(device));
  ncclUniqueId id;
  memcpy(id.internal, id128, sizeof(id.internal));
  ncclComm_t c = nullptr;
  FPB_NCCL(g_nccl.CommInitRank(&c, nranks, id, rank));
  *comm = c;
  return FPB_OK;
}

int fpb_nccl_comm_destroy(void* comm) {
  if (!comm) return FPB_OK;
  if (!nccl_load()) return FPB_ECONFIG;
  FPB_NCCL(g_nccl.CommDestroy(reinterpret_cast<ncclComm_t>(comm)));
  return FPB_OK;
}

int fpb_halo_exchange(void* comm, int nseg, const int32_t* peers, const int64_t* send_off, const int64_t* recv_off,
                      const int64_t* counts, int add, double* x, double* scratch, void* stream) {
  FPB_REQUIRE(nseg >= 0 && nseg <= kHaloMaxSeg, "at most %d halo segments (got %d)", kHaloMaxSeg, nseg);
  if (nseg == 0) return FPB_OK;
  if (!nccl_load()) return FPB_ECONFIG;
  cudaStream_t s = as_stream(stream);
  ncclComm_t c = reinterpret_cast<ncclComm_t>(comm);
  HaloSegs hs;
  hs.n = nseg;
  int64_t total = 0;
  for (int i = 0; i < nseg; ++i) {
    FPB_REQUIRE(counts[i] >= 0 && send_off[i] >= 0 && recv_off[i] >= 0, "bad halo segment %d", i);
    hs.off[i] = recv_off[i];
    hs.cnt[i] = counts[i];
    hs.soff[i] = total;
    total += counts[i];
  }
  FPB_REQUIRE(!add || scratch, "the summing exchange needs a scratch buffer");
  FPB_NCCL(g_nccl.GroupStart());
  for (int i = 0; i < nseg; ++i) {
    if (!counts[i]) continue;
    FPB_NCCL(g_nccl.Send(x + send_off[i], (size_t)counts[i], ncclFloat64, peers[i], c, s));
    // sum: receive into scratch, add below; copy: straight into place
    double* dst = add ? scratch + hs.soff[i] : x + recv_off[i];
    FPB_NCCL(g_nccl.Recv(dst, (size_t)counts[i], ncclFloat64, peers[i], c, s));
  }
  FPB_NCCL(g_nccl.GroupEnd());
  if (add && total > 0) {
    k_halo_add<<<grid_for(total, 256), 256, 0, s>>>(hs, total, scratch, x);
    FPB_LAUNCH_CHECK();
  }
  return FPB_OK;
}

int fpb_halo_sum(void* comm, int nseg, const int32_t* peers, const int64_t* offsets, const int64_t* counts,
                 double* x, double* scratch, void* stream) {
  return fpb_halo_exchange(comm, nseg, peers, offsets, offsets, counts, 1, x, scratch, stream);
}

int fpb_allreduce_sum(void* comm, double* x, int64_t count, void* stream) {
  if (count <= 0) return FPB_OK;
  if (!nccl_load()) return FPB_ECONFIG;
  FPB_NCCL(g_nccl.AllReduce(x, x, (size_t)count, ncclFloat64, ncclSum, reinterpret_cast<ncclComm_t>(comm),
                            as_stream(stream)));
  return FPB_OK;
}

}  // extern "C"
