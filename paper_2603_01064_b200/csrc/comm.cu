// Collectives of the slab-sharded mode: NCCL (one process per GPU) and an in-process
// emulation of W ranks on one GPU (see comm.h).
#include <dlfcn.h>
#include <nccl.h>

#include <chrono>
#include <condition_variable>
#include <cstring>
#include <memory>
#include <mutex>
#include <vector>

#include "comm.h"
#include "common.cuh"

namespace nmg {
namespace {

__global__ void sum_ranks_kernel(int world, int64_t count, const double* __restrict__ g, double* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  double s = 0.0;
  for (int q = 0; q < world; ++q) s += g[(int64_t)q * count + i];   // fixed rank order
  out[i] = s;
}

// ---------------------------------------------------------------- NCCL (dlopen)
struct NcclApi {
  void* so = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
};

NcclApi* nccl_api() {
  static NcclApi api;
  static bool tried = false;
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  if (tried) return api.so ? &api : nullptr;
  tried = true;
  api.so = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!api.so) return nullptr;
  bool ok = true;
  auto sym = [&](auto& fp, const char* name) {
    fp = reinterpret_cast<std::remove_reference_t<decltype(fp)>>(dlsym(api.so, name));
    ok = ok && fp != nullptr;
  };
  sym(api.GetUniqueId, "ncclGetUniqueId");
  sym(api.CommInitRank, "ncclCommInitRank");
  sym(api.CommDestroy, "ncclCommDestroy");
  sym(api.AllGather, "ncclAllGather");
  sym(api.Send, "ncclSend");
  sym(api.Recv, "ncclRecv");
  sym(api.GroupStart, "ncclGroupStart");
  sym(api.GroupEnd, "ncclGroupEnd");
  sym(api.GetErrorString, "ncclGetErrorString");
  sym(api.CommGetAsyncError, "ncclCommGetAsyncError");
  if (!ok) { dlclose(api.so); api.so = nullptr; return nullptr; }
  return &api;
}

#define NMG_NCCL(expr)                                                                          \
  do {                                                                                          \
    ncclResult_t _r = (expr);                                                                   \
    if (_r != ncclSuccess) return nmg::comm_fail(NMG_ERR_NCCL, "NCCL %s: %s", #expr, api->GetErrorString(_r)); \
  } while (0)

struct NcclComm final : nmg_comm {
  NcclApi* api = nullptr;
  ncclComm_t c = nullptr;
  ~NcclComm() override { if (c && api) api->CommDestroy(c); }
  nmg_status check_async() override {
    ncclResult_t ar = ncclSuccess;
    NMG_NCCL(api->CommGetAsyncError(c, &ar));
    if (ar != ncclSuccess && ar != ncclInProgress)
      return nmg::comm_fail(NMG_ERR_NCCL, "NCCL asynchronous error: %s", api->GetErrorString(ar));
    return NMG_OK;
  }
  nmg_status all_gather(const void* send, void* recv, size_t bytes, cudaStream_t s) override {
    NMG_NCCL(api->AllGather(send, recv, bytes, ncclChar, c, s));
    return NMG_OK;
  }
  nmg_status all_to_all(const void* send, void* recv, size_t bytes, cudaStream_t s) override {
    NMG_NCCL(api->GroupStart());
    for (int q = 0; q < world; ++q) {
      NMG_NCCL(api->Send(static_cast<const char*>(send) + q * bytes, bytes, ncclChar, q, c, s));
      NMG_NCCL(api->Recv(static_cast<char*>(recv) + q * bytes, bytes, ncclChar, q, c, s));
    }
    NMG_NCCL(api->GroupEnd());
    return NMG_OK;
  }
};

// ---------------------------------------------------------------- in-process emulation
struct EmuGroup {
  int W = 1;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  bool broken = false;
  struct Slot { const void* send = nullptr; void* recv = nullptr; size_t bytes = 0; cudaEvent_t ready{}, done{}; };
  std::vector<Slot> slots;
  // host barrier with a timeout: a rank that failed and left makes the others fail too
  bool barrier() {
    std::unique_lock<std::mutex> lk(mu);
    if (broken) return false;
    const uint64_t g = gen;
    if (++arrived == W) {
      arrived = 0;
      ++gen;
      cv.notify_all();
      return true;
    }
    if (!cv.wait_for(lk, std::chrono::seconds(120), [&] { return gen != g || broken; }) || broken) {
      broken = true;
      cv.notify_all();
      return false;
    }
    return true;
  }
};

struct EmuComm final : nmg_comm {
  std::shared_ptr<EmuGroup> g;
  ~EmuComm() override {
    cudaEventDestroy(g->slots[rank].ready);
    cudaEventDestroy(g->slots[rank].done);
  }
  nmg_status exchange(const void* send, void* recv, size_t bytes, bool a2a, cudaStream_t s) {
    EmuGroup& G = *g;
    auto& me = G.slots[rank];
    me.send = send; me.recv = recv; me.bytes = bytes;
    if (cudaEventRecord(me.ready, s) != cudaSuccess) return comm_fail(NMG_ERR_CUDA, "emulated collective: event record");
    if (!G.barrier()) return comm_fail(NMG_ERR_NCCL, "emulated collective: a peer rank failed or timed out");
    for (int q = 0; q < world; ++q) {
      if (G.slots[q].bytes != bytes) return comm_fail(NMG_ERR_INVALID_ARG, "emulated collective: size mismatch");
      cudaStreamWaitEvent(s, G.slots[q].ready, 0);
    }
    for (int q = 0; q < world; ++q) {
      const char* src = static_cast<const char*>(G.slots[q].send) + (a2a ? rank * bytes : 0);
      if (cudaMemcpyAsync(static_cast<char*>(recv) + q * bytes, src, bytes, cudaMemcpyDeviceToDevice, s) != cudaSuccess)
        return comm_fail(NMG_ERR_CUDA, "emulated collective: copy");
    }
    cudaEventRecord(me.done, s);
    if (!G.barrier()) return comm_fail(NMG_ERR_NCCL, "emulated collective: a peer rank failed or timed out");
    for (int q = 0; q < world; ++q) cudaStreamWaitEvent(s, G.slots[q].done, 0);   // peers finished reading `send`
    if (!G.barrier()) return comm_fail(NMG_ERR_NCCL, "emulated collective: a peer rank failed or timed out");
    return NMG_OK;
  }
  nmg_status all_gather(const void* send, void* recv, size_t bytes, cudaStream_t s) override {
    return exchange(send, recv, bytes, false, s);
  }
  nmg_status all_to_all(const void* send, void* recv, size_t bytes, cudaStream_t s) override {
    return exchange(send, recv, bytes, true, s);
  }
};

}  // namespace

void sum_ranks_f64(int world, size_t count, const double* gathered, double* out, cudaStream_t s) {
  sum_ranks_kernel<<<(int)ceil_div64((int64_t)count, 128), 128, 0, s>>>(world, (int64_t)count, gathered, out);
}

}  // namespace nmg

nmg_status nmg_comm::sum_f64(double* buf, size_t count, double* scratch, cudaStream_t s) {
  if (world == 1) return NMG_OK;
  nmg_status st = all_gather(buf, scratch, count * sizeof(double), s);
  if (st != NMG_OK) return st;
  nmg::sum_ranks_f64(world, count, scratch, buf, s);
  return cudaGetLastError() == cudaSuccess ? NMG_OK : nmg::comm_fail(NMG_ERR_CUDA, "sum_ranks launch");
}

extern "C" {

nmg_status nmg_comm_nccl_unique_id(void* out128) {
  if (!out128) return nmg::comm_fail(NMG_ERR_INVALID_ARG, "null argument");
  nmg::NcclApi* api = nmg::nccl_api();
  if (!api) return nmg::comm_fail(NMG_ERR_UNSUPPORTED, "libnccl.so.2 not loadable");
  ncclUniqueId id;
  NMG_NCCL(api->GetUniqueId(&id));
  static_assert(sizeof(ncclUniqueId) == NMG_COMM_ID_BYTES, "ncclUniqueId size");
  std::memcpy(out128, &id, sizeof id);
  return NMG_OK;
}

nmg_status nmg_comm_create_nccl(int32_t world, int32_t rank, const void* id128, int32_t device, nmg_comm** out) {
  if (!id128 || !out || world < 1 || rank < 0 || rank >= world)
    return nmg::comm_fail(NMG_ERR_INVALID_ARG, "bad world/rank/id");
  *out = nullptr;
  nmg::NcclApi* api = nmg::nccl_api();
  if (!api) return nmg::comm_fail(NMG_ERR_UNSUPPORTED, "libnccl.so.2 not loadable");
  if (cudaSetDevice(device) != cudaSuccess) return nmg::comm_fail(NMG_ERR_CUDA, "cudaSetDevice(%d)", device);
  auto c = std::make_unique<nmg::NcclComm>();
  c->api = api;
  c->world = world;
  c->rank = rank;
  ncclUniqueId id;
  std::memcpy(&id, id128, sizeof id);
  NMG_NCCL(api->CommInitRank(&c->c, world, id, rank));
  *out = c.release();
  return NMG_OK;
}

nmg_status nmg_comm_create_emulated(int32_t world, nmg_comm** out) {
  if (!out || world < 1) return nmg::comm_fail(NMG_ERR_INVALID_ARG, "bad world");
  auto g = std::make_shared<nmg::EmuGroup>();
  g->W = world;
  g->slots.resize(world);
  for (int r = 0; r < world; ++r) {
    if (cudaEventCreateWithFlags(&g->slots[r].ready, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&g->slots[r].done, cudaEventDisableTiming) != cudaSuccess)
      return nmg::comm_fail(NMG_ERR_CUDA, "cudaEventCreate (no CUDA device?)");
  }
  for (int r = 0; r < world; ++r) {
    auto* c = new nmg::EmuComm();
    c->world = world;
    c->rank = r;
    c->g = g;
    out[r] = c;
  }
  return NMG_OK;
}

void nmg_comm_destroy(nmg_comm* c) { delete c; }

}  // extern "C"
