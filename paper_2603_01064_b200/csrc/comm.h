// Collectives of the slab-sharded single-system mode (one operator
// row-sharded over the ranks).  Three collectives, all stream-ordered on the caller's stream:
//   all_gather  : recv = [world][bytes], rank q's `send` at offset q * bytes
//   all_to_all  : recv chunk q = rank q's send chunk `rank` (equal chunk sizes)
//   sum_f64     : element-wise sum over the ranks of `count` doubles, in place; computed as
//                 an all-gather followed by a fixed-order (rank 0, 1, ...) sum on every rank,
//                 so every rank holds bitwise the same result (the stop decisions of nmg_solve
//                 and the smoother norms agree across ranks)
// Implementations (comm.cu):
//   NcclComm : one process per GPU, NCCL (dlopen'ed libnccl.so.2, no link-time dependency),
//              ncclAllGather / grouped ncclSend+ncclRecv over NVLink/NVSwitch.
//   EmuComm  : W ranks in ONE process on one GPU, one host thread per rank (tests and the
//              single-GPU emulation of the multi-rank path).  Ranks meet at a host barrier and
//              exchange CUDA events; the copies are cudaMemcpyAsync on each rank's own stream
//              after stream waits on the peers' events.  No kernel ever waits on another rank's
//              kernel (no device-side spin), so W ranks on one GPU cannot deadlock the device.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include "../../include/nmg.h"

struct nmg_comm {
  int world = 1, rank = 0;
  virtual ~nmg_comm() {}
  virtual nmg_status all_gather(const void* send, void* recv, size_t bytes, cudaStream_t s) = 0;
  virtual nmg_status all_to_all(const void* send, void* recv, size_t bytes_per_peer, cudaStream_t s) = 0;
  // asynchronous communicator errors (NCCL: ncclCommGetAsyncError); NMG_OK when healthy
  virtual nmg_status check_async() { return NMG_OK; }
  // scratch: device, >= world * count doubles
  nmg_status sum_f64(double* buf, size_t count, double* scratch, cudaStream_t s);
};

namespace nmg {
nmg_status comm_fail(nmg_status st, const char* fmt, ...);
void sum_ranks_f64(int world, size_t count, const double* gathered, double* out, cudaStream_t s);
}  // namespace nmg
