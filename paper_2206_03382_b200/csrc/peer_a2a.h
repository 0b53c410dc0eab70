// Copy-engine flexible all-to-all over NVLink peer memory (one process per GPU).
//
// Every rank maps its peers' receive buffers (CUDA IPC) and pushes its blocks with
// cudaMemcpyAsync, one copy stream per destination so the W blocks of a chunk move on separate
// DMA engines at once: the copy engines drive NVLink, so the exchange takes no SMs from the
// persistent expert GEMMs it overlaps with. Ordering across
// processes uses 32-bit epoch flags in each receiver's memory:
//   ready[ch][src][chunk]  -- written (after the data) by src into dst's flags; the kernel on dst
//                             that first reads the chunk polls it (ld.acquire.sys >= epoch).
//   freed[ch][src]         -- written by src once it has consumed its channel-ch buffer for an
//                             epoch; a sender waits on its own copy before overwriting src's buffer
//                             in the next epoch.
// Epochs are per channel and advance identically on every rank (SPMD call sequence).
// Semantics are all2all_linear / flex_all2all (collectives.cpp:48-56, 116-162).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <cstdint>
#include <functional>
#include <vector>

#include "peer_flags.h"

namespace moe {

class PeerExchange {
 public:
  static constexpr int kChannels = 4;  // fwd dispatch, fwd combine, bwd dispatch, bwd combine
  static constexpr int kMaxChunks = 8;
  // ready-flag slots per (channel, source): one per chunk + kPartSlots for the leading row
  // parts of chunk 0 (its last part publishes the chunk's own slot 0)
  static constexpr int kPartSlots = 7;  // up to 8 row parts
  static constexpr int kPartSlot0 = kMaxChunks;
  static constexpr int kFlagSlots = kMaxChunks + kPartSlots;
  // optional profiling hook: called on the copy stream at the start (begin) and end of each
  // push, so the span covers exactly the concurrent per-destination copies
  std::function<void(int ch, cudaStream_t copy, bool begin)> probe;

  // bufs[ch]: this rank's receive buffer of channel ch (cudaMalloc base pointers).
  // norms (optional): this rank's fp32 per-row receive array of channel 0 (the ReLU certificate's
  // row norms, [rows of recv]); pushes with a norm source copy the rows' norms alongside.
  PeerExchange(int rank, int world, ncclComm_t comm, void* const bufs[kChannels],
               void* norms = nullptr);
  ~PeerExchange();
  PeerExchange(const PeerExchange&) = delete;
  PeerExchange& operator=(const PeerExchange&) = delete;

  // Copy stream: wait until every peer has freed its channel-ch buffer of epoch-1.
  void wait_peers_freed(cudaStream_t copy, int ch, uint32_t epoch);
  // Copy stream: push block p of `src` (offset so[p]) to peer p's channel buffer at the offset p
  // receives from this rank, ro[rank] (moe_a2a_plan is source-symmetric), then publish
  // ready[ch][me][chunk] = epoch to each peer.
  // local_done: recorded right after this rank's own block has been copied; nullptr: the own
  // block is not copied (the producing kernel wrote it into the receive buffer itself).
  // norm_src (optional, channel 0): fp32 norms of src's rows (row_len elements per row).
  void push_chunk(cudaStream_t copy, int ch, int chunk, const void* src, const int64_t* so,
                  const int64_t* ro, size_t block_bytes, size_t esz, uint32_t epoch,
                  cudaEvent_t local_done = nullptr, const float* norm_src = nullptr,
                  int64_t row_len = 1);
  // Copy stream: push rows [row0, row0 + rows) of each of `segs` expert segments (seg_bytes apart;
  // offsets so / ro in BYTES, per destination) to every peer, then publish ready[ch][me][slot].
  // Used to split the first chunk so its first rows land early (the own rows are written in
  // place by the producing kernel).
  void push_rows(cudaStream_t copy, int ch, int slot, const void* src, const int64_t* so,
                 const int64_t* ro, size_t segs, size_t seg_bytes, size_t row0_bytes,
                 size_t rows_bytes, uint32_t epoch, const float* norm_src = nullptr,
                 size_t row_bytes = 1);
  // Wait descriptor for every peer's chunk `chunk` of this epoch: polled on the device by the
  // first consuming kernel (or wait_flags_device). Flags of one source arrive in chunk order, so
  // waiting for chunk c also covers every earlier chunk of the channel.
  FlagWait ready_wait(int ch, int chunk, uint32_t epoch) const;
  // Stream st (after the consumers of channel ch's buffer): tell every peer it is free.
  void signal_freed(cudaStream_t st, int ch, uint32_t epoch);
  // Fused-combine protocol: the producing kernel stores into the peers' channel buffers itself;
  // before the first store, every peer's buffer must be free (device poll of freed[ch][*]) ...
  FlagWait freed_wait(int ch, uint32_t epoch) const;
  // ... and after each chunk's kernel, stream st publishes ready[ch][me][chunk] to every peer.
  void signal_ready(cudaStream_t st, int ch, int chunk, uint32_t epoch);
  // Channel-ch receive buffer of rank p (this rank's own for p == rank).
  void* buffer(int ch, int p) const { return p == rank_ ? local_bufs_[ch] : peer_bufs_[ch][p]; }
  // Channel-0 row-norm array of rank p (null when the exchange carries no norms).
  float* norms(int p) const {
    return static_cast<float*>(p == rank_ ? local_norms_ : (local_norms_ ? peer_norms_[p] : nullptr));
  }

 private:
  uint32_t* ready_local(int ch, int src, int chunk) const;
  uint32_t* freed_local(int ch, int src) const;
  uint32_t* ready_remote(int dst, int ch, int chunk) const;  // my slot in dst's flags
  uint32_t* freed_remote(int dst, int ch) const;
  uint32_t* stage(int slot) const;
  void publish(cudaStream_t st, int slot, uint32_t epoch, const std::vector<uint32_t*>& dsts);
  void publish_one(cudaStream_t st, int slot, uint32_t epoch, uint32_t* dst);

  int rank_, world_;
  void* flags_ = nullptr;                       // this rank's flag block (IPC exported)
  std::vector<void*> peer_flags_;               // mapped flag blocks of peers (nullptr for self)
  std::vector<std::vector<void*>> peer_bufs_;   // [ch][peer] mapped receive buffers
  void* local_bufs_[kChannels];
  void* local_norms_ = nullptr;
  std::vector<void*> peer_norms_;  // mapped norm arrays of peers
  size_t nflags_ = 0;
  std::vector<cudaStream_t> pstreams_;  // per-destination copy streams
  // MOE_CE_SPLIT = s > 1: each destination's block is cut into s pieces on s streams (s copy
  // engines per destination); helper streams / join events per destination (piece 0 on pstreams_)
  int split_ = 1;
  std::vector<std::vector<cudaStream_t>> xstreams_;
  std::vector<std::vector<cudaEvent_t>> xevents_;
  cudaEvent_t ev_in_ = nullptr;
  std::vector<cudaEvent_t> ev_out_;
};

// Driver stream memory operations (resolved through cudaGetDriverEntryPoint).
bool stream_memops_available();
int stream_write_u32(cudaStream_t st, void* addr, uint32_t value);
int stream_wait_geq_u32(cudaStream_t st, const void* addr, uint32_t value);

}  // namespace moe
