// Copy-engine all-to-all over NVLink peer memory. See peer_a2a.h.
#include "peer_a2a.h"

#include <algorithm>
#include <cstdlib>

#include <cudaTypedefs.h>

#include <cstring>
#include <stdexcept>
#include <string>

#include "layer.h"

namespace moe {

namespace {

PFN_cuStreamWaitValue32_v11070 g_wait = nullptr;
PFN_cuStreamWriteValue32_v11070 g_write = nullptr;
bool g_resolved = false;

void resolve() {
  if (g_resolved) return;
  g_resolved = true;
  cudaDriverEntryPointQueryResult q{};
  void* p = nullptr;
  if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
      q == cudaDriverEntryPointSuccess)
    g_wait = reinterpret_cast<PFN_cuStreamWaitValue32_v11070>(p);
  p = nullptr;
  if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
      q == cudaDriverEntryPointSuccess)
    g_write = reinterpret_cast<PFN_cuStreamWriteValue32_v11070>(p);
}

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw MoeError(MOE_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// stage words: [2 * channel + kind][destination] (one per destination stream: an epoch written
// for one peer can never be published to another by a lagging stream)
constexpr int kStageSlots = 2 * PeerExchange::kChannels;

}  // namespace

bool stream_memops_available() {
  resolve();
  return g_wait != nullptr && g_write != nullptr;
}

int stream_write_u32(cudaStream_t st, void* addr, uint32_t value) {
  resolve();
  if (!g_write) return -1;
  return g_write(reinterpret_cast<CUstream>(st), reinterpret_cast<CUdeviceptr>(addr), value,
                 CU_STREAM_WRITE_VALUE_DEFAULT) == CUDA_SUCCESS
             ? 0
             : -2;
}

int stream_wait_geq_u32(cudaStream_t st, const void* addr, uint32_t value) {
  resolve();
  if (!g_wait) return -1;
  return g_wait(reinterpret_cast<CUstream>(st), reinterpret_cast<CUdeviceptr>(addr), value,
                CU_STREAM_WAIT_VALUE_GEQ) == CUDA_SUCCESS
             ? 0
             : -2;
}

PeerExchange::PeerExchange(int rank, int world, ncclComm_t comm, void* const bufs[kChannels],
                           void* norms)
    : rank_(rank), world_(world), local_norms_(norms) {
  if (!stream_memops_available())
    throw MoeError(MOE_ECUDA, "peer all-to-all: CUDA stream memory operations unavailable");
  for (int c = 0; c < kChannels; ++c) local_bufs_[c] = bufs[c];
  nflags_ = static_cast<size_t>(kChannels) * world * kFlagSlots + static_cast<size_t>(kChannels) * world +
            static_cast<size_t>(kStageSlots) * world;
  ck(cudaMalloc(&flags_, nflags_ * sizeof(uint32_t) + 256), "cudaMalloc flags");
  ck(cudaMemset(flags_, 0, nflags_ * sizeof(uint32_t) + 256), "memset flags");

  // Exchange IPC handles of {flags, 4 receive buffers} through NCCL.
  constexpr int kH = 2 + kChannels;  // flags, channel buffers, norms (or a placeholder)
  std::vector<cudaIpcMemHandle_t> mine(kH);
  ck(cudaIpcGetMemHandle(&mine[0], flags_), "cudaIpcGetMemHandle");
  for (int c = 0; c < kChannels; ++c) ck(cudaIpcGetMemHandle(&mine[1 + c], bufs[c]), "cudaIpcGetMemHandle");
  if (norms) ck(cudaIpcGetMemHandle(&mine[1 + kChannels], norms), "cudaIpcGetMemHandle");
  const size_t hb = kH * sizeof(cudaIpcMemHandle_t);
  void* dev = nullptr;
  ck(cudaMalloc(&dev, hb * (world + 1)), "cudaMalloc handles");
  ck(cudaMemcpy(dev, mine.data(), hb, cudaMemcpyHostToDevice), "copy handles");
  cudaStream_t s;
  ck(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "stream");
  if (ncclAllGather(dev, static_cast<char*>(dev) + hb, hb, ncclUint8, comm, s) != ncclSuccess)
    throw MoeError(MOE_ECOMM, "peer all-to-all: handle all-gather failed");
  ck(cudaStreamSynchronize(s), "sync");
  cudaStreamDestroy(s);
  std::vector<cudaIpcMemHandle_t> all(static_cast<size_t>(kH) * world);
  ck(cudaMemcpy(all.data(), static_cast<char*>(dev) + hb, hb * world, cudaMemcpyDeviceToHost), "copy");
  cudaFree(dev);

  pstreams_.assign(world, nullptr);
  ev_out_.assign(world, nullptr);
  for (int p = 0; p < world; ++p) {
    ck(cudaStreamCreateWithFlags(&pstreams_[p], cudaStreamNonBlocking), "stream");
    ck(cudaEventCreateWithFlags(&ev_out_[p], cudaEventDisableTiming), "event");
  }
  ck(cudaEventCreateWithFlags(&ev_in_, cudaEventDisableTiming), "event");
  {
    const char* e = std::getenv("MOE_CE_SPLIT");
    split_ = e ? std::max(1, std::min(8, std::atoi(e))) : 1;
  }
  xstreams_.assign(world, {});
  xevents_.assign(world, {});
  for (int p = 0; p < world; ++p) {
    if (p == rank) continue;
    for (int j = 1; j < split_; ++j) {
      cudaStream_t xs;
      cudaEvent_t xe;
      ck(cudaStreamCreateWithFlags(&xs, cudaStreamNonBlocking), "stream");
      ck(cudaEventCreateWithFlags(&xe, cudaEventDisableTiming), "event");
      xstreams_[p].push_back(xs);
      xevents_[p].push_back(xe);
    }
  }

  peer_flags_.assign(world, nullptr);
  peer_norms_.assign(world, nullptr);
  peer_bufs_.assign(kChannels, std::vector<void*>(world, nullptr));
  for (int p = 0; p < world; ++p) {
    if (p == rank) continue;
    ck(cudaIpcOpenMemHandle(&peer_flags_[p], all[static_cast<size_t>(p) * kH], cudaIpcMemLazyEnablePeerAccess),
       "cudaIpcOpenMemHandle(flags)");
    for (int c = 0; c < kChannels; ++c)
      ck(cudaIpcOpenMemHandle(&peer_bufs_[c][p], all[static_cast<size_t>(p) * kH + 1 + c],
                              cudaIpcMemLazyEnablePeerAccess),
         "cudaIpcOpenMemHandle(buffer)");
    if (norms)  // every rank passes norms or none (same configuration on all ranks)
      ck(cudaIpcOpenMemHandle(&peer_norms_[p], all[static_cast<size_t>(p) * kH + 1 + kChannels],
                              cudaIpcMemLazyEnablePeerAccess),
         "cudaIpcOpenMemHandle(norms)");
  }
}

PeerExchange::~PeerExchange() {
  for (int p = 0; p < world_; ++p) {
    if (p == rank_) continue;
    if (peer_flags_[p]) cudaIpcCloseMemHandle(peer_flags_[p]);
    for (int c = 0; c < kChannels; ++c)
      if (peer_bufs_[c][p]) cudaIpcCloseMemHandle(peer_bufs_[c][p]);
    if (peer_norms_[p]) cudaIpcCloseMemHandle(peer_norms_[p]);
  }
  for (auto st : pstreams_)
    if (st) cudaStreamDestroy(st);
  for (auto& v : xstreams_)
    for (auto st : v) cudaStreamDestroy(st);
  for (auto& v : xevents_)
    for (auto e : v) cudaEventDestroy(e);
  for (auto e : ev_out_)
    if (e) cudaEventDestroy(e);
  if (ev_in_) cudaEventDestroy(ev_in_);
  if (flags_) cudaFree(flags_);
}

// Flag block layout (u32): ready[ch][src][chunk] | freed[ch][src] | stage[2*ch + kind]
uint32_t* PeerExchange::ready_local(int ch, int src, int chunk) const {
  return static_cast<uint32_t*>(flags_) + (static_cast<size_t>(ch) * world_ + src) * kFlagSlots + chunk;
}
uint32_t* PeerExchange::freed_local(int ch, int src) const {
  return static_cast<uint32_t*>(flags_) + static_cast<size_t>(kChannels) * world_ * kFlagSlots +
         static_cast<size_t>(ch) * world_ + src;
}
uint32_t* PeerExchange::ready_remote(int dst, int ch, int chunk) const {
  return static_cast<uint32_t*>(peer_flags_[dst]) + (static_cast<size_t>(ch) * world_ + rank_) * kFlagSlots +
         chunk;
}
uint32_t* PeerExchange::freed_remote(int dst, int ch) const {
  return static_cast<uint32_t*>(peer_flags_[dst]) + static_cast<size_t>(kChannels) * world_ * kFlagSlots +
         static_cast<size_t>(ch) * world_ + rank_;
}
uint32_t* PeerExchange::stage(int slot) const {
  return static_cast<uint32_t*>(flags_) + static_cast<size_t>(kChannels) * world_ * kFlagSlots +
         static_cast<size_t>(kChannels) * world_ + slot;
}

// Write epoch into a local stage word, then DMA it to each destination flag (all in stream
// order, so the flags land after every earlier copy on this stream).
void PeerExchange::publish(cudaStream_t st, int slot, uint32_t epoch, const std::vector<uint32_t*>& dsts) {
  uint32_t* w = stage(slot * world_ + rank_);
  if (stream_write_u32(st, w, epoch) != 0) throw MoeError(MOE_ECUDA, "cuStreamWriteValue32 failed");
  for (uint32_t* d : dsts)
    ck(cudaMemcpyAsync(d, w, sizeof(uint32_t), cudaMemcpyDeviceToDevice, st), "flag copy");
}

void PeerExchange::publish_one(cudaStream_t st, int slot, uint32_t epoch, uint32_t* dst) {
  if (stream_write_u32(st, stage(slot), epoch) != 0) throw MoeError(MOE_ECUDA, "cuStreamWriteValue32 failed");
  ck(cudaMemcpyAsync(dst, stage(slot), sizeof(uint32_t), cudaMemcpyDeviceToDevice, st), "flag copy");
}

void PeerExchange::wait_peers_freed(cudaStream_t copy, int ch, uint32_t epoch) {
  for (int p = 0; p < world_; ++p) {
    if (p == rank_) continue;
    if (stream_wait_geq_u32(copy, freed_local(ch, p), epoch - 1) != 0)
      throw MoeError(MOE_ECUDA, "cuStreamWaitValue32 failed");
  }
}

void PeerExchange::push_chunk(cudaStream_t copy, int ch, int chunk, const void* src, const int64_t* so,
                              const int64_t* ro, size_t block_bytes, size_t esz, uint32_t epoch,
                              cudaEvent_t local_done, const float* norm_src, int64_t row_len) {
  if (norm_src && (ch != 0 || !local_norms_)) throw MoeError(MOE_EINVAL, "peer all-to-all: norms");
  if (chunk >= kMaxChunks) throw MoeError(MOE_EINVAL, "peer all-to-all: too many chunks");
  // Push model: peer p receives my block where it receives "from rank_", i.e. at ro[rank_] of
  // the (source-symmetric) plan. One stream per destination: the blocks move concurrently, and
  // each peer's ready flag follows its own block.
  ck(cudaEventRecord(ev_in_, copy), "event");
  if (probe) probe(ch, copy, true);
  for (int i = 0; i < world_; ++i) {
    const int p = (rank_ + i) % world_;
    if (p == rank_ && local_done == nullptr) continue;
    cudaStream_t ps = pstreams_[p];
    ck(cudaStreamWaitEvent(ps, ev_in_, 0), "wait");
    char* dst = static_cast<char*>(p == rank_ ? local_bufs_[ch] : peer_bufs_[ch][p]) + ro[rank_] * esz;
    const char* sp = static_cast<const char*>(src) + so[p] * esz;
    const int pieces = p == rank_ ? 1 : split_;
    // pieces 1.. on helper streams (more copy engines per destination), joined before the flag
    const size_t piece = ((block_bytes / pieces) + 255) & ~static_cast<size_t>(255);
    for (int j = 1; j < pieces; ++j) {
      const size_t off = piece * j;
      if (off >= block_bytes) break;
      cudaStream_t xs = xstreams_[p][j - 1];
      ck(cudaStreamWaitEvent(xs, ev_in_, 0), "wait");
      ck(cudaMemcpyAsync(dst + off, sp + off, std::min(piece, block_bytes - off), cudaMemcpyDeviceToDevice,
                         xs),
         "peer copy");
    }
    ck(cudaMemcpyAsync(dst, sp, pieces > 1 ? std::min(piece, block_bytes) : block_bytes,
                       cudaMemcpyDeviceToDevice, ps),
       "peer copy");
    for (int j = 1; j < pieces; ++j) {
      if (piece * j >= block_bytes) break;
      ck(cudaEventRecord(xevents_[p][j - 1], xstreams_[p][j - 1]), "event");
      ck(cudaStreamWaitEvent(ps, xevents_[p][j - 1], 0), "wait");
    }
    if (norm_src) {  // the rows' norms travel with them (before the flag)
      float* nd = static_cast<float*>(p == rank_ ? local_norms_ : peer_norms_[p]) + ro[rank_] / row_len;
      ck(cudaMemcpyAsync(nd, norm_src + so[p] / row_len, block_bytes / esz / row_len * sizeof(float),
                         cudaMemcpyDeviceToDevice, ps),
         "peer copy (norms)");
    }
    if (p != rank_) publish_one(ps, (2 * ch) * world_ + p, epoch, ready_remote(p, ch, chunk));
    else if (local_done) ck(cudaEventRecord(local_done, ps), "event");
    ck(cudaEventRecord(ev_out_[p], ps), "event");
  }
  for (int p = 0; p < world_; ++p)
    if (p != rank_ || local_done) ck(cudaStreamWaitEvent(copy, ev_out_[p], 0), "wait");
  if (probe) probe(ch, copy, false);
}


void PeerExchange::push_rows(cudaStream_t copy, int ch, int slot, const void* src, const int64_t* so,
                             const int64_t* ro, size_t segs, size_t seg_bytes, size_t row0_bytes,
                             size_t rows_bytes, uint32_t epoch, const float* norm_src,
                             size_t row_bytes) {
  if (norm_src && (ch != 0 || !local_norms_)) throw MoeError(MOE_EINVAL, "peer all-to-all: norms");
  if (slot < 0 || slot >= kFlagSlots) throw MoeError(MOE_EINVAL, "peer all-to-all: flag slot");
  ck(cudaEventRecord(ev_in_, copy), "event");
  if (probe) probe(ch, copy, true);
  for (int i = 1; i < world_; ++i) {  // own rows are written in place by the producing kernel
    const int p = (rank_ + i) % world_;
    cudaStream_t ps = pstreams_[p];
    ck(cudaStreamWaitEvent(ps, ev_in_, 0), "wait");
    // segs expert segments of seg_bytes each; rows [row0, row0 + rows) of every segment
    char* dst = static_cast<char*>(peer_bufs_[ch][p]) + ro[rank_] + row0_bytes;
    const char* s0 = static_cast<const char*>(src) + so[p] + row0_bytes;
    // segments split over the helper streams (more copy engines per destination)
    const size_t per = (segs + split_ - 1) / split_;
    for (int j = 1; j < split_; ++j) {
      const size_t s0j = per * j;
      if (s0j >= segs) break;
      cudaStream_t xs = xstreams_[p][j - 1];
      ck(cudaStreamWaitEvent(xs, ev_in_, 0), "wait");
      ck(cudaMemcpy2DAsync(dst + s0j * seg_bytes, seg_bytes, s0 + s0j * seg_bytes, seg_bytes, rows_bytes,
                           std::min(per, segs - s0j), cudaMemcpyDeviceToDevice, xs),
         "peer copy (rows)");
    }
    ck(cudaMemcpy2DAsync(dst, seg_bytes, s0, seg_bytes, rows_bytes, split_ > 1 ? std::min(per, segs) : segs,
                         cudaMemcpyDeviceToDevice, ps),
       "peer copy (rows)");
    for (int j = 1; j < split_; ++j) {
      if (per * j >= segs) break;
      ck(cudaEventRecord(xevents_[p][j - 1], xstreams_[p][j - 1]), "event");
      ck(cudaStreamWaitEvent(ps, xevents_[p][j - 1], 0), "wait");
    }
    if (norm_src) {  // the rows' norms travel with them (before the flag)
      const size_t npitch = seg_bytes / row_bytes * sizeof(float);
      float* nd = static_cast<float*>(peer_norms_[p]) + (ro[rank_] + row0_bytes) / row_bytes;
      const float* ns = norm_src + (so[p] + row0_bytes) / row_bytes;
      ck(cudaMemcpy2DAsync(nd, npitch, ns, npitch, rows_bytes / row_bytes * sizeof(float), segs,
                           cudaMemcpyDeviceToDevice, ps),
         "peer copy (norms)");
    }
    publish_one(ps, (2 * ch) * world_ + p, epoch, ready_remote(p, ch, slot));
    ck(cudaEventRecord(ev_out_[p], ps), "event");
  }
  for (int p = 0; p < world_; ++p)
    if (p != rank_) ck(cudaStreamWaitEvent(copy, ev_out_[p], 0), "wait");
  if (probe) probe(ch, copy, false);
}

FlagWait PeerExchange::ready_wait(int ch, int chunk, uint32_t epoch) const {
  FlagWait w;
  w.base = ready_local(ch, 0, chunk);
  w.stride = kFlagSlots;
  w.world = world_;
  w.rank = rank_;
  w.epoch = epoch;
  return w;
}

FlagWait PeerExchange::freed_wait(int ch, uint32_t epoch) const {
  FlagWait w;
  w.base = freed_local(ch, 0);
  w.stride = 1;
  w.world = world_;
  w.rank = rank_;
  w.epoch = epoch;
  return w;
}

void PeerExchange::signal_ready(cudaStream_t st, int ch, int chunk, uint32_t epoch) {
  std::vector<uint32_t*> dsts;
  for (int p = 0; p < world_; ++p)
    if (p != rank_) dsts.push_back(ready_remote(p, ch, chunk));
  publish(st, 2 * ch, epoch, dsts);  // stage column `rank` of slot 2ch: unused by the push streams
}

void PeerExchange::signal_freed(cudaStream_t st, int ch, uint32_t epoch) {
  std::vector<uint32_t*> dsts;
  for (int p = 0; p < world_; ++p)
    if (p != rank_) dsts.push_back(freed_remote(p, ch));
  publish(st, 2 * ch + 1, epoch, dsts);
}

}  // namespace moe
