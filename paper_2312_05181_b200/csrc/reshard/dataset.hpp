// reshard/dataset.hpp — dataset index repartitioning (SPEC tensor-store module,
// SPEC.md:336-362, 378-383): epoch shuffle, per-rank positions after a DP change, and the
// sample location lookup, with the per-rank gather/scan/compaction done on the GPU (K5).
#pragma once

#include <cstdint>
#include <vector>

#include "reshard/executor.hpp"

namespace reshard {

// shuffle_epoch: Fisher-Yates, i from N-1 down to 1, j =
// next_below(i+1) of splitmix64 seeded (seed XOR epoch).  Host, O(N) sequential.
void shuffle_epoch(uint64_t n, uint64_t seed, uint64_t epoch, uint64_t* perm);

// repartition: batches i >= at_step; new rank d owns positions
// [i*B + d*B/D', i*B + (d+1)*B/D') of batch i, clipped at N for a trailing partial batch.
// Errors: InvalidJobConfig (B or D' zero), IndivisibleBatch, StepBeyondEpoch.
void repartition_check(uint64_t n, uint64_t B, uint64_t at_step, uint64_t new_dp);
uint64_t repartition_count(uint64_t n, uint64_t B, uint64_t at_step, uint64_t new_dp, uint64_t rank);
uint64_t repartition_position(uint64_t n, uint64_t B, uint64_t at_step, uint64_t new_dp, uint64_t rank, uint64_t k);

// Device-resident dataset index.  samples: N x {file, offset, length} (u64 each), packed
// 24-byte records as the reference stores them (entry_bytes 0 or 24) or the padded 32-byte
// device layout written by dataset_index_pad (entry_bytes 32: one record per 32-byte
// sector, so a random gather never straddles a DRAM line); file_class: the calling rank's
// locator class per file, 0 local / 1 peer / 2 remote (priority order of SPEC.md:357).
struct DatasetIndexView {
  const uint64_t* perm;
  const uint64_t* samples;
  const uint8_t* file_class;
  uint64_t n;
  uint64_t entry_bytes = 24;
};
// Packed -> padded index records on the device (one streaming pass; padded: 32 n bytes,
// 16-byte aligned).  The outputs of repartition are identical for either layout.
Timing dataset_index_pad(Context& ctx, int gpu, const uint64_t* packed, uint64_t* padded, uint64_t n);
// Outputs of one rank (device).  For the rank's k-th remaining sample: pos[k],
// ent[3k..3k+2] = samples[perm[pos[k]]], boff[k] = exclusive prefix sum of lengths (the
// sample's offset in the rank's read buffer); queue[c] lists the k with locator class c in
// increasing k, qcount[c] their number (written by the kernel).
struct PartitionOut {
  uint64_t* pos;
  uint64_t* ent;
  uint64_t* boff;
  uint32_t* queue[3];
  uint64_t* qcount;
};

// Host copies of one rank's outputs (pinned memory for full PCIe rate), same layout as
// PartitionOut; queue[c] receives exactly qcount[c] entries.
struct PartitionHost {
  uint64_t* pos;
  uint64_t* ent;
  uint64_t* boff;
  uint32_t* queue[3];
  uint64_t* qcount;
};

// K8: the same permutation as shuffle_epoch, computed on the GPU (bit-identical; parallel
// Fisher-Yates by deterministic reservations in windowed rounds, the reservations packed into
// the high words of perm while it runs).  perm: device, n entries (n < 2^32); scratch:
// shuffle_scratch_bytes(n) of device memory (the carried-iteration lists).  Timing.tiles = rounds.
uint64_t shuffle_scratch_bytes(uint64_t n);
Timing shuffle_epoch_device(Context& ctx, int gpu, uint64_t n, uint64_t seed, uint64_t epoch, uint64_t* perm,
                            void* scratch);

// Host -> device upload of an index (perm, packed samples) on the GPU's stream; with
// `padded` non-null the packed records are also rewritten there (dataset_index_pad).
// Timing.ms: event time of the whole upload; bytes: H2D bytes.
Timing dataset_index_upload(Context& ctx, int gpu, const uint64_t* host_perm, const uint64_t* host_samples,
                            uint64_t n, uint64_t* perm, uint64_t* samples, uint64_t* padded);

uint64_t repartition_scratch_bytes(uint64_t count);
// K5 for one rank: gather pass, tile scan, finalize (three launches; RESHARD_K5=lookback:
// one).  `scratch` (repartition_scratch_bytes) must be device memory.  Timing.main_ms is
// the gather pass alone.
Timing repartition_device(Context& ctx, int gpu, const DatasetIndexView& idx, uint64_t B, uint64_t at_step,
                          uint64_t new_dp, uint64_t rank, const PartitionOut& out, void* scratch);
// Several ranks' K5 on one GPU (a GPU hosting several new DP ranks; bench config 5 at N = 1).
// Default: all ranks in one launch per pass (multi-rank gather / tile scan / finalize kernels
// over a device rank table).  RESHARD_K5_FUSE=0: the gather passes one after another on a
// high-priority stream, each rank's tile scan + finalize on a low-priority second stream.
// Per job its own file_class (locator classes differ per rank), outputs and scratch.
// Timing.ms: batch start -> last finalize; main_ms: the gather pass(es); per_job (optional):
// tiles / bytes, and unfused each rank's gather-pass time in ms / main_ms.
struct RepartJob {
  uint64_t at_step, new_dp, rank;
  const uint8_t* file_class;
  PartitionOut out;
  void* scratch;
};
Timing repartition_batch_device(Context& ctx, int gpu, const DatasetIndexView& idx, uint64_t B, const RepartJob* jobs,
                                size_t n, std::vector<Timing>* per_job);
// repartition_device, then the rank's outputs device -> host (exactly count entries of
// pos / ent / boff and qcount[c] of each queue) on the same stream.  Timing.ms: kernels +
// D2H (events), main_ms: the gather pass, bytes: D2H bytes.
Timing repartition_to_host(Context& ctx, int gpu, const DatasetIndexView& idx, uint64_t B, uint64_t at_step,
                           uint64_t new_dp, uint64_t rank, const PartitionOut& out, void* scratch,
                           const PartitionHost& host);
// Diagnostic: best-of-`reps` time of K5's perm + entry gathers for the rank's positions
// plus all 44 output bytes per sample written coalesced, no scan (RESHARD_PROBE=read:
// nothing written) — the floor for any kernel that must produce the partition.
Timing repartition_gather_probe(Context& ctx, int gpu, const DatasetIndexView& idx, uint64_t B, uint64_t at_step,
                                uint64_t new_dp, uint64_t rank, int reps);

}  // namespace reshard
