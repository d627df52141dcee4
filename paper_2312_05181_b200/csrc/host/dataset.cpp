// Host side of the dataset repartitioner: shuffle and the closed-form
// rank positions.  The per-sample gather / scan / compaction runs on the GPU (cuda/dataset.cu).
#include "reshard/dataset.hpp"

#include <algorithm>
#include <numeric>

namespace reshard {

void shuffle_epoch(uint64_t n, uint64_t seed, uint64_t epoch, uint64_t* perm) {
  std::iota(perm, perm + n, uint64_t{0});
  SplitMix64 rng(seed ^ epoch);
  for (uint64_t i = n; i > 1; --i) std::swap(perm[i - 1], perm[rng.next_below(i)]);
}

void repartition_check(uint64_t n, uint64_t B, uint64_t at_step, uint64_t dp) {
  if (B == 0 || dp == 0) raise(Errc::InvalidJobConfig, "global batch and new_dp must be positive");
  if (B % dp) raise(Errc::IndivisibleBatch, "B=" + std::to_string(B) + " not divisible by new_dp=" + std::to_string(dp));
  const uint64_t batches = (n + B - 1) / B;
  if (at_step > batches) raise(Errc::StepBeyondEpoch, "at_step " + std::to_string(at_step) + " > " + std::to_string(batches) + " batches");
}

uint64_t repartition_count(uint64_t n, uint64_t B, uint64_t at_step, uint64_t dp, uint64_t rank) {
  repartition_check(n, B, at_step, dp);
  if (rank >= dp) raise(Errc::IndexOutOfRange, "rank " + std::to_string(rank) + " >= new_dp");
  const uint64_t b = B / dp, full = n / B;
  uint64_t c = full > at_step ? (full - at_step) * b : 0;
  if (n % B && at_step <= full) {  // trailing partial batch
    const uint64_t lo = full * B + rank * b;
    if (lo < n) c += std::min(b, n - lo);
  }
  return c;
}

uint64_t repartition_position(uint64_t n, uint64_t B, uint64_t at_step, uint64_t dp, uint64_t rank, uint64_t k) {
  const uint64_t cnt = repartition_count(n, B, at_step, dp, rank);
  if (k >= cnt) raise(Errc::IndexOutOfRange, "k beyond the rank's partition");
  const uint64_t b = B / dp, full = n / B;
  const uint64_t in_full = full > at_step ? (full - at_step) * b : 0;
  if (k < in_full) return (at_step + k / b) * B + rank * b + k % b;
  return full * B + rank * b + (k - in_full);
}

}  // namespace reshard
