// Static-memory ledger (memory.hpp; reference src/memory.cpp:13-42).
#include "hzp/memory.hpp"

namespace hzp {

std::int64_t mem_zero3(std::int64_t n, int dp) { return mem_hzp(n, dp, dp, dp); }

std::int64_t mem_zp(std::int64_t n, int z, int dp) {
  if (z > dp)
    throw MemoryError(MemoryError::Code::ReplicaExceedsWorld,
                      "replica group size " + std::to_string(z) + " exceeds dp world " + std::to_string(dp));
  return mem_hzp(n, z, z, z);
}

std::int64_t mem_hzp(std::int64_t n, int z1, int z2, int z3) {
  // 12 B optimizer state / z1 + 4 B gradient / z2 + 2 B working copy / z3
  return 12 * shard_elems(n, z1) + 4 * shard_elems(n, z2) + 2 * shard_elems(n, z3);
}

MemoryLedger ledger(const ModelSpec& spec, const ParallelConfig& cfg) {
  const std::int64_t n = spec.total_params();
  const std::int64_t s1 = shard_elems(n, cfg.z1);
  MemoryLedger m;
  m.params_bf16 = 2 * shard_elems(n, cfg.z3);
  m.grads_fp32 = 4 * shard_elems(n, cfg.z2);
  m.replica_fp32 = 4 * s1;
  m.momentum_fp32 = 4 * s1;
  m.variance_fp32 = 4 * s1;
  m.total_static = m.params_bf16 + m.grads_fp32 + m.replica_fp32 + m.momentum_fp32 + m.variance_fp32;
  return m;
}

}  // namespace hzp
