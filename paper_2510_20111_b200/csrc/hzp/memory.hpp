// Drop-in static-memory ledger of the B200 build (reference:
// /root/reference/proj/include/hzp/memory.hpp:18-50, src/memory.cpp:13-42).
// Same names, types and results; feeds memory_trace (sched.hpp).  The
// sharding-plan search (memory.hpp:52-72) stays out of scope (control plane).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>

#include "hzp/config.hpp"

namespace hzp {

// Per-rank bytes of the mixed-precision training states.
struct MemoryLedger {
  std::int64_t params_bf16 = 0;
  std::int64_t grads_fp32 = 0;
  std::int64_t replica_fp32 = 0;
  std::int64_t momentum_fp32 = 0;
  std::int64_t variance_fp32 = 0;
  std::int64_t total_static = 0;
};

class MemoryError : public std::runtime_error {
 public:
  enum class Code { ReplicaExceedsWorld, NoFeasibleConfig };
  MemoryError(Code code, const std::string& what) : std::runtime_error(what), code_(code) {}
  Code code() const { return code_; }

 private:
  Code code_;
};

// 18 bytes per element of the shard: 2 (bf16 param) + 4 (fp32 grad) + 12
// (master, m, v), all sharded dp / z / (z1, z2, z3) ways.
std::int64_t mem_zero3(std::int64_t n, int dp);
std::int64_t mem_zp(std::int64_t n, int z, int dp);  // throws ReplicaExceedsWorld if z > dp
std::int64_t mem_hzp(std::int64_t n, int z1, int z2, int z3);

MemoryLedger ledger(const ModelSpec& spec, const ParallelConfig& cfg);

}  // namespace hzp
