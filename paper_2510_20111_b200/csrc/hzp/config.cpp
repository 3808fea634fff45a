// Partition layer: validation and process-group construction.
// Behaviour matches /root/reference/proj/src/config.cpp:36-170 (checked
// bit-exactly against tests/golden/layout.json by tests/test_host.py).
#include "hzp/config.hpp"

#include <sstream>

namespace hzp {

const char* to_string(GroupKind kind) {
  static const char* const names[] = {"Z1", "Z2", "Z3", "DZP-replica", "PP", "CP", "TP"};
  const int i = static_cast<int>(kind);
  return (i >= 0 && i < 7) ? names[i] : "?";
}

namespace {

[[noreturn]] void fail(ValidationError::Code code, const std::string& msg) {
  throw ValidationError(code, msg);
}

bool spans(const std::vector<int>& ranks, const Topology& topo) {
  for (int r : ranks)
    if (topo.node_of(r) != topo.node_of(ranks.front())) return true;
  return false;
}

ProcessGroup make_group(GroupKind kind, std::vector<int> ranks, const Topology& topo) {
  ProcessGroup g;
  g.kind = kind;
  g.spans_nodes = !ranks.empty() && spans(ranks, topo);
  g.ranks = std::move(ranks);
  return g;
}

}  // namespace

ValidatedConfig validate_config(const ModelSpec& spec, const ParallelConfig& cfg,
                                const Topology& topo) {
  using C = ValidationError::Code;
  if (spec.num_layers < 0 || spec.params_per_layer < 0 || spec.embedding_params < 0)
    fail(C::BadField, "negative model field");
  if (spec.total_params() <= 0) fail(C::EmptyModel, "model has zero parameters");
  if (spec.num_microbatches < 1) fail(C::BadField, "num_microbatches must be >= 1");
  if (spec.seq_len < 1) fail(C::BadField, "seq_len must be >= 1");
  if (spec.micro_batch_size < 1) fail(C::BadField, "micro_batch_size must be >= 1");
  if (cfg.dp < 1 || cfg.pp < 1 || cfg.vpp < 1 || cfg.cp < 1 || cfg.tp < 1)
    fail(C::BadField, "parallel degrees must be >= 1");
  const std::pair<int, const char*> zs[] = {{cfg.z1, "z1"}, {cfg.z2, "z2"}, {cfg.z3, "z3"}};
  for (const auto& [z, name] : zs) {
    if (z < 1 || cfg.dp % z != 0) {
      std::ostringstream m;
      m << name << "=" << z << " does not divide dp=" << cfg.dp;
      fail(C::NonDivisible, m.str());
    }
  }
  if (cfg.vpp > 1 && cfg.pp == 1) fail(C::BadField, "vpp > 1 requires pp > 1");
  if (topo.num_nodes < 1 || topo.ranks_per_node < 1)
    fail(C::BadField, "topology counts must be >= 1");
  if (!(topo.inter_bw > 0 && topo.intra_bw >= topo.inter_bw))
    fail(C::BadField, "bandwidths must satisfy intra_bw >= inter_bw > 0");
  if (topo.intra_latency < 0 || topo.inter_latency < 0)
    fail(C::BadField, "latencies must be >= 0");
  const std::int64_t world = std::int64_t(cfg.dp) * cfg.pp * cfg.cp * cfg.tp;
  if (world != topo.total_ranks()) {
    std::ostringstream m;
    m << "dp*pp*cp*tp = " << world << " but topology has " << topo.total_ranks() << " ranks";
    fail(C::NonDivisible, m.str());
  }
  ValidatedConfig v;
  v.model = spec;
  v.parallel = cfg;
  v.topo = topo;
  v.total_params = spec.total_params();
  v.total_ranks = topo.total_ranks();
  const int outer = cfg.pp * cfg.cp * cfg.tp;
  v.groups_per_kind[GroupKind::Z1] = outer * (cfg.dp / cfg.z1);
  v.groups_per_kind[GroupKind::Z2] = outer * (cfg.dp / cfg.z2);
  v.groups_per_kind[GroupKind::Z3] = outer * (cfg.dp / cfg.z3);
  v.groups_per_kind[GroupKind::DzpReplica] = outer * cfg.z2;
  v.groups_per_kind[GroupKind::PP] = v.total_ranks / cfg.pp;
  v.groups_per_kind[GroupKind::CP] = v.total_ranks / cfg.cp;
  v.groups_per_kind[GroupKind::TP] = v.total_ranks / cfg.tp;
  return v;
}

GroupMap build_process_groups(const ParallelConfig& cfg, const Topology& topo) {
  GroupMap map;
  const int outer = cfg.pp * cfg.cp * cfg.tp;
  // dp is the fastest-varying rank dimension: every Z group is a contiguous
  // block [base + k*z, base + (k+1)*z) inside one dp-sized block.
  const std::pair<GroupKind, int> contiguous[] = {
      {GroupKind::Z1, cfg.z1}, {GroupKind::Z2, cfg.z2}, {GroupKind::Z3, cfg.z3}};
  for (const auto& [kind, z] : contiguous) {
    auto& list = map[kind];
    for (int blk = 0; blk < outer; ++blk)
      for (int k = 0; k < cfg.dp / z; ++k) {
        std::vector<int> r(z);
        for (int i = 0; i < z; ++i) r[i] = blk * cfg.dp + k * z + i;
        list.push_back(make_group(kind, std::move(r), topo));
      }
  }
  // DZP replicas: position i of every Z2 block, stride z2.
  auto& dzp = map[GroupKind::DzpReplica];
  for (int blk = 0; blk < outer; ++blk)
    for (int i = 0; i < cfg.z2; ++i) {
      std::vector<int> r(cfg.dp / cfg.z2);
      for (int b = 0; b < cfg.dp / cfg.z2; ++b) r[b] = blk * cfg.dp + b * cfg.z2 + i;
      dzp.push_back(make_group(GroupKind::DzpReplica, std::move(r), topo));
    }
  // Outer dimensions: rank = ((pp_i * cp + cp_i) * tp + tp_i) * dp + dp_i.
  const int world = cfg.dp * outer;
  const std::tuple<GroupKind, int, int> strided[] = {
      {GroupKind::PP, cfg.pp, cfg.dp * cfg.tp * cfg.cp},
      {GroupKind::CP, cfg.cp, cfg.dp * cfg.tp},
      {GroupKind::TP, cfg.tp, cfg.dp}};
  for (const auto& [kind, deg, stride] : strided) {
    std::vector<char> taken(world, 0);
    auto& list = map[kind];
    for (int r0 = 0; r0 < world; ++r0) {
      if (taken[r0]) continue;
      std::vector<int> r(deg);
      for (int k = 0; k < deg; ++k) {
        r[k] = r0 + k * stride;
        if (r[k] < world) taken[r[k]] = 1;
      }
      list.push_back(make_group(kind, std::move(r), topo));
    }
  }
  return map;
}

}  // namespace hzp
