// Pipeline schedule object over the scheduler's slot orders (pipeline.hpp).
#include "hzp/pipeline.hpp"

namespace hzp {

PipeVariant parse_variant(const std::string& name) {
  if (name == "1f1b") return PipeVariant::OneFOneB;
  if (name == "interleaved") return PipeVariant::Interleaved;
  throw PipeError(PipeError::Code::UnsupportedVariant, "unknown pipeline variant: " + name);
}

PipeSchedule build_schedule(int pp, int vpp, int microbatches, PipeVariant variant) {
  using C = PipeError::Code;
  if (pp < 1 || vpp < 1 || microbatches < 1) throw PipeError(C::BadShape, "degrees must be >= 1");
  if (vpp > 1 && variant != PipeVariant::Interleaved)
    throw PipeError(C::BadShape, "vpp > 1 requires the interleaved variant");
  if (variant == PipeVariant::Interleaved && vpp > 1 && microbatches % pp != 0)
    throw PipeError(C::BadShape, "interleaved schedule needs microbatches divisible by pp");
  PipeSchedule s;
  s.pp = pp;
  s.vpp = vpp;
  s.microbatches = microbatches;
  s.variant = variant;
  for (int rank = 0; rank < pp; ++rank) {
    std::vector<ScheduleSlot> slots = pipeline_order(pp, vpp, microbatches, rank);
    // leading forwards are the warm-up, trailing backwards the cool-down
    std::vector<Phase> ph(slots.size(), Phase::Steady);
    size_t i = 0, j = slots.size();
    for (; i < j && slots[i].pass == Pass::Forward; ++i) ph[i] = Phase::Warmup;
    for (; j > i && slots[j - 1].pass == Pass::Backward; --j) ph[j - 1] = Phase::Cooldown;
    s.per_rank.push_back(std::move(slots));
    s.phases.push_back(std::move(ph));
  }
  return s;
}

ReuseReport apply_reuse(const PipeSchedule& schedule, TaskGraph& graph) {
  using C = PipeError::Code;
  if (graph.rank < 0 || graph.rank >= static_cast<int>(schedule.per_rank.size()))
    throw PipeError(C::ScheduleGraphMismatch, "graph rank outside schedule");
  const std::vector<ScheduleSlot>& want = schedule.per_rank[graph.rank];
  const std::vector<ScheduleSlot> have = graph_slots(graph);
  bool same = have.size() == want.size();
  for (size_t i = 0; same && i < have.size(); ++i)
    same = have[i].pass == want[i].pass && have[i].microbatch == want[i].microbatch &&
           have[i].virtual_stage == want[i].virtual_stage;
  if (!same) throw PipeError(C::ScheduleGraphMismatch, "task graph was not built for this schedule");
  return apply_reuse(graph);
}

void recompute_rule(TaskGraph& graph, bool recompute) {
  if (recompute) recompute_rule(graph);
}

}  // namespace hzp
