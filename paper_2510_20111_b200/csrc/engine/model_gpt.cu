// GPT decoder model (filled in by a later milestone).
#include <stdexcept>

#include "engine/model.hpp"

namespace hzp {
std::unique_ptr<Model> make_gpt_model(const ModelConfig&) {
  throw std::invalid_argument("GPT model not built yet");
}
}  // namespace hzp
