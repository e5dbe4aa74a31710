// TEST INFRASTRUCTURE (oracle only). Declarations shared by ref_shim.cpp and
// ref_capi.cpp; see ref_shim.cpp for what each shim restates.
#ifndef BO_REF_SHIM_HPP_
#define BO_REF_SHIM_HPP_

#include <cstdint>
#include <string>
#include <vector>

#include "bertopt/model.hpp"

namespace refshim {

// One micro-batch worth of synthetic per-parameter gradients G_p (model
// order) and the first-use order the synthetic forward consumes them in.
struct SynthMicro {
  std::vector<std::vector<float>> G;
  std::vector<int> first_use_order;
};

struct ModelSpec {
  std::vector<std::string> names;
  std::vector<std::vector<int64_t>> shapes;
  std::vector<int> init;  // 0 randn(σ=0.02), 1 ones, 2 zeros (model.cpp:132-174)
};

void register_micro(int64_t handle, const SynthMicro* s);
void unregister_micro(int64_t handle);
bertopt::Model build_model_from_spec(const ModelSpec& spec, uint64_t seed);

}  // namespace refshim

#endif  // BO_REF_SHIM_HPP_
