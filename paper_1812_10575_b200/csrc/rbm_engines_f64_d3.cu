// rbm_engines_f64_d3.cu -- double d=3 instantiations of the per-config step
// engines (one translation unit per (dtype, d) so the build compiles in parallel).
#include "rbm_host.cuh"

namespace rbmhost {

EngineBase* make_engine_f64_d3(uint32_t kernel, uint32_t integ) {
  return make_for_kernel<double, 3>(kernel, integ);
}

}  // namespace rbmhost
