// rbm_engines_f64_d2.cu -- double d=2 instantiations of the per-config step
// engines (one translation unit per (dtype, d) so the build compiles in parallel).
#include "rbm_host.cuh"

namespace rbmhost {

EngineBase* make_engine_f64_d2(uint32_t kernel, uint32_t integ) {
  return make_for_kernel<double, 2>(kernel, integ);
}

}  // namespace rbmhost
