// rbm_engines_f32_d1.cu -- float d=1 instantiations of the per-config step
// engines (one translation unit per (dtype, d) so the build compiles in parallel).
#include "rbm_host.cuh"

namespace rbmhost {

EngineBase* make_engine_f32_d1(uint32_t kernel, uint32_t integ) {
  return make_for_kernel<float, 1>(kernel, integ);
}

}  // namespace rbmhost
