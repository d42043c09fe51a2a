// rbm_engines_f64.cu -- double instantiations of the per-config step engines.
#include "rbm_host.cuh"

namespace rbmhost {

template <typename T>
EngineBase* make_for_dim(uint32_t d, uint32_t kernel, uint32_t integ) {
  switch (d) {
    case 1: return make_for_kernel<T, 1>(kernel, integ);
    case 2: return make_for_kernel<T, 2>(kernel, integ);
    case 3: return make_for_kernel<T, 3>(kernel, integ);
  }
  return nullptr;
}

EngineBase* make_engine_f64(const rbm_config& k) {
  return make_for_dim<double>(k.d, k.kernel, k.integrator);
}

}  // namespace rbmhost
