// k_fiber_f32.cu -- fp32-storage instantiations of the fiber-block pass (k_fiber.cuh).
#include "k_fiber.cuh"

int fiber_pass_launch_f32(const FiberLaunch& L, unsigned mask, cudaStream_t st) {
  return fb_launch_t<float>(L, mask, st);
}

int fiber_xi_extract_f32(const FiberLaunch& L, unsigned mask, cudaStream_t st) {
  return fb_extract_t<float>(L, mask, st);
}
