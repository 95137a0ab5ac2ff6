// k_fiber_f64.cu -- fp64-storage instantiations of the fiber-block pass
// (k_fiber.cuh) and the engine-facing entry points (fiber_types.cuh).
#include "k_fiber.cuh"

int fiber_pass_launch_f32(const FiberLaunch& L, unsigned mask, cudaStream_t st);
int fiber_xi_extract_f32(const FiberLaunch& L, unsigned mask, cudaStream_t st);

int fiber_xi_extract(const FiberLaunch& L, cudaStream_t st) {
  const unsigned mask = fiber_pass_blocks(L.g, L.dtype);
  if (!mask) return 0;
  return L.dtype == 0 ? fb_extract_t<double>(L, mask, st) : fiber_xi_extract_f32(L, mask, st);
}

unsigned fiber_pass_blocks(const Geom& g, int dtype) {
  if (const char* env = getenv("RTCUR_FIBER_PASS"))
    if (env[0] == '0') return 0u;
  unsigned mask = 0;
  for (int b = 1; b < g.nblk; ++b)
    if (fb_block_ok(g, b, dtype)) mask |= 1u << b;
  // the core (bit 0) joins the error pass only
  const char* ec = getenv("RTCUR_FIBER_CORE");
  if (!(ec && ec[0] == '0') && fb_block_ok(g, 0, dtype)) mask |= 1u;
  return mask;
}

int fiber_pass_launch(const FiberLaunch& L, cudaStream_t st) {
  const unsigned mask = L.mask ? L.mask : fiber_pass_blocks(L.g, L.dtype);
  if (!mask) return 0;
  return L.dtype == 0 ? fb_launch_t<double>(L, mask, st) : fiber_pass_launch_f32(L, mask, st);
}
