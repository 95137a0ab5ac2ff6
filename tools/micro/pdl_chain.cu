// Micro-benchmark: a chain of short dependent kernels replayed as a CUDA graph, with and
// without programmatic dependent launch (griddepcontrol.wait at the top of every kernel,
// launch_dependents right after).  Measured on B200: 5.35 vs 5.13 us per kernel for a 4.07 us
// body, 11.50 vs 11.27 for a 10.18 us body -- a kernel boundary inside a graph costs ~1.3 us
// and PDL recovers ~0.25 us of it, so the iteration's time is in the kernels, not between them.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pdl_chain pdl_chain.cu
#include <cstdio>
#include <cuda_runtime.h>

template <bool PDL>
__global__ void k_step(const double* __restrict__ in, double* __restrict__ out, int n, long long spin) {
  extern __shared__ double sm[];
  if (PDL) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  }
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  double v = i < n ? in[i] : 0.0;
  const long long t0 = clock64();
  while (clock64() - t0 < spin) v = v * 1.0000001 + 1e-9;
  sm[threadIdx.x] = v;
  __syncthreads();
  if (i < n) out[i] = sm[threadIdx.x ^ 1];
}

template <bool PDL>
static float run(int nk, int grid, int threads, int smem, long long spin, cudaStream_t st, double* a, double* b, int n) {
  cudaError_t ae = cudaFuncSetAttribute(k_step<PDL>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem > 0 ? smem : 1024);
  if (ae != cudaSuccess) { printf("attr: %s\n", cudaGetErrorString(ae)); return -1.f; }
  printf("[run PDL=%d grid=%d]\n", (int)PDL, grid);
  cudaGraph_t g = nullptr;
  cudaGraphExec_t ex = nullptr;
  cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
  for (int k = 0; k < nk; ++k) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = PDL ? 1 : 0;
    const double* in = (k & 1) ? b : a;
    double* out = (k & 1) ? a : b;
    cudaError_t le = cudaLaunchKernelEx(&cfg, k_step<PDL>, in, out, n, spin);
    if (le != cudaSuccess) { printf("launch %d: %s\n", k, cudaGetErrorString(le)); break; }
  }
  cudaError_t e = cudaStreamEndCapture(st, &g);
  if (e != cudaSuccess || g == nullptr) { printf("end capture: %s\n", cudaGetErrorString(e)); cudaGetLastError(); return -1.f; }
  printf("[captured]\n");
  e = cudaGraphInstantiate(&ex, g, 0);
  printf("[instantiated %d]\n", (int)e);
  if (e != cudaSuccess) { printf("instantiate: %s\n", cudaGetErrorString(e)); return -1.f; }
  for (int i = 0; i < 5; ++i) cudaGraphLaunch(ex, st);
  cudaStreamSynchronize(st);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, st);
  const int reps = 50;
  for (int i = 0; i < reps; ++i) cudaGraphLaunch(ex, st);
  cudaEventRecord(e1, st);
  cudaStreamSynchronize(st);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  e = cudaGetLastError();
  if (e != cudaSuccess) printf("error: %s\n", cudaGetErrorString(e));
  cudaGraphExecDestroy(ex);
  cudaGraphDestroy(g);
  return ms * 1e3f / reps / nk;
}

int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  cudaStream_t st;
  if (cudaStreamCreate(&st) != cudaSuccess) { printf("no device\n"); return 1; }
  const int n = 296 * 384;
  double *a, *b;
  cudaMalloc(&a, n * 8);
  cudaMalloc(&b, n * 8);
  cudaMemset(a, 0, n * 8);
  cudaMemset(b, 0, n * 8);
  struct { int grid, threads, smem; long long spin; const char* what; } cases[] = {
      {296, 384, 100 * 1024, 8000, "296 CTAs x 384 thr, 100 KB smem, ~4 us body"},
      {296, 384, 100 * 1024, 20000, "296 CTAs x 384 thr, 100 KB smem, ~10 us body"},
  };
  for (auto& c : cases) {
    const float t0 = run<false>(18, c.grid, c.threads, c.smem, c.spin, st, a, b, n);
    const float t1 = run<true>(18, c.grid, c.threads, c.smem, c.spin, st, a, b, n);
    printf("%-50s plain %.2f us/kernel, PDL %.2f us/kernel (body %.2f us)\n", c.what, t0, t1, c.spin / 1965.0);
  }
  return 0;
}
