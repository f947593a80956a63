// launch_overhead.cu -- what a short persistent tcgen05 kernel pays before any
// work: back-to-back launches of otherwise empty kernels, CUDA-event timed per
// launch, in a plain stream and captured in a CUDA graph (with and without
// programmatic dependent launch), adding one ingredient at a time:
//   empty          320 threads
//   +smem          + 82 KB dynamic shared memory
//   +mbar          + mbarrier init + fence + __syncthreads
//   +tmem          + tcgen05.alloc / relinquish / dealloc (128 columns)
//   +param         + a 2 KB __grid_constant__ parameter block read by thread 0
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o lo tests/launch_overhead.cu && ./lo
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

struct Big {
  uint32_t w[512];
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

template <int LEVEL>
__global__ void __launch_bounds__(320, 1) k_over(const __grid_constant__ Big p, uint32_t* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar[8];
  __shared__ uint32_t tslot;
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (LEVEL >= 2) {
    if (threadIdx.x == 0) {
      for (int i = 0; i < 8; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[i])));
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
  }
  if (LEVEL >= 3 && threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (LEVEL >= 4 && threadIdx.x == 0 && p.w[blockIdx.x & 511] == 0xdeadbeef) sink[blockIdx.x] = sm[threadIdx.x];
  __syncthreads();
  if (LEVEL >= 3 && threadIdx.x < 32)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tslot));
}

template <int LEVEL>
float run(int ctas, size_t smem, bool graph, bool pdl) {
  Big b{};
  uint32_t* sink;
  cudaMalloc(&sink, 4096);
  auto k = k_over<LEVEL>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  const int reps = 200;
  auto launch = [&] {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(ctas);
    cfg.blockDim = dim3(320);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    cudaLaunchKernelEx(&cfg, k, b, sink);
  };
  cudaGraphExec_t ge = nullptr;
  if (graph) {
    cudaGraph_t g;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
    for (int i = 0; i < reps; ++i) launch();
    cudaStreamEndCapture(s, &g);
    cudaGraphInstantiate(&ge, g, 0);
  }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e9f;
  for (int t = 0; t < 3; ++t) {
    cudaEventRecord(e0, s);
    if (graph) cudaGraphLaunch(ge, s);
    else for (int i = 0; i < reps; ++i) launch();
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) std::printf("error %s\n", cudaGetErrorString(err));
  cudaFree(sink);
  return best * 1000.f / reps;
}

int main() {
  const char* names[] = {"empty", "+smem", "+mbar", "+tmem", "+param"};
  std::printf("{\"us_per_launch\": {\n");
  for (int ctas : {64, 148}) {
    for (int mode = 0; mode < 3; ++mode) {
      const bool graph = mode > 0, pdl = mode == 2;
      float t[5] = {run<0>(ctas, 0, graph, pdl), run<0>(ctas, 82 * 1024, graph, pdl), run<2>(ctas, 82 * 1024, graph, pdl),
                    run<3>(ctas, 82 * 1024, graph, pdl), run<4>(ctas, 82 * 1024, graph, pdl)};
      std::printf("  \"ctas=%d %s\": {", ctas, mode == 0 ? "stream" : mode == 1 ? "graph" : "graph+pdl");
      for (int i = 0; i < 5; ++i) std::printf("%s\"%s\": %.2f", i ? ", " : "", names[i], t[i]);
      std::printf("}%s\n", ctas == 148 && mode == 2 ? "" : ",");
    }
  }
  std::printf("}}\n");
  return 0;
}
