// tc_align.cu -- derived from tc_peak.cu: tcgen05.mma kind::i8 M=128 throughput
// with the conv kernel's operand layout (64-byte-swizzled K-major rows, SBO = 8
// rows x 64 B, K steps as 32-byte start advances) and the A start shifted by
// 0..7 rows (a 3x3 tap is a row shift of the staged tile), N in {64, 128}.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tc_align tests/tc_align.cu && ./tc_align
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

template <int KIND>
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  if (KIND == 0)
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
                 "l"(a), "l"(b), "r"(idesc), "r"(acc));
  else
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
                 "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

template <int KIND>
__global__ void __launch_bounds__(128, 1) k_peak(int iters, int n, unsigned long long* cycles, int shift) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < 64 * 1024; i += blockDim.x) sm[i] = static_cast<uint8_t>(i * 7);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tslot;
  // 64B-swizzled K-major descriptors (layout type 4), SBO = 512 B, LBO unused (16)
  auto desc = [](uint32_t addr, uint32_t) {
    const uint64_t hi = ((512u >> 4) & 0x3FFF) | (1u << 14) | (4u << 29);
    return (hi << 32) | (((addr >> 4) & 0x3FFF) | (((16u >> 4) & 0x3FFF) << 16));
  };
  const uint32_t a0 = smem_u32(sm) + static_cast<uint32_t>(shift) * 64, b0 = smem_u32(sm + 32768);
  uint32_t idesc = KIND == 0 ? ((2u << 4) | (1u << 7) | (1u << 10)) : ((1u << 4) | (1u << 7) | (1u << 10));
  idesc |= static_cast<uint32_t>(n >> 3) << 17;
  idesc |= static_cast<uint32_t>(128 >> 4) << 24;
  unsigned long long t0 = 0;
  if (threadIdx.x == 0) {
    const uint64_t ad = desc(a0, 2048), bd = desc(b0, static_cast<uint32_t>(n) * 16);
    t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      // 2 accumulators alternate so consecutive MMAs are independent
      mma<KIND>(tmem + (i & 1) * 256, ad, bd, idesc, i > 1 ? 1u : 0u);
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar))
                 : "memory");
    asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(
                     smem_u32(&bar))
                 : "memory");
    cycles[blockIdx.x] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int KIND>
void run(int n, int sms, int shift) {
  const int iters = 20000;
  unsigned long long* cyc;
  cudaMalloc(&cyc, sms * sizeof(unsigned long long));
  cudaFuncSetAttribute(k_peak<KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024 + 1024);
  k_peak<KIND><<<sms, 128, 64 * 1024 + 1024>>>(100, n, cyc, shift);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k_peak<KIND><<<sms, 128, 64 * 1024 + 1024>>>(iters, n, cyc, shift);
  cudaEventRecord(e1);
  cudaError_t err = cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long h[1024];
  cudaMemcpy(h, cyc, sms * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  double kbytes = KIND == 0 ? 32 : 16;  // K elements per instruction: 32 int8 or 16 bf16
  double ops = 2.0 * 128 * n * kbytes * iters * sms;
  printf("{\"kind\": \"%s\", \"N\": %d, \"shift_rows\": %d, \"tops\": %.1f, \"cycles_per_mma\": %.2f, \"err\": \"%s\"}\n",
         KIND == 0 ? "i8" : "f16", n, shift, ops / (ms * 1e-3) / 1e12, static_cast<double>(h[0]) / iters,
         cudaGetErrorString(err));
  cudaFree(cyc);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int n : {64, 128})
    for (int shift : {0, 1, 2, 3, 5, 8}) run<0>(n, sms, shift);
  return 0;
}
