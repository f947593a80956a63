// tc_issue.cu -- is the layer-1 conv's MMA issue loop the limit?  Back-to-back
// tcgen05.mma kind::i8 M=128 N=64 from one thread, the conv kernel's way:
//   param   step table in the kernel parameter block, runtime step count (18),
//           4 sub-tiles per step (k_conv_tc's MMA issuer)
//   unroll  the same table, compile-time step count (fully unrolled)
//   const   one descriptor pair (tc_align.cu's loop)
//   +tmem   param loop while 3 warps stream tcgen05.ld from other TMEM columns
//   +smem   param loop while 3 warps stream 16-byte shared-memory stores
// with the 64-byte-swizzled K-major layout of the layer-1 A halo tile.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_1904_08368_b200/csrc -o tc_issue tests/tc_issue.cu && ./tc_issue
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "tc_common.cuh"

using namespace mrb200::tc;

struct Step {
  uint32_t a_lo, b_lo;
};
struct Params {
  int n_steps, reps, mode;
  uint32_t idesc, desc_hi;
  Step steps[144];
};

template <int MODE>
__global__ void __launch_bounds__(128, 1) k_issue(const __grid_constant__ Params p, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 110 * 1024; i += blockDim.x) base[i] = static_cast<uint8_t>(i * 13);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  __shared__ volatile int stop;
  if (threadIdx.x == 0) stop = 0;
  __syncthreads();
  if (MODE >= 3 && threadIdx.x >= 32) {
    // interference: warps 1-3 read TMEM (mode 3: tcgen05.ld of columns 256-511, the
    // epilogue's traffic) or stream stores into shared memory (mode 4: TMA-like writes)
    const int w = threadIdx.x / 32;
    uint32_t sink = 0;
    while (!stop) {
      if (MODE == 3) {
        uint32_t r[16];
        tmem_ld16(tmem + (static_cast<uint32_t>(w * 32) << 16) + 256 + (sink & 3) * 16, r);
        sink += r[0] + r[15];
      } else {
        float4* dst = reinterpret_cast<float4*>(base + 72 * 1024) + (threadIdx.x - 32) + (sink & 7) * 96;
        *dst = make_float4(1.f, 2.f, 3.f, static_cast<float>(sink));
        sink += 1;
      }
    }
    if (sink == 0xdeadbeef) out[1] = sink;
  }
  if (threadIdx.x == 0) {
    const uint64_t hi = static_cast<uint64_t>(p.desc_hi) << 32;
    const uint32_t a16 = smem_u32(base) >> 4, b16 = smem_u32(base + 64 * 1024) >> 4;
    const uint32_t sub16 = (128 * 64) >> 4;
    const unsigned long long t0 = clock64();
    for (int r = 0; r < p.reps; ++r) {
      const uint32_t dacc = (r & 1) * 256;
      if (MODE == 0 || MODE >= 3) {
        for (int st = 0; st < p.n_steps; ++st) {
          const uint64_t bd = hi | (p.steps[st].b_lo + b16);
          const uint32_t alo = p.steps[st].a_lo + a16;
#pragma unroll
          for (uint32_t sb = 0; sb < 4; ++sb) umma<1>(tmem + dacc + sb * 64, hi | (alo + sb * sub16), bd, p.idesc, st != 0);
        }
      } else if (MODE == 1) {
#pragma unroll
        for (int st = 0; st < 18; ++st) {
          const uint64_t bd = hi | (p.steps[st].b_lo + b16);
          const uint32_t alo = p.steps[st].a_lo + a16;
#pragma unroll
          for (uint32_t sb = 0; sb < 4; ++sb) umma<1>(tmem + dacc + sb * 64, hi | (alo + sb * sub16), bd, p.idesc, st != 0);
        }
      } else {
        const uint64_t bd = hi | (p.steps[0].b_lo + b16);
        const uint32_t alo = p.steps[0].a_lo + a16;
        for (int st = 0; st < 18; ++st)
#pragma unroll
          for (uint32_t sb = 0; sb < 4; ++sb) umma<1>(tmem + dacc + sb * 64, hi | (alo + sb * sub16), bd, p.idesc, st != 0);
      }
    }
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    out[blockIdx.x] = clock64() - t0;
    stop = 1;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

int main() {
  Params p{};
  p.n_steps = 18;
  p.reps = 200;
  p.idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((64u >> 3) << 17) | ((128u >> 4) << 24);
  p.desc_hi = umma_desc_hi(8 * 64, 4);  // 64B swizzle, SBO 512
  // layer-1 taps over a 58-wide padded grid: row shifts (kh-1)*58 + (kw-1) + 59, 2 K steps of 32 B
  int n = 0;
  for (int t = 0; t < 9; ++t)
    for (int kk = 0; kk < 2; ++kk) {
      const int rel = (t / 3) * 58 + (t % 3);
      const uint32_t a_off = rel * 64 + kk * 32, b_off = t * 64 * 64 + kk * 32;
      p.steps[n].a_lo = ((a_off >> 4) & 0x3FFF) | (1u << 16);
      p.steps[n].b_lo = ((b_off >> 4) & 0x3FFF) | (1u << 16);
      ++n;
    }
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  const char* names[] = {"param_runtime_steps", "unrolled_steps", "const_descriptors", "with_tmem_reads",
                         "with_smem_writes"};
  std::printf("{");
  for (int mode = 0; mode < 5; ++mode) {
    auto k = mode == 0 ? k_issue<0> : mode == 1 ? k_issue<1> : mode == 2 ? k_issue<2> : mode == 3 ? k_issue<3> : k_issue<4>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 112 * 1024);
    k<<<1, 128, 112 * 1024>>>(p, d);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long c = 0;
    cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    std::printf("%s\"%s\": {\"err\": \"%s\", \"cycles_per_mma\": %.1f}", mode ? ", " : "", names[mode], cudaGetErrorString(e),
                static_cast<double>(c) / (p.reps * 72.0));
  }
  std::printf("}\n");
  return 0;
}
