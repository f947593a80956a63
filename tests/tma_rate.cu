// tma_rate.cu -- per-SM TMA load throughput for the conv kernel's A-operand
// boxes: a 4-D tiled map over a pixel-major chunk plane ({kb, rows, 1, 1} boxes of
// `hbox` kb-byte rows, 64B/128B swizzle or none), vs one 1-D cp.async.bulk of the
// same contiguous bytes.  One CTA per SM, one thread issues loads into a ring of
// `stages` buffers and waits on per-stage mbarriers.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_rate tests/tma_rate.cu -lcuda && ./tma_rate
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__global__ void __launch_bounds__(32, 1) k_tma(const __grid_constant__ CUtensorMap map, const uint8_t* src, int mode,
                                               int kb, int hbox, int stages, int iters, int64_t rows_total,
                                               unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bars[16];
  const int bytes = kb * hbox;
  if (threadIdx.x == 0) {
    for (int i = 0; i < stages; ++i)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  if (threadIdx.x != 0) return;
  const unsigned long long t0 = clock64();
  uint32_t phase[16] = {0};
  const int64_t per_cta = rows_total / gridDim.x;
  for (int it = 0; it < iters; ++it) {
    const int s = it % stages;
    if (it >= stages) {  // wait for this buffer's previous load
      asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}\n" ::"r"(
                       smem_u32(&bars[s])), "r"(phase[s]) : "memory");
      phase[s] ^= 1;
    }
    const int64_t row = blockIdx.x * per_cta + (static_cast<int64_t>(it) * hbox) % (per_cta - hbox);
    uint8_t* dst = sm + s * bytes;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bars[s])), "r"(bytes) : "memory");
    if (mode == 0) {
      asm volatile(
          "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];" ::
              "r"(smem_u32(dst)), "l"(&map), "r"(smem_u32(&bars[s])), "r"(0), "r"(static_cast<int>(row)), "r"(0), "r"(0)
          : "memory");
    } else {
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       smem_u32(dst)), "l"(src + row * kb), "r"(bytes), "r"(smem_u32(&bars[s]))
                   : "memory");
    }
  }
  for (int s = 0; s < stages && s < iters; ++s)
    asm volatile("{\n.reg .pred p;\nW2:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W2;\n}\n" ::"r"(
                     smem_u32(&bars[s])), "r"(phase[s]) : "memory");
  cyc[blockIdx.x] = clock64() - t0;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int64_t rows_total = int64_t(1) << 22;  // 4M rows x kb bytes (256 / 512 MB)
  uint8_t* buf;
  cudaMalloc(&buf, rows_total * 128);
  cudaMemset(buf, 1, rows_total * 128);
  unsigned long long* cyc;
  cudaMalloc(&cyc, sms * sizeof(unsigned long long));
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc), cudaEnableDefault, &q);
  for (int mode : {0, 1})
    for (int kb : {64, 128})
      for (int hbox : {64, 224})
        for (int stages : {2, 4, 8}) {
          if (kb * hbox * stages > 200 * 1024) continue;
          CUtensorMap map;
          cuuint64_t dims[4] = {static_cast<cuuint64_t>(kb), static_cast<cuuint64_t>(rows_total), 1, 1};
          cuuint64_t strides[3] = {static_cast<cuuint64_t>(kb), static_cast<cuuint64_t>(rows_total) * kb,
                                   static_cast<cuuint64_t>(rows_total) * kb};
          cuuint32_t box[4] = {static_cast<cuuint32_t>(kb), static_cast<cuuint32_t>(hbox), 1, 1};
          cuuint32_t es[4] = {1, 1, 1, 1};
          enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              kb == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
          const int iters = 2000;
          const size_t smem = static_cast<size_t>(kb) * hbox * stages;
          cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
          k_tma<<<sms, 32, smem>>>(map, buf, mode, kb, hbox, stages, 50, rows_total, cyc);
          cudaEvent_t e0, e1;
          cudaEventCreate(&e0);
          cudaEventCreate(&e1);
          cudaEventRecord(e0);
          k_tma<<<sms, 32, smem>>>(map, buf, mode, kb, hbox, stages, iters, rows_total, cyc);
          cudaEventRecord(e1);
          cudaError_t err = cudaEventSynchronize(e1);
          float ms = 0;
          cudaEventElapsedTime(&ms, e0, e1);
          const double bytes = static_cast<double>(kb) * hbox * iters * sms;
          printf("{\"mode\": \"%s\", \"kb\": %d, \"hbox\": %d, \"stages\": %d, \"GBps_total\": %.0f, \"GBps_per_sm\": %.1f, \"err\": \"%s\"}\n",
                 mode == 0 ? "tensor4d" : "bulk1d", kb, hbox, stages, bytes / (ms * 1e-3) / 1e9,
                 bytes / (ms * 1e-3) / 1e9 / sms, cudaGetErrorString(err));
        }
  return 0;
}
