// tc_pair.cu -- CTA-pair (cluster of 2, tcgen05 cta_group::2) semantics and
// throughput probe for the conv kernel's pair mode:
//  1. correctness: A 256x128 int8 / B Nx128 int8, 128B-swizzled K-major; each
//     CTA TMA-loads its 128 A rows and its N/2 B rows (cta_group::2 form,
//     completing on the leader's mbarrier); the leader issues 4 M=256 kind::i8
//     MMAs (K = 4 x 32 bytes) and multicasts the commit; each CTA reads its 128
//     accumulator rows from its own TMEM.  Compared with a CPU GEMM.
//  2. throughput: back-to-back MMAs from shared memory, M=128 (one CTA) vs
//     M=256 (pair), N in {64, 128, 256}: cycles per MMA and MACs per SM-cycle.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_1904_08368_b200/csrc -o tc_pair tests/tc_pair.cu -lcuda && ./tc_pair
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "tc_common.cuh"

using namespace mrb200::tc;

__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map, uint32_t bar_cluster, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], "
      "[%2];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(bar_cluster), "r"(c0), "r"(c1)
      : "memory");
}

__device__ __forceinline__ uint64_t sw128_desc(uint32_t addr) {
  const uint64_t hi = umma_desc_hi(1024, 2);
  return (hi << 32) | (((addr >> 4) & 0x3FFF) | ((1u) << 16));
}

__global__ void __launch_bounds__(192, 1) k_pair_gemm(const __grid_constant__ CUtensorMap tmA,
                                                      const __grid_constant__ CUtensorMap tmB, int N, int* D) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = base;
  uint8_t* sB = base + 16384;
  __shared__ uint64_t full, tfull;
  __shared__ uint32_t slot;
  const uint32_t rank = cluster_rank();
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    mbar_init(&full, 1);
    mbar_init(&tfull, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    const uint32_t lf = mapa_u32(&full, 0);
    if (rank == 0) mbar_expect_tx(&full, 2 * (16384 + N / 2 * 128));
    tma_load_2d_pair(sA, &tmA, lf, 0, rank * 128);
    tma_load_2d_pair(sB, &tmB, lf, 0, rank * (N / 2));
  }
  if (warp == 1 && rank == 0) {
    if (elect_one()) {
      mbar_wait(&full, 0);
      tc_fence_after();
      uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10);
      idesc |= static_cast<uint32_t>(N >> 3) << 17;
      idesc |= static_cast<uint32_t>(256 >> 4) << 24;
      for (int k = 0; k < 4; ++k)
        umma_pair<1>(tmem, sw128_desc(smem_u32(sA) + 32 * k), sw128_desc(smem_u32(sB) + 32 * k), idesc, k > 0);
      umma_commit_pair(&tfull, 3);
    }
    __syncwarp();
  }
  if (warp >= 2) {
    const int quarter = warp & 3;
    mbar_wait(&tfull, 0);
    tc_fence_after();
    for (int c = 0; c < N; c += 16) {
      uint32_t r[16];
      tmem_ld16(tmem + (static_cast<uint32_t>(quarter * 32) << 16) + c, r);
      const int row = rank * 128 + quarter * 32 + lane;
      for (int k = 0; k < 16; ++k) D[row * N + c + k] = static_cast<int>(r[k]);
    }
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 256;" ::"r"(tmem));
  }
}

// throughput: PAIR 0 = one CTA, M=128 cta_group::1; PAIR 1 = cluster of 2, M=256 cta_group::2
template <int PAIR>
__global__ void __launch_bounds__(128, 1) k_rate(int iters, int n, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 96 * 1024; i += blockDim.x) base[i] = static_cast<uint8_t>(i * 7);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) {
    if (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  tc_fence_before();
  if (PAIR) cluster_sync_all();
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  const bool issuer = threadIdx.x == 0 && (!PAIR || cluster_rank() == 0);
  if (issuer) {
    uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10);
    idesc |= static_cast<uint32_t>(n >> 3) << 17;
    idesc |= static_cast<uint32_t>((PAIR ? 256 : 128) >> 4) << 24;
    const uint64_t ad = sw128_desc(smem_u32(base)), bd = sw128_desc(smem_u32(base + 32768));
    const unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      if (PAIR) umma_pair<1>(tmem + (i & 1) * 256, ad, bd, idesc, i > 1);
      else umma<1>(tmem + (i & 1) * 256, ad, bd, idesc, i > 1);
    }
    if (PAIR) umma_commit_pair(&bar, 1);
    else umma_commit(&bar);
    mbar_wait(&bar, 0);
    cycles[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before();
  if (PAIR) cluster_sync_all();
  else __syncthreads();
  if (threadIdx.x < 32) {
    tc_fence_after();
    if (PAIR) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    else asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 enc() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
}

static bool make_map(CUtensorMap* m, void* g, int rows, int box_rows) {
  cuuint64_t dims[2] = {128, static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {128};
  cuuint32_t box[2] = {128, static_cast<cuuint32_t>(box_rows)};
  cuuint32_t es[2] = {1, 1};
  return enc()(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, g, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
}

template <class K, class... A>
static cudaError_t launch(K k, int grid, int block, size_t smem, int cluster, A... args) {
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cluster;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = cluster > 1 ? 1 : 0;
  cudaLaunchKernelEx(&cfg, k, args...);
  return cudaDeviceSynchronize();
}

int main() {
  int ok_all = 1;
  std::printf("{\"correctness\": {");
  for (int N : {64, 128, 256}) {
    std::vector<int8_t> A(256 * 128), B(N * 128);
    srand(N);
    for (auto& v : A) v = static_cast<int8_t>(rand() % 255 - 127);
    for (auto& v : B) v = static_cast<int8_t>(rand() % 255 - 127);
    int8_t *dA, *dB;
    int* dD;
    cudaMalloc(&dA, A.size());
    cudaMalloc(&dB, B.size());
    cudaMalloc(&dD, 256 * N * 4);
    cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice);
    cudaMemset(dD, 0xff, 256 * N * 4);
    CUtensorMap mA, mB;
    make_map(&mA, dA, 256, 128);
    make_map(&mB, dB, N, N / 2);
    cudaError_t e = launch(k_pair_gemm, 2, 192, 16384 + 16384 + 1024, 2, mA, mB, N, dD);
    std::vector<int> D(256 * N);
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    long bad = 0;
    for (int i = 0; i < 256; ++i)
      for (int j = 0; j < N; ++j) {
        int s = 0;
        for (int k = 0; k < 128; ++k) s += A[i * 128 + k] * B[j * 128 + k];
        bad += s != D[i * N + j];
      }
    ok_all &= bad == 0 && e == cudaSuccess;
    std::printf("%s\"N%d\": {\"err\": \"%s\", \"mismatches\": %ld}", N == 64 ? "" : ", ", N, cudaGetErrorString(e), bad);
    cudaFree(dA);
    cudaFree(dB);
    cudaFree(dD);
  }
  std::printf("}, \"rate\": {");
  unsigned long long* cyc;
  cudaMalloc(&cyc, 2 * 148 * 8);
  bool first = true;
  for (int N : {64, 128, 256}) {
    for (int pair : {0, 1}) {
      const int iters = 4096;
      cudaError_t e = pair ? launch(k_rate<1>, 2, 128, 97 * 1024, 2, iters, N, cyc)
                           : launch(k_rate<0>, 1, 128, 97 * 1024, 1, iters, N, cyc);
      unsigned long long c = 0;
      cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      const double per = static_cast<double>(c) / iters;
      const double macs_per_sm_cycle = (pair ? 256.0 : 128.0) * N * 128 / per / (pair ? 2 : 1);
      std::printf("%s\"N%d_%s\": {\"err\": \"%s\", \"cycles_per_mma\": %.1f, \"macs_per_sm_cycle\": %.0f}", first ? "" : ", ",
                  N, pair ? "pair_M256" : "single_M128", cudaGetErrorString(e), per, macs_per_sm_cycle);
      first = false;
    }
  }
  std::printf("}, \"ok\": %s}\n", ok_all ? "true" : "false");
  return ok_all ? 0 : 1;
}
