// dense_tc.cu -- tcgen05 dense (kernels::dense, kernels.cpp:609-638) for sm_100a.
//
// y[n, j] = sum_k x[n, k] * w[j, k]: the batch rows are the GEMM's M, the
// output columns its N, both operands K-major ("NT", the reference's weight
// layout [M, K] row-major).  int8 realized groups run kind::i8 (int8 x int8 ->
// int32, exact: the int32 sum scaled once equals the reference's fp32 sum of
// dequantized products under the 2^24 bound, proven per group at weight load);
// float groups run kind::f16 (bf16 x bf16 -> fp32 accumulate, tolerance).
//
// Three launches per dense group (dense_tc_launch):
//   k_dense_operand  the group's data prologue (pre-multiply, realize chain or
//                    bf16 rounding) applied ONCE per element of the float32
//                    [N, K] input, written as the A operand [Npad, Kp]
//   k_dense_tc       warp 0 TMA producer (A and B 128-byte swizzled K-major
//                    boxes through an mbarrier ring), warp 1 tcgen05.mma issuer
//                    (up to two 128-row M sub-tiles share each B stage, so a
//                    weight tile is read once per 256 batch rows), warps 2-9
//                    the epilogue (tcgen05.ld -> bias / relu / requantize ->
//                    row-major stores).  Split-K over grid.z for large K (VGG-16
//                    fc6: 205 MB of weights need every SM streaming): each split
//                    writes raw int32 / fp32 partials instead,
//   k_dense_reduce   and this kernel sums them in split order (deterministic)
//                    and applies the epilogue.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "dense_tc.hpp"
#include "launch.hpp"
#include "tc_common.cuh"

namespace mrb200 {
namespace {
using namespace tc;

constexpr int kDenseEpiWarps = 8;
constexpr int kDenseThreads = (2 + kDenseEpiWarps) * 32;
constexpr int kKBlockBytes = 128;  // K bytes per stage (one 128B-swizzle row)

struct DenseTcArgs {
  int32_t N, M;        // batch rows, output columns (logical)
  int32_t Npad, Mpad;  // operand rows (multiple of 128), weight rows (multiple of bn)
  int32_t kblocks;     // 128-byte K blocks of the padded K
  int32_t kb_per_split, splits;
  int32_t bn, ms;      // output-column tile; 128-row M sub-tiles per CTA (1 or 2)
  int32_t stages, a_stage_bytes, b_stage_bytes;
  uint32_t idesc, desc_hi;
  float acc_scale;
  void* ws;  // splits > 1: partials [splits][Npad][Mpad] (int32 / fp32)
  int32_t dbg;  // MRB200_DENSE_DBG timing experiments (wrong results): 1 no TMA, 2 no MMA, 4 no epilogue,
                //   8 exit right after setup
  EpiDev epi;
  OutDev out;
};

// Final value of one output element: reference order acc * scale (int8), then
// the group's epilogue ops (kernels.cuh apply_epi), stored by store_out.
template <int EB>
__device__ __forceinline__ void dense_finish(const DenseTcArgs& a, uint32_t raw, int n, int j) {
  float v = EB == 1 ? __fmul_rn(static_cast<float>(static_cast<int32_t>(raw)), a.acc_scale) : __uint_as_float(raw);
  int32_t code = 0;
  v = apply_epi(a.epi, v, n, j, &code);
  store_out(a.out, v, code, n, j);
}

// Compile-time epilogues for the sequences the fuse pass leaves after a dense
// (the ResNet / MobileNet heads: bias; VGG / DQN hidden layers: bias + relu);
// anything else (and non-float32 outputs) is interpreted by apply_epi.
enum DenseSig : int { DSIG_ANY = 0, DSIG_BIAS = 1, DSIG_BIAS_RELU = 2 };

template <int EB, int SIG>
__global__ void __launch_bounds__(kDenseThreads, 1)
    k_dense_tc(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, const DenseTcArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* smA = base;
  uint8_t* smB = smA + a.stages * a.a_stage_bytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smB + a.stages * a.b_stage_bytes);
  uint64_t* full = bars;
  uint64_t* empty = bars + a.stages;
  uint64_t* tfull = empty + a.stages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 1);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int n_tile = blockIdx.x, m_group = blockIdx.y, split = blockIdx.z;
  const int kb0 = split * a.kb_per_split;
  const int kb1 = min(a.kblocks, kb0 + a.kb_per_split);
  const uint32_t tcols = static_cast<uint32_t>(a.ms * a.bn);
  const uint32_t tmem_cols = tcols <= 32 ? 32 : tcols <= 64 ? 64 : tcols <= 128 ? 128 : tcols <= 256 ? 256 : 512;
  pdl_trigger();
  if (threadIdx.x == 0) {
    for (int i = 0; i < a.stages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    mbar_init(tfull, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(tmem_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_wait();  // the A operand (and every output buffer) belongs to the previous kernels until here
  if (a.dbg & 8) goto dense_done;

  if (warp == 0) {
    if (lane == 0) {
      // ===== TMA producer =====
      int stage = 0;
      uint32_t phase = 0;
      for (int kb = kb0; kb < kb1; ++kb) {
        mbar_wait(&empty[stage], phase ^ 1);
        if (a.dbg & 1) {
          mbar_arrive(&full[stage]);
        } else {
          mbar_expect_tx(&full[stage], a.a_stage_bytes + a.b_stage_bytes);
          tma_load_2d(smA + stage * a.a_stage_bytes, &tmA, &full[stage], kb * kKBlockBytes, m_group * a.ms * 128);
          tma_load_2d(smB + stage * a.b_stage_bytes, &tmB, &full[stage], kb * kKBlockBytes, n_tile * a.bn);
        }
        if (++stage == a.stages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    // ===== MMA issuer =====
    if (elect_one()) {
      const uint64_t hi = static_cast<uint64_t>(a.desc_hi) << 32;
      int stage = 0;
      uint32_t phase = 0;
      for (int kb = kb0; kb < kb1; ++kb) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        const uint32_t sa = smem_u32(smA + stage * a.a_stage_bytes), sb = smem_u32(smB + stage * a.b_stage_bytes);
        if (!(a.dbg & 2))
#pragma unroll
        for (int kk = 0; kk < kKBlockBytes / 32; ++kk) {  // 32 K bytes per tcgen05.mma
          const uint64_t bd = hi | (((sb + kk * 32) >> 4) & 0x3FFF) | (1u << 16);
          for (int m = 0; m < a.ms; ++m) {
            const uint64_t ad = hi | (((sa + m * 128 * kKBlockBytes + kk * 32) >> 4) & 0x3FFF) | (1u << 16);
            umma<EB>(tmem_base + static_cast<uint32_t>(m * a.bn), ad, bd, a.idesc, (kb > kb0 || kk > 0) ? 1u : 0u);
          }
        }
        umma_commit(&empty[stage]);  // the stage is free once these MMAs retire
        if (++stage == a.stages) {
          stage = 0;
          phase ^= 1;
        }
      }
      umma_commit(tfull);
    }
    __syncwarp();
  } else {
    // ===== epilogue ===== warp w: TMEM lane quarter w % 4, column half (w - 2) / 4
    const int quarter = warp & 3, half = (warp - 2) >> 2;
    mbar_wait(tfull, 0);
    tc_fence_after();
    const int cw = a.bn / 2;
    for (int m = 0; m < ((a.dbg & 4) ? 0 : a.ms); ++m) {
      const int n = (m_group * a.ms + m) * 128 + quarter * 32 + lane;
      for (int c = half * cw; c < (half + 1) * cw; c += 16) {
        float bias[16];
        if (SIG != DSIG_ANY && a.splits == 1 && n_tile * a.bn + c + 16 <= a.M) {  // before the TMEM load
          const float4* bp = reinterpret_cast<const float4*>(a.epi.vec[0] + n_tile * a.bn + c);
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const float4 f = __ldg(bp + q);
            bias[4 * q] = f.x; bias[4 * q + 1] = f.y; bias[4 * q + 2] = f.z; bias[4 * q + 3] = f.w;
          }
        }
        uint32_t raw[16];
        tmem_ld16(tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + static_cast<uint32_t>(m * a.bn + c), raw);
        const int j0 = n_tile * a.bn + c;
        if (a.splits > 1) {  // raw partials, row n of split `split` (Npad x Mpad: always in range)
          uint4* dst = reinterpret_cast<uint4*>(static_cast<uint32_t*>(a.ws) +
                                                (static_cast<int64_t>(split) * a.Npad + n) * a.Mpad + j0);
#pragma unroll
          for (int q = 0; q < 4; ++q) dst[q] = make_uint4(raw[4 * q], raw[4 * q + 1], raw[4 * q + 2], raw[4 * q + 3]);
        } else if (n < a.N) {
          if (SIG != DSIG_ANY && j0 + 16 <= a.M) {
            // row-major float32 result (checked on the host): acc * s + bias [, relu]
            // in the reference's order, four 16-byte stores per 16 columns
            float v[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              v[i] = EB == 1 ? __fmul_rn(static_cast<float>(static_cast<int32_t>(raw[i])), a.acc_scale)
                             : __uint_as_float(raw[i]);
              v[i] = __fadd_rn(v[i], bias[i]);
              if (SIG == DSIG_BIAS_RELU) v[i] = relu_ref(v[i]);
            }
            float4* dst = reinterpret_cast<float4*>(static_cast<float*>(a.out.primary) + static_cast<int64_t>(n) * a.M + j0);
#pragma unroll
            for (int q = 0; q < 4; ++q) dst[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
          } else {
#pragma unroll
            for (int i = 0; i < 16; ++i)
              if (j0 + i < a.M) dense_finish<EB>(a, raw[i], n, j0 + i);
          }
        }
      }
    }
  }
dense_done:
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(tmem_cols));
  }
}

// Split-K: partial sums in split order (int32 exact / fp32 deterministic), then the epilogue.
template <int EB>
__global__ void __launch_bounds__(256) k_dense_reduce(const DenseTcArgs a) {
  pdl_trigger();
  pdl_wait();
  const int64_t total = static_cast<int64_t>(a.N) * a.M;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int n = static_cast<int>(i / a.M), j = static_cast<int>(i - static_cast<int64_t>(n) * a.M);
    const uint32_t* p = static_cast<const uint32_t*>(a.ws) + static_cast<int64_t>(n) * a.Mpad + j;
    const int64_t sstride = static_cast<int64_t>(a.Npad) * a.Mpad;
    uint32_t r;
    if (EB == 1) {
      int32_t s = 0;
      for (int k = 0; k < a.splits; ++k) s += static_cast<int32_t>(p[k * sstride]);
      r = static_cast<uint32_t>(s);
    } else {
      float s = __uint_as_float(p[0]);
      for (int k = 1; k < a.splits; ++k) s = __fadd_rn(s, __uint_as_float(p[k * sstride]));
      r = __float_as_uint(s);
    }
    dense_finish<EB>(a, r, n, j);
  }
}

// The group's data prologue once per element: x[n, k] (float32 row-major) ->
// A[n, k] (int8 code or bf16), zero padding to [Npad, Kp].  Mirrors the row
// staging of k_dense_ks (kernels_simt.cu): optional pre-multiply, then the
// realize chain (quant) or bf16 rounding.
template <int EB, bool CAL>
__global__ void __launch_bounds__(256) k_dense_operand(const float* __restrict__ x, int N, int K, int Npad, int Kp,
                                                       float pre_mul, int quant, QDev q, void* __restrict__ A) {
  pdl_trigger();
  pdl_wait();
  const int kp4 = Kp / 4;
  const int64_t total = static_cast<int64_t>(Npad) * kp4;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int n = static_cast<int>(i / kp4), k = 4 * static_cast<int>(i - static_cast<int64_t>(n) * kp4);
    float t[4];
    bool live[4];
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      live[b] = n < N && k + b < K;
      t[b] = live[b] ? x[static_cast<int64_t>(n) * K + k + b] : 0.f;
      if (live[b] && pre_mul != 0.f) t[b] = __fmul_rn(t[b], pre_mul);
    }
    if constexpr (EB == 4) {  // tf32: rounded to tf32 (the MMA would truncate to its top 19 bits)
      static_cast<float4*>(A)[i] = make_float4(tf32_rn(t[0]), tf32_rn(t[1]), tf32_rn(t[2]), tf32_rn(t[3]));
    } else if constexpr (EB == 1) {
      uint32_t packed = 0;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int32_t code = live[b] ? (quant ? quant_code_t<CAL>(t[b], q) : static_cast<int32_t>(t[b])) : 0;
        packed |= (static_cast<uint32_t>(code) & 0xffu) << (8 * b);
      }
      static_cast<uint32_t*>(A)[i] = packed;
    } else {
      uint2 w;
      w.x = pack_bf16x2(t[0], t[1]);
      w.y = pack_bf16x2(t[2], t[3]);
      static_cast<uint2*>(A)[i] = w;
    }
  }
}

// [M, K] float32 weight after its prologue (folded scale, realize chain) ->
// B rows [Mpad, Kp] (int8 codes / bf16), zero padded.
__global__ void k_dense_weight_rows(const float* __restrict__ w, int M, int K, int Mpad, int Kp,
                                    const float* __restrict__ oc_scale, float scalar, int eb, int quant, QDev q,
                                    void* out) {
  const int64_t total = static_cast<int64_t>(Mpad) * Kp;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int j = static_cast<int>(i / Kp), k = static_cast<int>(i - static_cast<int64_t>(j) * Kp);
    const bool live = j < M && k < K;
    float v = 0.f;
    if (live) {
      v = w[static_cast<int64_t>(j) * K + k];
      if (oc_scale) v = __fmul_rn(v, oc_scale[j]);
      if (scalar != 0.f) v = __fmul_rn(v, scalar);
    }
    if (eb == 1) static_cast<int8_t*>(out)[i] = static_cast<int8_t>(live ? (quant ? quant_code(v, q) : static_cast<int32_t>(v)) : 0);
    else if (eb == 4) static_cast<float*>(out)[i] = live ? tf32_rn(v) : 0.f;
    else static_cast<uint16_t*>(out)[i] = live ? f32_to_bf16(v) : 0;
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_tiled() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult qr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qr) == cudaSuccess &&
        qr == cudaDriverEntryPointSuccess)
      return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    return static_cast<PFN_cuTensorMapEncodeTiled_v12000>(nullptr);
  }();
  return fn;
}

// K-major [rows, Kp] operand as bytes: a stage is one box {128 bytes, box_rows}
// with the 128-byte swizzle (the UMMA canonical K-major SWIZZLE_128B layout).
bool encode_operand(CUtensorMap* m, const void* p, int rows, int row_bytes, int box_rows) {
  auto enc = encode_tiled();
  if (!enc) return false;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(row_bytes), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(row_bytes)};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(kKBlockBytes), static_cast<cuuint32_t>(box_rows)};
  cuuint32_t es[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(p), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

struct DenseTcPlan {
  DenseTcSpec spec;
  DenseTcArgs args;
  dim3 grid;
  size_t smem = 0;
  const void* map_a = nullptr;
  const void* map_b = nullptr;
  CUtensorMap tmA, tmB;
};

DenseTcPlan* dense_tc_create(const DenseTcSpec& sp) {
  if (sp.eb != 1 && sp.eb != 2 && sp.eb != 4) return nullptr;
  if (!encode_tiled()) return nullptr;
  auto* p = new DenseTcPlan();
  p->spec = sp;
  DenseTcArgs& a = p->args;
  std::memset(&a, 0, sizeof(a));
  a.N = sp.N;
  a.M = sp.M;
  // latency-bound heads get more, narrower tiles; weight-streaming layers wide
  // tiles with two M sub-tiles sharing each weight stage
  a.bn = sp.M >= 2048 ? 128 : sp.M >= 1024 ? 64 : 32;
  if (sp.M < 2048 && sp.K * sp.eb <= 4096) a.bn = 32;
  a.Npad = (sp.N + 127) / 128 * 128;
  a.Mpad = (sp.M + a.bn - 1) / a.bn * a.bn;
  a.ms = a.Npad >= 256 && (a.Mpad / a.bn) * (a.Npad / 128) > 96 ? 2 : 1;
  if (a.Npad % (128 * a.ms)) a.ms = 1;
  a.kblocks = dense_tc_kp(sp.K, sp.eb) * sp.eb / kKBlockBytes;
  const int n_tiles = a.Mpad / a.bn, m_groups = a.Npad / (128 * a.ms);
  // split K until the grid covers the SMs (each split keeps >= 4 K blocks)
  int splits = std::max(1, std::min(a.kblocks / 4, 148 / std::max(1, n_tiles * m_groups)));
  a.kb_per_split = (a.kblocks + splits - 1) / splits;
  a.splits = (a.kblocks + a.kb_per_split - 1) / a.kb_per_split;
  a.a_stage_bytes = a.ms * 128 * kKBlockBytes;
  a.b_stage_bytes = a.bn * kKBlockBytes;
  const int per_stage = a.a_stage_bytes + a.b_stage_bytes;
  a.stages = std::max(2, std::min(6, (200 * 1024) / per_stage));
  a.stages = std::min(a.stages, std::max(2, a.kb_per_split));
  p->smem = 1024 + static_cast<size_t>(a.stages) * per_stage + 256;
  // instruction descriptor: D format, A/B formats, K-major both, N >> 3, M >> 4
  uint32_t idesc = 0;
  if (sp.eb == 1) idesc |= (2u << 4) | (1u << 7) | (1u << 10);       // S32 <- s8 x s8
  else if (sp.eb == 4) idesc |= (1u << 4) | (2u << 7) | (2u << 10);  // F32 <- tf32 x tf32
  else idesc |= (1u << 4) | (1u << 7) | (1u << 10);                  // F32 <- bf16 x bf16
  idesc |= static_cast<uint32_t>(a.bn >> 3) << 17;
  idesc |= static_cast<uint32_t>(128 >> 4) << 24;
  a.idesc = idesc;
  a.desc_hi = umma_desc_hi(8 * kKBlockBytes, 2);  // 128B swizzle: SBO = 8 rows x 128 B
  p->grid = dim3(static_cast<unsigned>(n_tiles), static_cast<unsigned>(m_groups), static_cast<unsigned>(a.splits));
  return p;
}

void dense_tc_destroy(DenseTcPlan* p) { delete p; }

int dense_tc_kp(int K, int eb) {
  const int per = kKBlockBytes / eb;
  return (K + per - 1) / per * per;
}

int64_t dense_tc_operand_bytes(const DenseTcPlan* p) {
  return static_cast<int64_t>(p->args.Npad) * dense_tc_kp(p->spec.K, p->spec.eb) * p->spec.eb;
}

int64_t dense_tc_workspace_bytes(const DenseTcPlan* p) {
  return p->args.splits > 1 ? static_cast<int64_t>(p->args.splits) * p->args.Npad * p->args.Mpad * 4 : 0;
}

int64_t dense_tc_weight_rows(const DenseTcPlan* p) { return p->args.Mpad; }

int dense_tc_launches(const DenseTcPlan* p) { return p->args.splits > 1 ? 3 : 2; }

const char* dense_tc_describe(const DenseTcPlan* p, char* buf, int n) {
  const DenseTcArgs& a = p->args;
  std::snprintf(buf, n, "tcgen05 %s dense %dx(M128)xN%d kblocks=%d splits=%d stages=%d grid=%ux%ux%u smem=%zu",
                p->spec.eb == 1 ? "i8" : p->spec.eb == 4 ? "tf32" : "bf16", a.ms, a.bn, a.kblocks, a.splits, a.stages, p->grid.x, p->grid.y,
                p->grid.z, p->smem);
  return buf;
}

void dense_tc_prep_weight(const DenseTcPlan* p, const float* w, const float* oc_scale, float scalar, int quant,
                          QDev q, void* out, cudaStream_t s) {
  const int Kp = dense_tc_kp(p->spec.K, p->spec.eb);
  const int64_t total = static_cast<int64_t>(p->args.Mpad) * Kp;
  const unsigned blocks = static_cast<unsigned>(std::min<int64_t>((total + 255) / 256, 148 * 32));
  k_dense_weight_rows<<<blocks, 256, 0, s>>>(w, p->spec.M, p->spec.K, p->args.Mpad, Kp, oc_scale, scalar, p->spec.eb,
                                             quant, q, out);
}

bool dense_tc_launch(DenseTcPlan* p, const float* x, float pre_mul, int quant, QDev q, void* operand, const void* w,
                     void* ws, float acc_scale, const EpiDev& epi, const OutDev& out, cudaStream_t s) {
  const DenseTcSpec& sp = p->spec;
  const int Kp = dense_tc_kp(sp.K, sp.eb);
  DenseTcArgs a = p->args;
  static const int dbg = [] {
    const char* e = std::getenv("MRB200_DENSE_DBG");
    return e ? std::atoi(e) : 0;
  }();
  a.dbg = dbg;
  a.acc_scale = acc_scale;
  a.epi = epi;
  a.out = out;
  a.ws = ws;
  bool cal = quant && q.ovf;
  for (int k = 0; k < epi.n_ops; ++k) cal = cal || (epi.op[k] == E_REQ && epi.q[k].ovf);
  // 1. operand (x == nullptr: the producer already wrote it -- the fused sum)
  if (x) {
    const int64_t total = static_cast<int64_t>(a.Npad) * (Kp / 4);
    const unsigned blocks = static_cast<unsigned>(std::min<int64_t>((total + 255) / 256, 148 * 8));
    if (sp.eb == 1)
      pdl_launch(cal ? k_dense_operand<1, true> : k_dense_operand<1, false>, dim3(blocks), dim3(256), 0, s, x, sp.N,
                 sp.K, a.Npad, Kp, pre_mul, quant, q, operand);
    else if (sp.eb == 4)
      pdl_launch(k_dense_operand<4, false>, dim3(blocks), dim3(256), 0, s, x, sp.N, sp.K, a.Npad, Kp, pre_mul, 0, q,
                 operand);
    else
      pdl_launch(k_dense_operand<2, false>, dim3(blocks), dim3(256), 0, s, x, sp.N, sp.K, a.Npad, Kp, pre_mul, 0, q,
                 operand);
  }
  // 2. contraction
  if (p->map_a != operand || p->map_b != w) {
    if (!encode_operand(&p->tmA, operand, a.Npad, Kp * sp.eb, 128 * a.ms)) return false;
    if (!encode_operand(&p->tmB, w, a.Mpad, Kp * sp.eb, a.bn)) return false;
    p->map_a = operand;
    p->map_b = w;
  }
  int sig = DSIG_ANY;
  if (out.primary_fmt == FMT_F32 && out.plan.cpc == 0 && !out.side && (sp.M & 3) == 0 && a.splits == 1) {
    if (epi.n_ops == 1 && epi.op[0] == E_BIAS) sig = DSIG_BIAS;
    if (epi.n_ops == 2 && epi.op[0] == E_BIAS && epi.op[1] == E_RELU) sig = DSIG_BIAS_RELU;
  }
  using KFn = void (*)(CUtensorMap, CUtensorMap, DenseTcArgs);
  static const KFn kfns[3][3] = {{k_dense_tc<1, DSIG_ANY>, k_dense_tc<1, DSIG_BIAS>, k_dense_tc<1, DSIG_BIAS_RELU>},
                                 {k_dense_tc<2, DSIG_ANY>, k_dense_tc<2, DSIG_BIAS>, k_dense_tc<2, DSIG_BIAS_RELU>},
                                 {k_dense_tc<4, DSIG_ANY>, k_dense_tc<4, DSIG_BIAS>, k_dense_tc<4, DSIG_BIAS_RELU>}};
  static bool attr_set[3][3] = {};
  const int ei = sp.eb == 1 ? 0 : sp.eb == 2 ? 1 : 2;
  KFn kern = kfns[ei][sig];
  if (!attr_set[ei][sig]) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    attr_set[ei][sig] = true;
  }
  pdl_launch(kern, p->grid, dim3(kDenseThreads), p->smem, s, p->tmA, p->tmB, a);
  // 3. split-K reduction + epilogue
  if (a.splits > 1) {
    const int64_t total = static_cast<int64_t>(sp.N) * sp.M;  // (split-K reduction)
    const unsigned blocks = static_cast<unsigned>(std::min<int64_t>((total + 255) / 256, 148 * 8));
    pdl_launch(sp.eb == 1 ? k_dense_reduce<1> : sp.eb == 4 ? k_dense_reduce<4> : k_dense_reduce<2>, dim3(blocks),
               dim3(256), 0, s, a);
  }
  return true;
}

}  // namespace mrb200
