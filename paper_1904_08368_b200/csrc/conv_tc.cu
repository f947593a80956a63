// conv_tc.cu -- tcgen05 implicit-GEMM convolution for sm_100a.
//
// One launch executes a whole fused conv group: the
// realize-chain prologue was hoisted (weights) or emitted by the producer
// (activation codes), the contraction runs on the 5th-gen tensor cores
// (kind::i8 int8 x int8 -> int32, or kind::f16 bf16 x bf16 -> fp32) with the
// accumulator in TMEM, and the elementwise epilogue (scale, bias_add, add,
// relu, requantize, clip) is applied in registers after tcgen05.ld before
// 16-byte vector stores -- no intermediate tensor touches HBM.
//
// Halo implicit GEMM.  Activations are stored P16 (kernels.cuh): per 16-byte
// channel chunk, one plane over the zero-padded pixel grid.  The GEMM's M
// dimension enumerates that padded grid directly (M = N*(H+2)*(W+2)), so for
// a stride-1 "same" conv every tap (kh, kw) of output pixel q reads input
// pixel q + (kh-1)*Wp + (kw-1).  A 128-row output tile therefore needs ONE
// contiguous input range of 128 + 2*Wp + 2 pixels per chunk plane, fetched by
// a single TMA load; the 9 taps are 9 UMMA shared-memory descriptors whose
// start addresses differ by whole 16-byte rows (K-major, no-swizzle canonical
// layout: core matrices of 8 rows x 16 bytes, SBO = 128 B between 8-row
// groups, LBO = plane stride between the two 16-byte K halves).  L2->SM
// traffic for A is ~(128 + 2Wp + 2)/128 of the output tile instead of the 9x
// of an im2col gather.  Border rows of the padded grid are computed and
// written as zeros, which is exactly the zero border the next conv needs.
//
// Kernel structure (persistent, warp-specialised, one CTA per SM):
//   warp 0      TMA producer: weights once (resident) or per stage, A halo
//               stages through an mbarrier ring
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer
//   warps 2-5   epilogue: tcgen05.ld -> epilogue -> st.global.v4
//   TMEM        2 accumulator buffers (tile i epilogue overlaps tile i+1 MMA)
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>

#include "conv_tc.hpp"

namespace mrb200 {

namespace {

constexpr int kTileM = 128;
constexpr int kEpiWarps = 8;
constexpr int kThreadsTc = (2 + kEpiWarps) * 32;
constexpr int kMaxTaps = 9;
constexpr int kSmemBudget = 227 * 1024 - 1024;

enum EpiSig : int { SIG_ANY = 0, SIG_BIAS = 1, SIG_BIAS_RELU = 2, SIG_BIAS_RELU_REQ = 3, SIG_BIAS_RES_RELU = 4 };

// Compile-time epilogue for the op sequences the realize/fuse passes emit.
inline int epi_signature(const EpiDev& e, const OutDev& o) {
  auto q_ok = [](const QDev& q) {
    return q.lo >= -2147483520.f && q.hi <= 2147483520.f && q.lo == q.lo && q.hi == q.hi;
  };
  if (o.side && !q_ok(o.side_q)) return SIG_ANY;
  if (e.n_ops == 1 && e.op[0] == E_BIAS && o.primary_fmt != FMT_I8) return SIG_BIAS;
  if (e.n_ops == 2 && e.op[0] == E_BIAS && e.op[1] == E_RELU && o.primary_fmt != FMT_I8) return SIG_BIAS_RELU;
  if (e.n_ops == 3 && e.op[0] == E_BIAS && e.op[1] == E_RELU && e.op[2] == E_REQ && o.primary_fmt == FMT_I8 &&
      !o.side && q_ok(e.q[2]))
    return SIG_BIAS_RELU_REQ;
  if (e.n_ops == 3 && e.op[0] == E_BIAS && e.op[1] == E_RES && e.op[2] == E_RELU && o.primary_fmt != FMT_I8)
    return SIG_BIAS_RES_RELU;
  return SIG_ANY;
}

struct TcArgs {
  int32_t Wp, Hp, H, W;
  int64_t Pp;           // pixels per plane (input grid == output grid)
  int32_t m_tiles, n_tiles, Cc, pps, k_stages, halo;
  int32_t taps;
  int32_t delta[kMaxTaps];  // tap row offset inside the halo
  int32_t bn;
  int32_t resident_b;
  int32_t a_stage_bytes, b_stage_bytes, b_res_bytes, n_stages;
  uint32_t idesc;
  float acc_scale;
  EpiDev epi;
  OutDev out;
};

// ---- PTX helpers -------------------------------------------------------------------

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::
          "r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2,
                                            int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], "
      "[%2];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}

// K-major, no-swizzle UMMA shared-memory descriptor (sm_100 version 1):
// start>>4 [0,14), LBO>>4 [16,30), SBO>>4 [32,46), version [46,48) = 1,
// base offset 0, layout type SWIZZLE_NONE (0) [61,64).
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  return d;
}

template <int EB>
__device__ __forceinline__ void umma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  if constexpr (EB == 1) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
  } else {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
  }
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ uint32_t pack4_i8(int a, int b, int c, int d) {
  return (static_cast<uint32_t>(a) & 0xff) | ((static_cast<uint32_t>(b) & 0xff) << 8) |
         ((static_cast<uint32_t>(c) & 0xff) << 16) | ((static_cast<uint32_t>(d) & 0xff) << 24);
}

// 16 channels [c0, c0+16) of pixel q through the epilogue, stored as 16-byte chunks.
// SIG selects a compile-time op sequence for the common fused groups; SIG_ANY
// interprets EpiDev.  The arithmetic is identical either way (kernels.cuh).
template <int EB, int SIG>
__device__ __forceinline__ void epilogue_chunk(const TcArgs& a, const uint32_t* raw, int64_t q, bool border, int c0) {
  const OutDev& o = a.out;
  const int pf = o.primary_fmt;
  if (border) {
    // padded-grid border: the zero border of the P16 output (and side codes)
    const int chunks = pf == FMT_F32 ? 4 : pf == FMT_BF16 ? 2 : 1;
    const int cpc = 16 / chunks;
    for (int k = 0; k < chunks; ++k)
      *reinterpret_cast<int4*>(static_cast<char*>(o.primary) + ((static_cast<int64_t>(c0 / cpc + k) * o.plan.Pp + q) * 16)) =
          make_int4(0, 0, 0, 0);
    if (o.side)
      *reinterpret_cast<int4*>(reinterpret_cast<char*>(o.side) + ((static_cast<int64_t>(c0 / 16) * o.slay.Pp + q) * 16)) =
          make_int4(0, 0, 0, 0);
    return;
  }
  float v[16];
  int32_t code[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    if constexpr (EB == 1) v[i] = __fmul_rn(static_cast<float>(static_cast<int32_t>(raw[i])), a.acc_scale);
    else v[i] = __uint_as_float(raw[i]);
    code[i] = 0;
  }
  const EpiDev& e = a.epi;
  auto vec16 = [&](const float* base, float (&t)[16]) {
    const float4* p = reinterpret_cast<const float4*>(base + c0);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float4 f = __ldg(p + j);
      t[4 * j] = f.x; t[4 * j + 1] = f.y; t[4 * j + 2] = f.z; t[4 * j + 3] = f.w;
    }
  };
  auto res16 = [&](int k, float (&t)[16]) {
    const Lay& L = e.res_lay[k];
    if (e.res_fmt[k] == FMT_F32) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float4 f = *reinterpret_cast<const float4*>(static_cast<const char*>(e.res[k]) +
                                                    (static_cast<int64_t>(c0 / 4 + j) * L.Pp + q) * 16);
        t[4 * j] = f.x; t[4 * j + 1] = f.y; t[4 * j + 2] = f.z; t[4 * j + 3] = f.w;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        uint4 u = *reinterpret_cast<const uint4*>(static_cast<const char*>(e.res[k]) +
                                                  (static_cast<int64_t>(c0 / 8 + j) * L.Pp + q) * 16);
        uint32_t w4[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          t[8 * j + 2 * h] = __uint_as_float(w4[h] << 16);
          t[8 * j + 2 * h + 1] = __uint_as_float(w4[h] & 0xffff0000u);
        }
      }
    }
  };
  if constexpr (SIG == SIG_ANY) {
    for (int k = 0; k < e.n_ops; ++k) {
      const int op = e.op[k];
      if (op == E_MULS) {
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = __fmul_rn(v[i], e.s[k]);
      } else if (op == E_MULC || op == E_BIAS) {
        float t[16];
        vec16(e.vec[k], t);
        if (op == E_MULC) {
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] = __fmul_rn(v[i], t[i]);
        } else {
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] = __fadd_rn(v[i], t[i]);
        }
      } else if (op == E_RES) {
        float t[16];
        res16(k, t);
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = __fadd_rn(v[i], t[i]);
      } else if (op == E_RELU) {
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = relu_ref(v[i]);
      } else if (op == E_REQ) {
        const QDev qd = e.q[k];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          code[i] = quant_code(v[i], qd);
          v[i] = __fmul_rn(static_cast<float>(code[i]), qd.c2);
        }
      } else if (op == E_CLIP) {
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = clip_ref(v[i], e.s[k], e.s2[k]);
      }
    }
  } else {
    // op 0 is always bias_add for the specialised signatures
    float t[16];
    vec16(e.vec[0], t);
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __fadd_rn(v[i], t[i]);
    if constexpr (SIG == SIG_BIAS_RES_RELU) {
      float r[16];
      res16(1, r);
#pragma unroll
      for (int i = 0; i < 16; ++i) v[i] = __fadd_rn(v[i], r[i]);
    }
    if constexpr (SIG == SIG_BIAS_RELU || SIG == SIG_BIAS_RELU_REQ || SIG == SIG_BIAS_RES_RELU) {
#pragma unroll
      for (int i = 0; i < 16; ++i) v[i] = relu_ref(v[i]);
    }
    if constexpr (SIG == SIG_BIAS_RELU_REQ) {
      const QDev qd = e.q[2];
#pragma unroll
      for (int i = 0; i < 16; ++i) code[i] = quant_code_fast(v[i], qd);
      // v (= code * c2) is only needed for a side output, never emitted here
    }
  }
  char* prim = static_cast<char*>(o.primary);
  if (pf == FMT_I8) {
    uint4 u = make_uint4(pack4_i8(code[0], code[1], code[2], code[3]), pack4_i8(code[4], code[5], code[6], code[7]),
                         pack4_i8(code[8], code[9], code[10], code[11]), pack4_i8(code[12], code[13], code[14], code[15]));
    *reinterpret_cast<uint4*>(prim + (static_cast<int64_t>(c0 / 16) * o.plan.Pp + q) * 16) = u;
  } else if (pf == FMT_F32) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      *reinterpret_cast<float4*>(prim + (static_cast<int64_t>(c0 / 4 + j) * o.plan.Pp + q) * 16) =
          make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
  } else {
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      uint32_t w4[4];
#pragma unroll
      for (int h = 0; h < 4; ++h)
        w4[h] = static_cast<uint32_t>(f32_to_bf16(v[8 * j + 2 * h])) |
                (static_cast<uint32_t>(f32_to_bf16(v[8 * j + 2 * h + 1])) << 16);
      *reinterpret_cast<uint4*>(prim + (static_cast<int64_t>(c0 / 8 + j) * o.plan.Pp + q) * 16) =
          make_uint4(w4[0], w4[1], w4[2], w4[3]);
    }
  }
  if (o.side) {
    int sc[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) sc[i] = quant_code_fast(v[i], o.side_q);
    uint4 u = make_uint4(pack4_i8(sc[0], sc[1], sc[2], sc[3]), pack4_i8(sc[4], sc[5], sc[6], sc[7]),
                         pack4_i8(sc[8], sc[9], sc[10], sc[11]), pack4_i8(sc[12], sc[13], sc[14], sc[15]));
    *reinterpret_cast<uint4*>(reinterpret_cast<char*>(o.side) + (static_cast<int64_t>(c0 / 16) * o.slay.Pp + q) * 16) = u;
  }
}

template <int EB, int SIG>
__global__ void __launch_bounds__(kThreadsTc, 1)
    k_conv_tc(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, const TcArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // carve: [B resident or B stages][A stages][barriers]
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* smB = base;
  uint8_t* smA = smB + (a.resident_b ? a.b_res_bytes : a.b_stage_bytes * a.n_stages);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smA + a.a_stage_bytes * a.n_stages);
  uint64_t* full = bars;
  uint64_t* empty = bars + a.n_stages;
  uint64_t* tfull = bars + 2 * a.n_stages;
  uint64_t* tempty = tfull + 2;
  uint64_t* bfull = tempty + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bfull + 1);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int n_tile = blockIdx.x % a.n_tiles;
  const int m_start = blockIdx.x / a.n_tiles;
  const int m_step = gridDim.x / a.n_tiles;
  const uint32_t tmem_cols = a.bn * 2 <= 32 ? 32 : a.bn * 2 <= 64 ? 64 : a.bn * 2 <= 128 ? 128 : a.bn * 2 <= 256 ? 256 : 512;

  if (threadIdx.x == 0) {
    for (int i = 0; i < a.n_stages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], kEpiWarps);
    }
    mbar_init(bfull, 1);
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

  if (warp == 0) {
    if (lane == 0) {
      // ===== TMA producer =====
      if (a.resident_b) {
        mbar_expect_tx(bfull, a.b_res_bytes);
        tma_load_4d(smB, &tmB, bfull, 0, n_tile * a.bn, 0, 0);
      }
      int stage = 0;
      uint32_t phase = 0;
      for (int mt = m_start; mt < a.m_tiles; mt += m_step) {
        const int64_t q0 = static_cast<int64_t>(mt) * kTileM;
        const int row0 = static_cast<int>(q0 - (a.taps > 1 ? a.Wp + 1 : 0));
        for (int ks = 0; ks < a.k_stages; ++ks) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* dA = smA + stage * a.a_stage_bytes;
          mbar_expect_tx(&full[stage], a.a_stage_bytes + (a.resident_b ? 0 : a.b_stage_bytes));
          tma_load_3d(dA, &tmA, &full[stage], 0, row0, ks * a.pps);
          if (!a.resident_b)
            tma_load_4d(smB + stage * a.b_stage_bytes, &tmB, &full[stage], 0, n_tile * a.bn, ks * a.pps, 0);
          if (++stage == a.n_stages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ===== MMA issuer (one thread) =====
      if (a.resident_b) mbar_wait(bfull, 0);
      const uint32_t a_plane = static_cast<uint32_t>(a.halo) * 16;  // LBO of A
      const uint32_t b_plane = static_cast<uint32_t>(a.bn) * 16;    // LBO of B
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int mt = m_start; mt < a.m_tiles; mt += m_step) {
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + static_cast<uint32_t>(acc * a.bn);
        for (int ks = 0; ks < a.k_stages; ++ks) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t sA = smem_u32(smA + stage * a.a_stage_bytes);
          const uint32_t sB = a.resident_b ? smem_u32(smB) : smem_u32(smB + stage * a.b_stage_bytes);
          for (int t = 0; t < a.taps; ++t) {
            for (int kp = 0; kp < a.pps; kp += 2) {
              const uint32_t aaddr = sA + static_cast<uint32_t>(kp) * a_plane + static_cast<uint32_t>(a.delta[t]) * 16;
              uint32_t bplane;
              if (a.resident_b) bplane = static_cast<uint32_t>(t * a.Cc + ks * a.pps + kp);
              else bplane = static_cast<uint32_t>(t * a.pps + kp);
              const uint32_t baddr = sB + bplane * b_plane;
              const uint32_t accum = (ks | t | kp) != 0 ? 1u : 0u;
              umma<EB>(tmem_d, umma_desc(aaddr, a_plane, 128), umma_desc(baddr, b_plane, 128), a.idesc, accum);
            }
          }
          umma_commit(&empty[stage]);  // frees the smem stage when these MMAs retire
          if (++stage == a.n_stages) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit(&tfull[acc]);  // accumulator ready for the epilogue
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else {
    // ===== epilogue warps =====
    // warp w (2..9): TMEM lane quarter w % 4 (hardware lane-access rule),
    // column half (w - 2) / 4.
    const int quarter = warp & 3;
    const int half = (warp - 2) >> 2;
    const int row = quarter * 32 + lane;
    const int cols = a.bn / 2;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int mt = m_start; mt < a.m_tiles; mt += m_step) {
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const int64_t q = static_cast<int64_t>(mt) * kTileM + row;
      bool valid = q < a.Pp;
      bool border = true;
      if (valid) {
        int wp = static_cast<int>(q % a.Wp);
        int hp = static_cast<int>((q / a.Wp) % a.Hp);
        border = wp == 0 || wp == a.Wp - 1 || hp == 0 || hp == a.Hp - 1;
      }
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) +
                             static_cast<uint32_t>(acc * a.bn + half * cols);
      for (int c = 0; c < cols; c += 16) {
        uint32_t raw[16];
        tmem_ld16(taddr + static_cast<uint32_t>(c), raw);  // warp-collective: every lane executes it
        if (valid) epilogue_chunk<EB, SIG>(a, raw, q, border, n_tile * a.bn + half * cols + c);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(tmem_cols));
  }
}

// ---- host side -------------------------------------------------------------------------

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

}  // namespace

struct TcConvPlan {
  ConvGeom g;
  int eb;
  TcArgs args;
  int grid;
  size_t smem;
  const void* map_x = nullptr;
  const void* map_w = nullptr;
  CUtensorMap tmA, tmB;
};

static bool choose(TcConvPlan& p) {
  const ConvGeom& g = p.g;
  const int eb = p.eb;
  const int cpc = 16 / eb;
  TcArgs& a = p.args;
  std::memset(&a, 0, sizeof(a));
  if (g.sh != 1 || g.sw != 1) return false;
  bool k3 = g.KH == 3 && g.KW == 3 && g.ph == 1 && g.pw == 1;
  bool k1 = g.KH == 1 && g.KW == 1 && g.ph == 0 && g.pw == 0;
  if (!k3 && !k1) return false;
  if (g.OH != g.H || g.OW != g.W) return false;
  if (g.C % (2 * cpc) != 0) return false;  // whole 32-byte MMA K steps, no stale chunk lanes
  if (g.OC % 16 != 0) return false;
  a.Wp = g.W + 2 * kPad;
  a.Hp = g.H + 2 * kPad;
  a.H = g.H;
  a.W = g.W;
  a.Pp = static_cast<int64_t>(g.N) * a.Hp * a.Wp;
  a.taps = k3 ? 9 : 1;
  int halo = k3 ? kTileM + 2 * a.Wp + 2 : kTileM;
  halo = (halo + 7) / 8 * 8;
  if (halo > 256) return false;  // one TMA box per plane
  a.halo = halo;
  for (int kh = 0, t = 0; kh < g.KH; ++kh)
    for (int kw = 0; kw < g.KW; ++kw, ++t) a.delta[t] = k3 ? kh * a.Wp + kw : 0;
  a.Cc = g.C / cpc;
  a.m_tiles = static_cast<int>((a.Pp + kTileM - 1) / kTileM);
  // tile N: largest of 256/128/64/32/16 dividing OC
  int bn = 0;
  for (int c : {256, 128, 64, 32, 16})
    if (g.OC % c == 0) {
      bn = c;
      break;
    }
  if (!bn) return false;
  // resident weights if they fit beside >= 3 A stages, else stream them
  const int barrier_bytes = 256;
  auto a_stage = [&](int pps) { return pps * halo * 16; };
  int best = -1;
  for (int cand_bn = bn; cand_bn >= 16; cand_bn /= 2) {
    if (g.OC % cand_bn) continue;
    int b_res = a.taps * a.Cc * cand_bn * 16;
    for (int pps : {8, 4, 2}) {
      if (a.Cc % pps) continue;
      int ns = (kSmemBudget - barrier_bytes - b_res) / a_stage(pps);
      if (ns >= 3) {
        a.bn = cand_bn;
        a.resident_b = 1;
        a.b_res_bytes = b_res;
        a.pps = pps;
        a.n_stages = ns > 8 ? 8 : ns;
        best = 1;
        break;
      }
    }
    if (best > 0) break;
    if (cand_bn <= 64) break;  // below 64 columns prefer streaming B at a wide tile
  }
  if (best < 0) {
    a.bn = bn > 256 ? 256 : bn;
    a.resident_b = 0;
    for (int pps : {4, 2}) {
      if (a.Cc % pps) continue;
      int bst = a.taps * pps * a.bn * 16;
      int ns = (kSmemBudget - barrier_bytes) / (a_stage(pps) + bst);
      if (ns >= 2) {
        a.pps = pps;
        a.b_stage_bytes = bst;
        a.n_stages = ns > 6 ? 6 : ns;
        best = 2;
        break;
      }
    }
    if (best < 0) return false;
  }
  a.a_stage_bytes = a_stage(a.pps);
  a.k_stages = a.Cc / a.pps;
  a.n_tiles = g.OC / a.bn;
  // instruction descriptor: D fmt [4,6), A fmt [7,10), B fmt [10,13), K-major A/B,
  // N>>3 [17,23), M>>4 [24,29)
  uint32_t idesc = 0;
  if (eb == 1) idesc |= (2u << 4) | (1u << 7) | (1u << 10);  // S32 <- s8 x s8
  else idesc |= (1u << 4) | (1u << 7) | (1u << 10);          // F32 <- bf16 x bf16
  idesc |= static_cast<uint32_t>(a.bn >> 3) << 17;
  idesc |= static_cast<uint32_t>(kTileM >> 4) << 24;
  a.idesc = idesc;
  int sms = 148;
  int dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int per_n = sms / a.n_tiles;
  if (per_n < 1) per_n = 1;
  if (per_n > a.m_tiles) per_n = a.m_tiles;
  p.grid = per_n * a.n_tiles;
  int body = a.resident_b ? a.b_res_bytes : a.b_stage_bytes * a.n_stages;
  p.smem = 1024 + body + a.a_stage_bytes * a.n_stages + barrier_bytes;
  return true;
}

bool tc_conv_eligible(const ConvGeom& g, int elem_bytes) {
  TcConvPlan p;
  p.g = g;
  p.eb = elem_bytes;
  return choose(p);
}

TcConvPlan* tc_conv_create(const ConvGeom& g, int elem_bytes) {
  auto* p = new TcConvPlan();
  p->g = g;
  p->eb = elem_bytes;
  if (!choose(*p) || !encode_fn()) {
    delete p;
    return nullptr;
  }
  return p;
}

static bool encode_maps(TcConvPlan& p, const void* x, const void* w) {
  TcArgs& a = p.args;
  auto enc = encode_fn();
  // A: [planes][pixels][16 B] -> dims {16, Pp, Cc}, box {16, halo, pps}
  {
    cuuint64_t dims[3] = {16, static_cast<cuuint64_t>(a.Pp), static_cast<cuuint64_t>(a.Cc)};
    cuuint64_t strides[2] = {16, static_cast<cuuint64_t>(a.Pp) * 16};
    cuuint32_t box[3] = {16, static_cast<cuuint32_t>(a.halo), static_cast<cuuint32_t>(a.pps)};
    cuuint32_t es[3] = {1, 1, 1};
    if (enc(&p.tmA, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<void*>(x), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return false;
  }
  // B: [taps][planes][OC][16 B] -> dims {16, OC, Cc, taps}
  {
    cuuint64_t dims[4] = {16, static_cast<cuuint64_t>(p.g.OC), static_cast<cuuint64_t>(a.Cc),
                          static_cast<cuuint64_t>(a.taps)};
    cuuint64_t strides[3] = {16, static_cast<cuuint64_t>(p.g.OC) * 16,
                             static_cast<cuuint64_t>(p.g.OC) * 16 * static_cast<cuuint64_t>(a.Cc)};
    cuuint32_t box[4] = {16, static_cast<cuuint32_t>(a.bn),
                         static_cast<cuuint32_t>(a.resident_b ? a.Cc : a.pps), static_cast<cuuint32_t>(a.taps)};
    cuuint32_t es[4] = {1, 1, 1, 1};
    if (enc(&p.tmB, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<void*>(w), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return false;
  }
  p.map_x = x;
  p.map_w = w;
  return true;
}

bool tc_conv_launch(TcConvPlan* p, const void* x, const void* w, float acc_scale, const EpiDev& epi,
                    const OutDev& out, cudaStream_t s) {
  if (p->map_x != x || p->map_w != w) {
    if (!encode_maps(*p, x, w)) return false;
  }
  TcArgs a = p->args;
  a.acc_scale = acc_scale;
  a.epi = epi;
  a.out = out;
  const int sig = epi_signature(epi, out);
#define MRB_TC_LAUNCH(EB_, SIG_)                                                                          \
  do {                                                                                                    \
    cudaFuncSetAttribute(k_conv_tc<EB_, SIG_>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(p->smem)); \
    k_conv_tc<EB_, SIG_><<<p->grid, kThreadsTc, p->smem, s>>>(p->tmA, p->tmB, a);                       \
  } while (0)
#define MRB_TC_SIGS(EB_)                                          \
  switch (sig) {                                                  \
    case SIG_BIAS: MRB_TC_LAUNCH(EB_, SIG_BIAS); break;           \
    case SIG_BIAS_RELU: MRB_TC_LAUNCH(EB_, SIG_BIAS_RELU); break; \
    case SIG_BIAS_RELU_REQ: MRB_TC_LAUNCH(EB_, SIG_BIAS_RELU_REQ); break; \
    case SIG_BIAS_RES_RELU: MRB_TC_LAUNCH(EB_, SIG_BIAS_RES_RELU); break; \
    default: MRB_TC_LAUNCH(EB_, SIG_ANY); break;                  \
  }
  if (p->eb == 1) {
    MRB_TC_SIGS(1)
  } else {
    MRB_TC_SIGS(2)
  }
#undef MRB_TC_SIGS
#undef MRB_TC_LAUNCH
  return true;
}

void tc_conv_destroy(TcConvPlan* p) { delete p; }

const char* tc_conv_describe(const TcConvPlan* p, char* buf, int n) {
  const TcArgs& a = p->args;
  std::snprintf(buf, n, "tcgen05 %s M128xN%d taps=%d halo=%d pps=%d stages=%d B=%s grid=%d smem=%zu",
                p->eb == 1 ? "i8" : "bf16", a.bn, a.taps, a.halo, a.pps, a.n_stages, a.resident_b ? "resident" : "streamed",
                p->grid, p->smem);
  return buf;
}

}  // namespace mrb200
