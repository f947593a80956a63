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

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "conv_tc.hpp"

namespace mrb200 {

namespace {

constexpr int kTileM = 128;
constexpr int kEpiWarps = 16;
constexpr int kThreadsTc = (2 + kEpiWarps) * 32;
constexpr int kSmemBudget = 227 * 1024 - 1024;

enum EpiSig : int { SIG_ANY = 0, SIG_BIAS = 1, SIG_BIAS_RELU = 2, SIG_BIAS_RELU_REQ = 3, SIG_BIAS_RES_RELU = 4 };

// Compile-time epilogue for the op sequences the realize/fuse passes emit.
inline int epi_signature(const EpiDev& e, const OutDev& o) {
  auto q_ok = [](const QDev& q) {
    return q.lo >= -2147483520.f && q.hi <= 2147483520.f && q.lo == q.lo && q.hi == q.hi;
  };
  if (o.side && o.side_fmt == FMT_I8 && !q_ok(o.side_q)) return SIG_ANY;
  if (e.n_ops == 1 && e.op[0] == E_BIAS && o.primary_fmt != FMT_I8) return SIG_BIAS;
  if (e.n_ops == 2 && e.op[0] == E_BIAS && e.op[1] == E_RELU && o.primary_fmt != FMT_I8) return SIG_BIAS_RELU;
  if (e.n_ops == 3 && e.op[0] == E_BIAS && e.op[1] == E_RELU && e.op[2] == E_REQ && o.primary_fmt == FMT_I8 &&
      !o.side && q_ok(e.q[2]) && e.q[2].lo <= 0.f && e.q[2].c1 > 0.f &&
      e.q[2].hi <= (e.q[2].is_signed ? 127.f : 255.f) && e.q[2].hi >= 0.f)
    return SIG_BIAS_RELU_REQ;
  if (e.n_ops == 3 && e.op[0] == E_BIAS && e.op[1] == E_RES && e.op[2] == E_RELU && o.primary_fmt != FMT_I8)
    return SIG_BIAS_RES_RELU;
  return SIG_ANY;
}

constexpr int kMaxSteps = 40;

// One tcgen05.mma of a tile's K loop: byte offsets (relative to the A stage
// base + row shift, and to the B stage / resident base) and the leading byte
// offsets (distance between the two 16-byte K halves of the instruction).
struct MmaStep {
  uint32_t a_off, a_lbo, b_off, b_lbo;
};

enum OutMode : int32_t { OUT_SAME = 0, OUT_REMAP = 1 };

struct TcArgs {
  // M grid: the pixel grid of the A source (padded grid, phase grid, s2d grid)
  int32_t N, Hg, Wg;
  int64_t Pg;  // N*Hg*Wg
  int32_t m_tiles, n_tiles, bn, Cc, pps, k_stages, sub0, subs, hg;
  int32_t dmin;  // smallest tap row offset (tile row 0 + dmin = first halo row)
  int32_t n_steps;
  MmaStep steps[kMaxSteps];
  uint32_t b_ks_stride;  // resident B: bytes between consecutive K stages
  int32_t resident_b;
  int32_t a_stage_bytes, b_stage_bytes, b_res_bytes, n_stages;
  uint32_t idesc;
  int32_t out_mode, OH, OW;  // OUT_REMAP: valid outputs are grid (y < OH, x < OW)
  float acc_scale;
  int32_t dbg;  // MRB200_TC_DBG bit 0: skip epilogue math, bit 1: skip MMAs (timing experiments only)
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

// Where one output row (pixel) of the tile lands.
struct RowDst {
  int64_t pix;        // NORMAL padded-grid index of the output pixel (primary, residual)
  int64_t side_base;  // side chunk index of plane 0
  int64_t side_pstride;
  bool border;        // OUT_SAME: padded-grid border -> zeros
};

__device__ __forceinline__ void store16(void* base, int64_t chunk, uint4 v) {
  *reinterpret_cast<uint4*>(static_cast<char*>(base) + chunk * 16) = v;
}

// 16 channels [c0, c0+16) of one output pixel through the epilogue, stored as
// 16-byte chunks.  SIG selects a compile-time op sequence for the common
// fused groups; SIG_ANY interprets EpiDev.  The arithmetic is identical either
// way (kernels.cuh).
template <int EB, int SIG>
__device__ __forceinline__ void epilogue_chunk(const TcArgs& a, const uint32_t* raw, const RowDst& d, int c0) {
  const OutDev& o = a.out;
  const int pf = o.primary_fmt;
  const int pcpc = pf == FMT_F32 ? 4 : pf == FMT_BF16 ? 8 : 16;
  const int scpc = o.side_fmt == FMT_BF16 ? 8 : 16;
  if (d.border) {
    for (int k = 0; k < 16 / pcpc; ++k) store16(o.primary, (c0 / pcpc + k) * o.plan.Pp + d.pix, make_uint4(0, 0, 0, 0));
    if (o.side)
      for (int k = 0; k < 16 / scpc; ++k)
        store16(o.side, d.side_base + (c0 / scpc + k) * d.side_pstride, make_uint4(0, 0, 0, 0));
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
                                                    (static_cast<int64_t>(c0 / 4 + j) * L.Pp + d.pix) * 16);
        t[4 * j] = f.x; t[4 * j + 1] = f.y; t[4 * j + 2] = f.z; t[4 * j + 3] = f.w;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        uint4 u = *reinterpret_cast<const uint4*>(static_cast<const char*>(e.res[k]) +
                                                  (static_cast<int64_t>(c0 / 8 + j) * L.Pp + d.pix) * 16);
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
      // v >= +0 after relu and c1 > 0 (checked on the host), so rint(v*c1) >= 0 >= lo:
      // clip(t, lo, hi) == min(t, hi); the value is integral and < 2^31 -> exact cvt.
      const QDev qd = e.q[2];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        float t = fminf(rintf(__fmul_rn(v[i], qd.c1)), qd.hi);
        code[i] = __float2int_rz(t);
      }
      // v (= code * c2) is only needed for a side output, never emitted here
    }
  }
  if (pf == FMT_I8) {
    store16(o.primary, (c0 / 16) * o.plan.Pp + d.pix,
            make_uint4(pack4_i8(code[0], code[1], code[2], code[3]), pack4_i8(code[4], code[5], code[6], code[7]),
                       pack4_i8(code[8], code[9], code[10], code[11]), pack4_i8(code[12], code[13], code[14], code[15])));
  } else if (pf == FMT_F32) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      store16(o.primary, (c0 / 4 + j) * o.plan.Pp + d.pix,
              make_uint4(__float_as_uint(v[4 * j]), __float_as_uint(v[4 * j + 1]), __float_as_uint(v[4 * j + 2]),
                         __float_as_uint(v[4 * j + 3])));
  } else {
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      uint32_t w4[4];
#pragma unroll
      for (int h = 0; h < 4; ++h)
        w4[h] = static_cast<uint32_t>(f32_to_bf16(v[8 * j + 2 * h])) |
                (static_cast<uint32_t>(f32_to_bf16(v[8 * j + 2 * h + 1])) << 16);
      store16(o.primary, (c0 / 8 + j) * o.plan.Pp + d.pix, make_uint4(w4[0], w4[1], w4[2], w4[3]));
    }
  }
  if (o.side) {
    if (o.side_fmt == FMT_I8) {
      int sc[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) sc[i] = quant_code_fast(v[i], o.side_q);
      store16(o.side, d.side_base + (c0 / 16) * d.side_pstride,
              make_uint4(pack4_i8(sc[0], sc[1], sc[2], sc[3]), pack4_i8(sc[4], sc[5], sc[6], sc[7]),
                         pack4_i8(sc[8], sc[9], sc[10], sc[11]), pack4_i8(sc[12], sc[13], sc[14], sc[15])));
    } else {
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        uint32_t w4[4];
#pragma unroll
        for (int h = 0; h < 4; ++h)
          w4[h] = static_cast<uint32_t>(f32_to_bf16(v[8 * j + 2 * h])) |
                  (static_cast<uint32_t>(f32_to_bf16(v[8 * j + 2 * h + 1])) << 16);
        store16(o.side, d.side_base + (c0 / 8 + j) * d.side_pstride, make_uint4(w4[0], w4[1], w4[2], w4[3]));
      }
    }
  }
}

__device__ __forceinline__ int floor_div8(int v) { return v >= 0 ? v / 8 : -((7 - v) / 8); }

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
        tma_load_4d(smB, &tmB, bfull, 0, n_tile * a.bn / 8, 0, 0);
      }
      int stage = 0;
      uint32_t phase = 0;
      for (int mt = m_start; mt < a.m_tiles; mt += m_step) {
        const int row0 = mt * kTileM + a.dmin;
        const int g0 = floor_div8(row0);
        for (int ks = 0; ks < a.k_stages; ++ks) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_expect_tx(&full[stage], a.a_stage_bytes + (a.resident_b ? 0 : a.b_stage_bytes));
          tma_load_4d(smA + stage * a.a_stage_bytes, &tmA, &full[stage], 0, g0, a.sub0, ks * a.pps);
          if (!a.resident_b)
            tma_load_4d(smB + stage * a.b_stage_bytes, &tmB, &full[stage], 0, n_tile * a.bn / 8, ks * a.pps, 0);
          if (++stage == a.n_stages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ===== MMA issuer =====
    // The whole warp walks the loop so tile/stage/descriptor values are
    // warp-uniform (uniform registers); lane 0 issues tcgen05.mma / commit.
    // Descriptors: base | (start >> 4); LBO/SBO/version fixed per step.
    if (a.resident_b) mbar_wait(bfull, 0);
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    const uint32_t smB_u = smem_u32(smB);
    const uint32_t smA_u = smem_u32(smA);
    for (int mt = m_start; mt < a.m_tiles; mt += m_step) {
      const int row0 = mt * kTileM + a.dmin;
      const uint32_t shift16 = static_cast<uint32_t>(row0 - 8 * floor_div8(row0)) * 16;
      mbar_wait(&tempty[acc], acc_phase ^ 1);
      tc_fence_after();
      const uint32_t tmem_d = tmem_base + static_cast<uint32_t>(acc * a.bn);
      for (int ks = 0; ks < a.k_stages; ++ks) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        const uint32_t sA = smA_u + stage * a.a_stage_bytes + shift16;
        const uint32_t sB = a.resident_b ? smB_u + ks * a.b_ks_stride : smB_u + stage * a.b_stage_bytes;
#pragma unroll 2
        for (int st = 0; st < a.n_steps; ++st) {
          const MmaStep m = a.steps[st];
          const uint32_t aaddr = (a.dbg & 4) ? ((sA + m.a_off) & ~127u) : sA + m.a_off;
          const uint64_t ad = umma_desc(aaddr, m.a_lbo, 128);
          const uint64_t bd = umma_desc(sB + m.b_off, m.b_lbo, 128);
          if (lane == 0 && !(a.dbg & 2)) umma<EB>(tmem_d, ad, bd, a.idesc, (ks | st) != 0 ? 1u : 0u);
        }
        __syncwarp();
        if (lane == 0) umma_commit(&empty[stage]);  // frees the smem stage when these MMAs retire
        __syncwarp();
        if (++stage == a.n_stages) {
          stage = 0;
          phase ^= 1;
        }
      }
      if (lane == 0) umma_commit(&tfull[acc]);  // accumulator ready for the epilogue
      __syncwarp();
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  } else {
    // ===== epilogue warps =====
    // warp w (2..17): TMEM lane quarter w % 4 (hardware lane-access rule),
    // 16-column chunks slice, slice + 4, ... with slice = (w - 2) / 4.
    const int quarter = warp & 3;
    const int slice = (warp - 2) >> 2;
    const int row = quarter * 32 + lane;
    const Lay& sl = a.out.slay;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int mt = m_start; mt < a.m_tiles; mt += m_step) {
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t q = static_cast<uint32_t>(mt) * kTileM + row;  // grids < 2^31 pixels (checked on the host)
      RowDst d;
      bool valid = q < static_cast<uint32_t>(a.Pg);
      d.border = false;
      d.pix = 0;
      if (valid) {
        const uint32_t t = q / static_cast<uint32_t>(a.Wg);
        const int x = static_cast<int>(q - t * static_cast<uint32_t>(a.Wg));
        const uint32_t n32 = t / static_cast<uint32_t>(a.Hg);
        const int y = static_cast<int>(t - n32 * static_cast<uint32_t>(a.Hg));
        const int n = static_cast<int>(n32);
        if (a.out_mode == OUT_SAME) {
          d.pix = q;
          d.border = x == 0 || x == a.Wg - 1 || y == 0 || y == a.Hg - 1;
        } else {
          valid = y < a.OH && x < a.OW;
          d.pix = (static_cast<int64_t>(n) * (a.OH + 2 * kPad) + y + kPad) * (a.OW + 2 * kPad) + x + kPad;
        }
        if (a.out.side) {
          if (sl.kind == LAY_PHASE) {
            const uint32_t p32 = static_cast<uint32_t>(d.pix);
            const uint32_t tt = p32 / static_cast<uint32_t>(sl.Wp);
            const int wp = static_cast<int>(p32 - tt * static_cast<uint32_t>(sl.Wp));
            const uint32_t nn = tt / static_cast<uint32_t>(sl.Hp);
            const int hp = static_cast<int>(tt - nn * static_cast<uint32_t>(sl.Hp));
            d.side_base = static_cast<int64_t>((hp & 1) * 2 + (wp & 1)) * sl.Pp +
                          (static_cast<int64_t>(nn) * sl.Hq + hp / 2) * sl.Wq + wp / 2;
            d.side_pstride = 4 * sl.Pp;
          } else {
            d.side_base = d.pix;
            d.side_pstride = sl.Pp;
          }
        }
      }
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + static_cast<uint32_t>(acc * a.bn);
      for (int c = slice * 16; c < a.bn; c += 64) {
        uint32_t raw[16];
        tmem_ld16(taddr + static_cast<uint32_t>(c), raw);  // warp-collective: every lane executes it
        if (valid && !(a.dbg & 1)) epilogue_chunk<EB, SIG>(a, raw, d, n_tile * a.bn + c);
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
  TcConvSpec spec;
  TcArgs args;
  int grid = 0;
  size_t smem = 0;
  const void* map_x = nullptr;
  const void* map_w = nullptr;
  CUtensorMap tmA, tmB;
};

// Taps of a conv kind: (sub-grid, row offset in the sub-grid's pixel space).
struct Tap {
  int sub, delta;
};

static bool choose(TcConvPlan& p) {
  const TcConvSpec& sp = p.spec;
  TcArgs& a = p.args;
  std::memset(&a, 0, sizeof(a));
  const int eb = sp.elem_bytes;
  const int cpc = 16 / eb;
  if (sp.OC % 16 != 0) return false;
  std::vector<Tap> taps;
  int cc = 0;       // A chunk planes
  bool pair_taps = false;  // int8 stem: K halves = two adjacent taps (LBO 16 B)
  a.N = sp.N;
  switch (sp.kind) {
    case TC_S1: {
      // stride-1 3x3/pad-1 or 1x1/pad-0 over the NORMAL padded grid; output
      // grid == input grid
      bool k3 = sp.KH == 3 && sp.KW == 3, k1 = sp.KH == 1 && sp.KW == 1;
      if (!k3 && !k1) return false;
      if (sp.C % (2 * cpc)) return false;
      a.Hg = sp.H + 2 * kPad;
      a.Wg = sp.W + 2 * kPad;
      a.out_mode = OUT_SAME;
      cc = sp.C / cpc;
      a.subs = 1;
      for (int kh = 0; kh < sp.KH; ++kh)
        for (int kw = 0; kw < sp.KW; ++kw) taps.push_back({0, k3 ? (kh - 1) * a.Wg + (kw - 1) : 0});
      break;
    }
    case TC_S2_PHASE: {
      // stride-2 3x3/pad-1 (4 phases) or 1x1/pad-0 (phase (1,1)) over the
      // PHASE layout: tap (kh, kw) reads sub-grid (kh&1, kw&1) at (kh/2, kw/2)
      bool k3 = sp.KH == 3 && sp.KW == 3, k1 = sp.KH == 1 && sp.KW == 1;
      if (!k3 && !k1) return false;
      if (sp.C % (2 * cpc)) return false;
      if ((sp.H & 1) || (sp.W & 1)) return false;
      a.Hg = (sp.H + 2 * kPad + 1) / 2;
      a.Wg = (sp.W + 2 * kPad + 1) / 2;
      a.out_mode = OUT_REMAP;
      a.OH = sp.OH;
      a.OW = sp.OW;
      cc = sp.C / cpc;
      a.subs = 4;
      if (k3) {
        for (int kh = 0; kh < 3; ++kh)
          for (int kw = 0; kw < 3; ++kw) taps.push_back({(kh & 1) * 2 + (kw & 1), (kh / 2) * a.Wg + kw / 2});
      } else {
        a.sub0 = 3;  // only phase (1, 1) is read: load just that sub-grid
        a.subs = 1;
        taps.push_back({0, 0});
      }
      break;
    }
    case TC_STEM_S2D: {
      // KxK stride-2 over the space-to-depth input: TA x TA stride-1 taps of
      // 4*C s2d channels; output (oh, ow) at s2d grid (oh, ow)
      const int TA = (sp.KH + 1) / 2;
      if (sp.KH != sp.KW || 4 * sp.C > 16) return false;
      a.Hg = sp.Hs;
      a.Wg = sp.Ws;
      a.out_mode = OUT_REMAP;
      a.OH = sp.OH;
      a.OW = sp.OW;
      cc = (4 * sp.C + cpc - 1) / cpc;  // 1 (int8) or 2 (bf16)
      a.subs = 1;
      for (int ta = 0; ta < TA; ++ta)
        for (int tb = 0; tb < TA; ++tb) taps.push_back({0, ta * a.Wg + tb});
      pair_taps = cc == 1;
      if (pair_taps && (TA & 1)) return false;
      break;
    }
    default:
      return false;
  }
  a.Pg = static_cast<int64_t>(a.N) * a.Hg * a.Wg;
  if (a.Pg + kTileM >= (int64_t(1) << 31)) return false;
  a.m_tiles = static_cast<int>((a.Pg + kTileM - 1) / kTileM);
  int dmin = 1 << 30, dmax = -(1 << 30);
  for (const Tap& t : taps) {
    dmin = std::min(dmin, t.delta);
    dmax = std::max(dmax, t.delta + (pair_taps ? 1 : 0));
  }
  a.dmin = dmin;
  a.hg = (7 + kTileM + dmax - dmin + 7) / 8;  // 8-pixel rows per sub-grid and plane
  if (a.hg > 256) return false;
  const int ntaps = static_cast<int>(taps.size());
  // weights (TMA B): [ntaps][cc][OC][16 B]
  const int barrier_bytes = 256;
  auto a_stage = [&](int pps) { return pps * a.subs * a.hg * 128; };
  auto steps_for = [&](int pps) { return pair_taps ? ntaps / 2 : ntaps * pps / 2; };
  int bn = 0;
  for (int c : {256, 128, 64, 32, 16})
    if (sp.OC % c == 0) {
      bn = c;
      break;
    }
  if (!bn) return false;
  bool found = false;
  static const int force_stream = [] {
    const char* e = std::getenv("MRB200_TC_STREAM");
    return e ? std::atoi(e) : 0;
  }();
  // resident weights if they fit beside >= 3 A stages, else stream them
  for (int cand = bn; cand >= 16 && !found && !force_stream; cand /= 2) {
    if (sp.OC % cand) continue;
    int b_res = ntaps * cc * cand * 16;
    for (int pps : {8, 4, 2, 1}) {
      if (cc % pps || (pps & 1 && !pair_taps) || steps_for(pps) > kMaxSteps) continue;
      int ns = (kSmemBudget - barrier_bytes - b_res) / a_stage(pps);
      if (ns >= 3) {
        a.bn = cand;
        a.resident_b = 1;
        a.b_res_bytes = b_res;
        a.pps = pps;
        a.n_stages = ns > 8 ? 8 : ns;
        found = true;
        break;
      }
    }
    if (cand <= 64) break;  // below 64 columns prefer streaming B at a wide tile
  }
  if (!found) {
    a.bn = bn > 256 ? 256 : bn;
    a.resident_b = 0;
    for (int pps : {4, 2}) {
      if (cc % pps || pair_taps || steps_for(pps) > kMaxSteps) continue;
      int bst = ntaps * pps * a.bn * 16;
      int ns = (kSmemBudget - barrier_bytes) / (a_stage(pps) + bst);
      if (ns >= 2) {
        a.pps = pps;
        a.b_stage_bytes = bst;
        a.n_stages = ns > 6 ? 6 : ns;
        found = true;
        break;
      }
    }
    if (!found) return false;
  }
  a.Cc = cc;
  a.a_stage_bytes = a_stage(a.pps);
  a.k_stages = cc / a.pps;
  a.n_tiles = sp.OC / a.bn;
  // MMA step table (byte offsets; A relative to stage base + row shift)
  const uint32_t a_sub = static_cast<uint32_t>(a.hg) * 128;
  const uint32_t a_plane = a_sub * static_cast<uint32_t>(a.subs);
  const uint32_t b_plane = static_cast<uint32_t>(a.bn) * 16;
  const int bplanes = a.resident_b ? cc : a.pps;  // planes per tap in the smem B buffer
  a.b_ks_stride = a.resident_b ? static_cast<uint32_t>(a.pps) * b_plane : 0;
  a.n_steps = 0;
  if (pair_taps) {
    for (int t = 0; t < ntaps; t += 2) {
      MmaStep m;
      m.a_off = static_cast<uint32_t>(taps[t].delta - dmin) * 16;
      m.a_lbo = 16;
      m.b_off = static_cast<uint32_t>(t * bplanes) * b_plane;
      m.b_lbo = static_cast<uint32_t>(bplanes) * b_plane;
      a.steps[a.n_steps++] = m;
    }
  } else {
    for (int t = 0; t < ntaps; ++t)
      for (int kp = 0; kp < a.pps; kp += 2) {
        MmaStep m;
        m.a_off = static_cast<uint32_t>(kp) * a_plane + static_cast<uint32_t>(taps[t].sub) * a_sub +
                  static_cast<uint32_t>(taps[t].delta - dmin) * 16;
        m.a_lbo = a_plane;
        m.b_off = static_cast<uint32_t>(t * bplanes + kp) * b_plane;
        m.b_lbo = b_plane;
        a.steps[a.n_steps++] = m;
      }
  }
  p.spec.taps = ntaps;
  p.spec.wplanes = cc;
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

bool tc_conv_plan_ok(TcConvSpec& spec) {
  TcConvPlan p;
  p.spec = spec;
  if (!choose(p)) return false;
  spec = p.spec;
  return true;
}

TcConvPlan* tc_conv_create(const TcConvSpec& spec) {
  auto* p = new TcConvPlan();
  p->spec = spec;
  if (!choose(*p) || !encode_fn()) {
    delete p;
    return nullptr;
  }
  return p;
}

static bool encode_maps(TcConvPlan& p, const void* x, const Lay& xl, const void* w) {
  TcArgs& a = p.args;
  auto enc = encode_fn();
  // A: chunk planes of `subs` sub-grids of Pp pixels (multiple of 8) x 16 B,
  // moved as 128-byte (8-pixel) rows: dims {128 B, Pp/8, subs, Cc}
  {
    const cuuint64_t tsubs = xl.kind == LAY_PHASE ? 4 : 1;
    cuuint64_t dims[4] = {128, static_cast<cuuint64_t>(xl.Pp / 8), tsubs, static_cast<cuuint64_t>(a.Cc)};
    cuuint64_t strides[3] = {128, static_cast<cuuint64_t>(xl.Pp) * 16, static_cast<cuuint64_t>(xl.Pp) * 16 * tsubs};
    cuuint32_t box[4] = {128, static_cast<cuuint32_t>(a.hg), static_cast<cuuint32_t>(a.subs),
                         static_cast<cuuint32_t>(a.pps)};
    cuuint32_t es[4] = {1, 1, 1, 1};
    if (enc(&p.tmA, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<void*>(x), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return false;
  }
  // B: [taps][planes][OC][16 B] -> dims {128 B (8 rows), OC/8, planes, taps}
  {
    const int OC = p.spec.OC;
    cuuint64_t dims[4] = {128, static_cast<cuuint64_t>(OC / 8), static_cast<cuuint64_t>(a.Cc),
                          static_cast<cuuint64_t>(p.spec.taps)};
    cuuint64_t strides[3] = {128, static_cast<cuuint64_t>(OC) * 16, static_cast<cuuint64_t>(OC) * 16 * a.Cc};
    cuuint32_t box[4] = {128, static_cast<cuuint32_t>(a.bn / 8),
                         static_cast<cuuint32_t>(a.resident_b ? a.Cc : a.pps), static_cast<cuuint32_t>(p.spec.taps)};
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

bool tc_conv_launch(TcConvPlan* p, const void* x, const Lay& xl, const void* w, float acc_scale, const EpiDev& epi,
                    const OutDev& out, cudaStream_t s) {
  if (p->map_x != x || p->map_w != w) {
    if (!encode_maps(*p, x, xl, w)) return false;
  }
  TcArgs a = p->args;
  a.acc_scale = acc_scale;
  static const int dbg = [] {
    const char* e = std::getenv("MRB200_TC_DBG");
    return e ? std::atoi(e) : 0;
  }();
  a.dbg = dbg;
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
  if (p->spec.elem_bytes == 1) {
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
  static const char* kinds[] = {"s1", "s2-phase", "stem-s2d"};
  std::snprintf(buf, n, "tcgen05 %s %s M128xN%d taps=%d steps=%d grid=%dx%d hg=%d pps=%d stages=%d B=%s ctas=%d smem=%zu",
                p->spec.elem_bytes == 1 ? "i8" : "bf16", kinds[p->spec.kind], a.bn, p->spec.taps, a.n_steps, a.Hg,
                a.Wg, a.hg, a.pps, a.n_stages, a.resident_b ? "resident" : "streamed", p->grid, p->smem);
  return buf;
}

}  // namespace mrb200
