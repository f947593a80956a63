// kernels.cuh -- device-side parameter blocks shared by every kernel and the
// host executor, plus the bit-exact epilogue arithmetic.
//
// Arithmetic mirrors the reference kernels (core/src/kernels.cpp):
//  * multiply / add on float32 compute in double and round once
//    (binary_broadcast, kernels.cpp:94-131) == IEEE __fmul_rn / __fadd_rn;
//  * bias_add is a float add (kernels.cpp:731);
//  * relu is `x > 0 ? x : 0.0f` (kernels.cpp:285), so -0 -> +0 and NaN -> 0;
//  * round is nearbyintf under FE_TONEAREST = rintf (kernels.cpp:288-294);
//  * clip is std::min(std::max(x, lo), hi) with float bounds (kernels.cpp:306-307);
//  * cast f32->int8 truncates then wraps (kernels.cpp:320-348).
// Everything is compiled with -fmad=false, no fast-math, denormals kept.
#pragma once

#include <cstdint>

namespace mrb200 {

enum Fmt : int32_t { FMT_F32 = 0, FMT_BF16 = 1, FMT_I8 = 2 };

struct QDev {
  float c1, lo, hi, c2;
  int32_t is_signed;
  // calibration (mr_calibrate): when set, every quantization of a value x
  // raises *ovf if the site would overflow -- quant_calibrate's observer,
  // |nearbyint(x / rho * 2^(bits-sign))| > 2^(bits-1) (signed) or outside
  // [0, 2^bits] (unsigned) (quantize.cpp:149-161)
  int32_t* ovf;
};

// Physical layout of an activation tensor ("PK"): channels are split into
// chunks of kb bytes (kb = 16, 64 or 128; cpc = kb / element-bytes channels
// each); each chunk is a plane over the zero-padded pixel grid (pad kPad):
//   LAY_NORMAL  element (n, c, h, w) at ((c / cpc) * Pp + pix) * cpc + c % cpc,
//               pix = (n * Hp + h + kPad) * Wp + (w + kPad)
//   LAY_PHASE   the padded grid split into its 4 stride-2 phases, so a
//               stride-2 conv reads each phase with stride 1: padded pixel
//               (hp, wp) -> sub-grid (hp & 1) * 2 + (wp & 1), position
//               (n * Hq + hp / 2) * Wq + wp / 2; sub-grids of Pp pixels
//   LAY_S2D     the network input in space-to-depth form for a 7x7/s2 stem
//               (written by input_convert, read by the stem tcgen05 conv only)
//   LAY_S2DP    LAY_S2D shifted by 2 s2d pixels (zero rows/columns on top and
//               left) and split into its 4 stride-2 phase sub-grids of Hq x Wq:
//               s2d pixel (si, sj) -> sub-grid ((si+2)&1)*2 + ((sj+2)&1),
//               position (n*Hq + (si+2)/2)*Wq + (sj+2)/2, sub-grid stride Pp.
//               Read by the fused stem + 3x3/s2 max_pool2d kernel, whose M
//               rows are pooled pixels (conv_tc.cu TC_STEM_POOL).
// A pixel's kb-byte chunk is one row of a tcgen05 operand tile: kb = 128 / 64
// rows are TMA-loaded with the matching 128B / 64B swizzle, and a stride-1
// 3x3 conv reads its 9 taps as 9 row shifts of one contiguous pixel range
// (conv_tc.cu).  kb = 16 ("P16") is used where no tensor-core conv reads the
// tensor (float32 residual stream: warp-coalesced epilogue loads) and for the
// 16-byte stem input.  Plane strides are padded to a multiple of 8 pixels.
// Borders hold zeros.  cpc == 0 marks a plain row-major [N, C] tensor (pix = n).
enum LayKind : int32_t { LAY_NORMAL = 0, LAY_PHASE = 1, LAY_S2D = 2, LAY_S2DP = 3 };

struct Lay {
  int32_t cpc;
  int32_t C;     // logical channels (row length when cpc == 0)
  int64_t Pp;    // pixel stride of a plane (NORMAL) / sub-grid (PHASE, S2D)
  int32_t kind;  // LayKind
  int32_t kb;    // chunk bytes
  int32_t Hp, Wp;  // padded grid
  int32_t Hq, Wq;  // PHASE / S2D sub-grid
};

enum EpiCode : int32_t {
  E_MULS = 1, E_MULC = 2, E_BIAS = 3, E_RES = 4, E_RELU = 5, E_REQ = 6, E_CLIP = 7
};

constexpr int kMaxEpi = 8;

struct EpiDev {
  int32_t n_ops;
  int32_t op[kMaxEpi];
  float s[kMaxEpi];          // MulScalar / Clip lo
  float s2[kMaxEpi];         // Clip hi
  const float* vec[kMaxEpi]; // MulChannel / Bias, [C]
  const void* res[kMaxEpi];  // Residual tensor (same pixel grid as the output)
  int32_t res_fmt[kMaxEpi];
  Lay res_lay[kMaxEpi];
  QDev q[kMaxEpi];
};

// Where a kernel writes its (per element) final value.
struct OutDev {
  void* primary;        // P16 (or row-major [N, C])
  int32_t primary_fmt;  // FMT_I8 => the epilogue's last op is a Requant; the code is stored
  Lay plan;             // primary layout
  void* side;           // optional second copy of the final float value for other consumers:
  int32_t side_fmt;     //   FMT_I8 (realize codes with side_q), FMT_BF16 or (tf32 mode) FMT_F32, any kind
  Lay slay;
  QDev side_q;
  int32_t tf32;         // tf32 mode: float32 activations are stored rounded to tf32 (the tensor
                        //   cores read only the top 19 bits; truncation would bias every product)
  // optional stride-2 decimated copy of the int8 side codes (tcgen05 conv only):
  // pixel (2i, 2j) of the image -> (i, j) of the LAY_NORMAL layout s2lay, the
  // A2 operand of a consumer conv with a fused 1x1/stride-2 shortcut
  void* side2;
  Lay s2lay;
};

// Division by a launch-constant divisor d for dividends n < 2^31 as a
// multiply-high and a shift (round-up magic number: s = ceil(log2 d),
// m = ceil(2^(31+s) / d) < 2^32; exact for every n < 2^31).
struct FastDiv {
  uint32_t d, m;
  int32_t s;  // -1: d == 1
};

inline FastDiv make_fastdiv(uint32_t d) {
  FastDiv f{d, 0u, -1};
  if (d <= 1) return f;
  int s = 0;
  while ((1ull << s) < d) ++s;
  f.s = s;
  f.m = static_cast<uint32_t>(((1ull << (31 + s)) + d - 1) / d);
  return f;
}

#ifdef __CUDACC__

// Programmatic dependent launch: every graph kernel lets the next one start
// its independent prologue at once (trigger) and waits for the previous
// kernel's results before touching activations (wait; a no-op without PDL).
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ uint32_t fdiv(uint32_t n, const FastDiv& f) {
  return f.s < 0 ? n : (__umulhi(n, f.m) >> (f.s - 1));
}

__device__ __forceinline__ float bf16_to_f32(uint16_t h) { return __uint_as_float(static_cast<uint32_t>(h) << 16); }

// Round-to-nearest-even float -> bf16 (NaN kept quiet).
__device__ __forceinline__ uint16_t f32_to_bf16(float f) {
  uint32_t u = __float_as_uint(f);
  if ((u & 0x7fffffffu) > 0x7f800000u) return static_cast<uint16_t>((u >> 16) | 0x40);
  u += 0x7fffu + ((u >> 16) & 1u);
  return static_cast<uint16_t>(u >> 16);
}

// Two floats -> packed bf16x2 (lo in the low half), round to nearest even in one
// cvt (the bf16 pipeline's stores; matches f32_to_bf16 except NaN payloads).
__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
#ifdef MRB200_NO_BF16X2_CVT
  return static_cast<uint32_t>(f32_to_bf16(lo)) | (static_cast<uint32_t>(f32_to_bf16(hi)) << 16);
#else
  uint32_t d;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(hi), "f"(lo));
  return d;
#endif
}

__device__ __forceinline__ float relu_ref(float x) { return x > 0.f ? x : 0.0f; }

// float32 -> the nearest tf32 value (10 explicit mantissa bits, ties away), as a float32.
__device__ __forceinline__ float tf32_rn(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}
// A float32 activation as stored by `o` (rounded to tf32 in the tf32 mode).
__device__ __forceinline__ float f32_out(const OutDev& o, float v) { return o.tf32 ? tf32_rn(v) : v; }

__device__ __forceinline__ float clip_ref(float x, float lo, float hi) {
  float a = x < lo ? lo : x;   // std::max(x, lo)
  return hi < a ? hi : a;      // std::min(a, hi)
}

// cast(float32 -> int8/uint8): checked_trunc then wrap_int (kernels.cpp:320-348).
__device__ __forceinline__ int32_t cast_int_ref(float v, int32_t is_signed) {
  long long t;
  if (!(v > -9.2e18f && v < 9.2e18f)) t = v > 0 ? 0x7fffffffffffffffLL : (-0x7fffffffffffffffLL - 1);
  else t = static_cast<long long>(v);  // truncation toward zero
  int32_t lo8 = static_cast<int32_t>(t & 0xff);
  return is_signed ? static_cast<int32_t>(static_cast<int8_t>(lo8)) : lo8;
}

// quant_calibrate's overflow test on the value entering a quantize site.
// x / rho * 2^(bits-sign) in double == v * c1 in float here (c1 is a power of
// two), so the rounded products agree.
__device__ __forceinline__ void quant_observe(float v, const QDev& q) {
  if (q.ovf) {
    const float t = rintf(__fmul_rn(v, q.c1));
    if (q.is_signed ? fabsf(t) > 128.f : (t < 0.f || t > 256.f)) atomicOr(q.ovf, 1);
  }
}
// The realize chain's integer code: cast(clip(round(v * c1), lo, hi)).
// CAL = false compiles the calibration observer out (hot kernels are
// instantiated both ways; the launchers pick CAL only for a calibration run).
template <bool CAL>
__device__ __forceinline__ int32_t quant_code_t(float v, const QDev& q);

__device__ __forceinline__ int32_t quant_code(float v, const QDev& q) { return quant_code_t<true>(v, q); }

template <bool CAL>
__device__ __forceinline__ int32_t quant_code_t(float v, const QDev& q) {
  if constexpr (CAL) quant_observe(v, q);
  float t = __fmul_rn(v, q.c1);
  t = rintf(t);
  t = clip_ref(t, q.lo, q.hi);
  return cast_int_ref(t, q.is_signed);
}

// log2(cpc): chunk widths are powers of two (kb in {16, 64, 128} bytes over
// 1/2/4-byte elements), so channel -> (plane, lane) is a shift and a mask.
__host__ __device__ __forceinline__ int32_t lay_lg(const Lay& L) {
#ifdef __CUDA_ARCH__
  return 31 - __clz(L.cpc);
#else
  return __builtin_ctz(static_cast<unsigned>(L.cpc));
#endif
}

// Chunk index (16-byte units) of the chunk holding channel c of the padded
// pixel pix (NORMAL-grid linear index) in layout L.
__host__ __device__ __forceinline__ int64_t lay_chunk(const Lay& L, int64_t pix, int32_t c) {
  const int64_t plane = c >> lay_lg(L);
  if (L.kind == LAY_PHASE) {
    int32_t wp = static_cast<int32_t>(pix % L.Wp);
    int64_t t = pix / L.Wp;
    int32_t hp = static_cast<int32_t>(t % L.Hp);
    int64_t n = t / L.Hp;
    int32_t sub = (hp & 1) * 2 + (wp & 1);
    return (plane * 4 + sub) * L.Pp + (n * L.Hq + hp / 2) * L.Wq + wp / 2;
  }
  return plane * L.Pp + pix;
}

__host__ __device__ __forceinline__ int64_t lay_off(const Lay& L, int64_t pix, int32_t c) {
  if (L.cpc == 0) return pix * L.C + c;
  return lay_chunk(L, pix, c) * L.cpc + (c & (L.cpc - 1));
}

// Byte offset of channel c (c % (16 / eb) == 0 for a 16-byte granule).
__host__ __device__ __forceinline__ int64_t lay_byte(const Lay& L, int64_t pix, int32_t c) {
  return lay_chunk(L, pix, c) * L.kb + static_cast<int64_t>(c & (L.cpc - 1)) * (L.kb >> lay_lg(L));
}

// quant_code when the clip bounds lie inside int32 (every realize site:
// [-128, 127] or [0, 255]): the clipped value is integral, so the truncating
// cast is exact and the wrap to 8 bits is a plain narrowing.  NaN: clip keeps
// NaN, cvt.rzi gives 0 == the reference's INT64_MIN & 0xff.
// rint + clip to the 8-bit range + cast in ONE conversion: cvt.rni.sat.{s8,u8}.f32
// (round to nearest even, saturate; NaN -> 0), equal to the reference chain
// clip(rint(y), lo, hi) -> trunc -> wrap whenever [lo, hi] is exactly the
// 8-bit range (every realize site: int8 [-128, 127], uint8 [0, 255]).
__device__ __forceinline__ int32_t cvt_rn_sat_s8(float y) {
  int32_t r;
  asm("cvt.rni.sat.s8.f32 %0, %1;" : "=r"(r) : "f"(y));
  return r;
}
__device__ __forceinline__ int32_t cvt_rn_sat_u8(float y) {
  uint32_t r;
  asm("cvt.rni.sat.u8.f32 %0, %1;" : "=r"(r) : "f"(y));
  return static_cast<int32_t>(r);
}

template <bool CAL>
__device__ __forceinline__ int32_t quant_code_fast_t(float v, const QDev& q) {
  if constexpr (CAL) quant_observe(v, q);
  float t = clip_ref(rintf(__fmul_rn(v, q.c1)), q.lo, q.hi);
  int32_t k = __float2int_rz(t);
  return q.is_signed ? static_cast<int32_t>(static_cast<int8_t>(k)) : (k & 0xff);
}

// quant_code_fast with the saturating conversion for the 8-bit ranges (the
// network-input conversion; measured slower inside the conv epilogues)
template <bool CAL>
__device__ __forceinline__ int32_t quant_code_cvt_t(float v, const QDev& q) {
  if (q.is_signed && q.lo == -128.f && q.hi == 127.f) {  // uniform branch
    if constexpr (CAL) quant_observe(v, q);
    return cvt_rn_sat_s8(__fmul_rn(v, q.c1));
  }
  return quant_code_fast_t<CAL>(v, q);
}

__device__ __forceinline__ int32_t quant_code_fast(float v, const QDev& q) { return quant_code_fast_t<true>(v, q); }

__device__ __forceinline__ float load_fmt(const void* p, int32_t fmt, int64_t i) {
  if (fmt == FMT_F32) return static_cast<const float*>(p)[i];
  return bf16_to_f32(static_cast<const uint16_t*>(p)[i]);
}

// Applies the interpreted epilogue to v (the anchor's float32 result at
// output pixel pix, channel c).  Returns the final float; *code receives the
// int8 code of the last Requant (if any).
__device__ __forceinline__ float apply_epi(const EpiDev& e, float v, int64_t pix, int32_t c, int32_t* code) {
  for (int i = 0; i < e.n_ops; ++i) {
    switch (e.op[i]) {
      case E_MULS: v = __fmul_rn(v, e.s[i]); break;
      case E_MULC: v = __fmul_rn(v, e.vec[i][c]); break;
      case E_BIAS: v = __fadd_rn(v, e.vec[i][c]); break;
      case E_RES: v = __fadd_rn(v, load_fmt(e.res[i], e.res_fmt[i], lay_off(e.res_lay[i], pix, c))); break;
      case E_RELU: v = relu_ref(v); break;
      case E_REQ: {
        int32_t k = quant_code(v, e.q[i]);
        *code = k;
        v = __fmul_rn(static_cast<float>(k), e.q[i].c2);
        break;
      }
      case E_CLIP: v = clip_ref(v, e.s[i], e.s2[i]); break;
      default: break;
    }
  }
  return v;
}

__device__ __forceinline__ void store_out(const OutDev& o, float v, int32_t code, int64_t pix, int32_t c) {
  int64_t i = lay_off(o.plan, pix, c);
  if (o.primary_fmt == FMT_F32) {
    static_cast<float*>(o.primary)[i] = f32_out(o, v);
  } else if (o.primary_fmt == FMT_BF16) {
    static_cast<uint16_t*>(o.primary)[i] = f32_to_bf16(v);
  } else {
    static_cast<int8_t*>(o.primary)[i] = static_cast<int8_t>(code);
  }
  if (o.side) {
    if (o.side_fmt == FMT_I8) static_cast<int8_t*>(o.side)[lay_off(o.slay, pix, c)] = static_cast<int8_t>(quant_code(v, o.side_q));
    else if (o.side_fmt == FMT_F32) static_cast<float*>(o.side)[lay_off(o.slay, pix, c)] = f32_out(o, v);
    else static_cast<uint16_t*>(o.side)[lay_off(o.slay, pix, c)] = f32_to_bf16(v);
  }
}

#endif  // __CUDACC__

// ---- host-visible launch parameter blocks --------------------------------

struct ConvGeom {
  int32_t N, H, W, C;      // input (logical)
  Lay in;                  // input layout (P16, pad kPad)
  int32_t OH, OW, OC;
  int32_t KH, KW, sh, sw, ph, pw;
  int32_t Cs;              // weight channel stride per tap (SIMT layouts)
  int32_t Kp;              // weight row length (I8/BF16: KH*KW*Cs; strict: IC*KH*KW)
};

// Every 4-D activation is stored with a one-pixel zero border.
constexpr int kPad = 1;

__host__ __device__ __forceinline__ int64_t pad_pix(int32_t n, int32_t h, int32_t w, int32_t H, int32_t W) {
  return (static_cast<int64_t>(n) * (H + 2 * kPad) + h + kPad) * (W + 2 * kPad) + w + kPad;
}

}  // namespace mrb200
