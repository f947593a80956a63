// kernels_simt.cu -- CUDA-core kernels: boundary conversions, hoisted weight
// prologues, pooling, the HW sum, dense heads, and the CUDA-core convolution
// variants (int8 dp4a, bf16, and the fp32 reference-order "strict" conv used
// to check the float lowering bit for bit).  The tensor-core convolutions
// live in conv_tc.cu; these are the baseline they are measured against.
#include <cuda_runtime.h>

#include "kernels.cuh"
#include "launch.hpp"

namespace mrb200 {

namespace {

constexpr int kThreads = 256;

inline unsigned blocks_for(int64_t n, int t = kThreads) { return static_cast<unsigned>((n + t - 1) / t); }

// ---- boundary: NCHW float32 -> internal NHWC ---------------------------------

__global__ void k_input_convert(const float* __restrict__ x, int N, int C, int H, int W, void* out,
                                int fmt, int Cs, float pre_mul, QDev q) {
  int64_t total = static_cast<int64_t>(N) * H * W * Cs;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int c = static_cast<int>(i % Cs);
    int64_t p = i / Cs;
    int w = static_cast<int>(p % W);
    int64_t t = p / W;
    int h = static_cast<int>(t % H);
    int n = static_cast<int>(t / H);
    float v = c < C ? x[((static_cast<int64_t>(n) * C + c) * H + h) * W + w] : 0.f;
    if (pre_mul != 0.f) v = __fmul_rn(v, pre_mul);
    if (fmt == FMT_F32) {
      static_cast<float*>(out)[i] = v;
    } else if (fmt == FMT_BF16) {
      static_cast<uint16_t*>(out)[i] = f32_to_bf16(v);
    } else {
      static_cast<int8_t*>(out)[i] = c < C ? static_cast<int8_t>(quant_code(v, q)) : 0;
    }
  }
}

// ---- NHWC float32 -> NCHW float32 (a 4-D @main result) -------------------------

// fmt FMT_I8: x holds realize codes, the value is code * c2 (exact).
__global__ void k_nhwc_to_nchw(const void* __restrict__ x, int fmt, int Cs, float c2, float* __restrict__ y, int N,
                               int C, int H, int W) {
  int64_t total = static_cast<int64_t>(N) * C * H * W;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int w = static_cast<int>(i % W);
    int64_t t = i / W;
    int h = static_cast<int>(t % H);
    t /= H;
    int c = static_cast<int>(t % C);
    int n = static_cast<int>(t / C);
    int64_t src = ((static_cast<int64_t>(n) * H + h) * W + w) * Cs + c;
    if (fmt == FMT_I8) y[i] = __fmul_rn(static_cast<float>(static_cast<const int8_t*>(x)[src]), c2);
    else y[i] = load_fmt(x, fmt, src);
  }
}

// ---- hoisted weight prologue ----------------------------------------------------
// OIHW float32 -> kernel layout.  v = w [* oc_scale[o]] [* scalar]; then
//   I8:   code(v) at [O][KH][KW][Cs]           (K ordered kh, kw, ic; NHWC taps)
//   BF16: bf16(v) at [O][KH][KW][Cs]
//   F32:  v       at [O][IC][KH][KW]           (strict: reference loop order)
__global__ void k_weight_prep(const float* __restrict__ w, int O, int I, int KH, int KW, int Cs,
                              const float* __restrict__ oc_scale, float scalar, int fmt,
                              int quant, QDev q, void* out) {
  int64_t per = static_cast<int64_t>(KH) * KW * Cs;
  int64_t total = fmt == FMT_F32 ? static_cast<int64_t>(O) * I * KH * KW : static_cast<int64_t>(O) * per;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int o, ic, kh, kw;
    if (fmt == FMT_F32) {
      kw = static_cast<int>(i % KW);
      int64_t t = i / KW;
      kh = static_cast<int>(t % KH);
      t /= KH;
      ic = static_cast<int>(t % I);
      o = static_cast<int>(t / I);
    } else {
      ic = static_cast<int>(i % Cs);
      int64_t t = i / Cs;
      kw = static_cast<int>(t % KW);
      t /= KW;
      kh = static_cast<int>(t % KH);
      o = static_cast<int>(t / KH);
    }
    float v = 0.f;
    bool live = ic < I;
    if (live) {
      v = w[((static_cast<int64_t>(o) * I + ic) * KH + kh) * KW + kw];
      if (oc_scale) v = __fmul_rn(v, oc_scale[o]);
      if (scalar != 0.f) v = __fmul_rn(v, scalar);
    }
    if (fmt == FMT_F32) {
      static_cast<float*>(out)[i] = v;
    } else if (fmt == FMT_BF16) {
      static_cast<uint16_t*>(out)[i] = live ? f32_to_bf16(v) : 0;
    } else {
      int32_t code = 0;
      if (live) code = quant ? quant_code(v, q) : static_cast<int32_t>(v);
      static_cast<int8_t*>(out)[i] = static_cast<int8_t>(code);
    }
  }
}

// ---- convolution, int8 codes, dp4a, int32 accumulate -----------------------------
// Implicit GEMM: M = N*OH*OW output pixels, N = OC, K = KH*KW*Cs (tap-major,
// channel-minor, matching NHWC activations and the [O][KH][KW][Cs] weights).
// 64x64 tile, 256 threads x (4 pixels x 4 channels), K staged 32 bytes at a time.
// Integer accumulation is exact; the float32 conversion times acc_scale
// (= c2_x * c2_w, a power of two) equals the reference's fake-quant fp32 conv
// whenever every sequential partial sum stays below 2^24 quanta.
__global__ void __launch_bounds__(256) k_conv_i8_simt(const int8_t* __restrict__ x, const int8_t* __restrict__ w,
                                                      ConvGeom g, float acc_scale, EpiDev epi, OutDev out) {
  __shared__ int32_t As[8][64 + 4];
  __shared__ int32_t Bs[8][64 + 4];
  const int64_t M = static_cast<int64_t>(g.N) * g.OH * g.OW;
  const int64_t m0 = static_cast<int64_t>(blockIdx.x) * 64;
  const int n0 = blockIdx.y * 64;
  const int tid = threadIdx.x;
  const int tm = tid & 15, tn = tid >> 4;
  const int Kw = g.Kp / 4;
  int acc[4][4] = {};
  // per-thread A-load pixel coordinates (2 loads per stage, same pixel column)
  const int lp = tid & 63;
  const int64_t pm = m0 + lp;
  int pn = 0, poh = 0, pow_ = 0;
  bool pvalid = pm < M;
  if (pvalid) {
    pow_ = static_cast<int>(pm % g.OW);
    int64_t t = pm / g.OW;
    poh = static_cast<int>(t % g.OH);
    pn = static_cast<int>(t / g.OH);
  }
  for (int k0 = 0; k0 < Kw; k0 += 8) {
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      int kk = (tid >> 6) + r * 4;
      int word = k0 + kk;
      int32_t av = 0;
      if (pvalid && word < Kw) {
        int k = word * 4;
        int tap = k / g.Cs, ic = k - tap * g.Cs;
        int kh = tap / g.KW, kwi = tap - kh * g.KW;
        int h = poh * g.sh - g.ph + kh, ww = pow_ * g.sw - g.pw + kwi;
        if (h >= 0 && h < g.H && ww >= 0 && ww < g.W)
          av = *reinterpret_cast<const int32_t*>(x + ((static_cast<int64_t>(pn) * g.H + h) * g.W + ww) * g.Cs + ic);
      }
      As[kk][lp] = av;
      int oc = n0 + lp;
      int32_t bv = 0;
      if (oc < g.OC && word < Kw) bv = *reinterpret_cast<const int32_t*>(w + static_cast<int64_t>(oc) * g.Kp + word * 4);
      Bs[kk][lp] = bv;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      int32_t a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][tm * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tn * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = __dp4a(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int64_t m = m0 + tm * 4 + i;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int c = n0 + tn * 4 + j;
      if (c >= g.OC) continue;
      int32_t code = 0;
      float v = apply_epi(epi, __fmul_rn(static_cast<float>(acc[i][j]), acc_scale), m, c, g.OC, &code);
      store_out(out, v, code, m, c);
    }
  }
}

// ---- convolution, bf16 operands, fp32 accumulate (CUDA cores) --------------------
__global__ void __launch_bounds__(256) k_conv_bf16_simt(const uint16_t* __restrict__ x, const uint16_t* __restrict__ w,
                                                        ConvGeom g, EpiDev epi, OutDev out) {
  __shared__ float As[16][64 + 4];
  __shared__ float Bs[16][64 + 4];
  const int64_t M = static_cast<int64_t>(g.N) * g.OH * g.OW;
  const int64_t m0 = static_cast<int64_t>(blockIdx.x) * 64;
  const int n0 = blockIdx.y * 64;
  const int tid = threadIdx.x;
  const int tm = tid & 15, tn = tid >> 4;
  float acc[4][4] = {};
  const int lp = tid & 63;
  const int64_t pm = m0 + lp;
  int pn = 0, poh = 0, pow_ = 0;
  bool pvalid = pm < M;
  if (pvalid) {
    pow_ = static_cast<int>(pm % g.OW);
    int64_t t = pm / g.OW;
    poh = static_cast<int>(t % g.OH);
    pn = static_cast<int>(t / g.OH);
  }
  for (int k0 = 0; k0 < g.Kp; k0 += 16) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      int kk = (tid >> 6) + r * 4;
      int k = k0 + kk;
      float av = 0.f;
      if (pvalid && k < g.Kp) {
        int tap = k / g.Cs, ic = k - tap * g.Cs;
        int kh = tap / g.KW, kwi = tap - kh * g.KW;
        int h = poh * g.sh - g.ph + kh, ww = pow_ * g.sw - g.pw + kwi;
        if (h >= 0 && h < g.H && ww >= 0 && ww < g.W)
          av = bf16_to_f32(x[((static_cast<int64_t>(pn) * g.H + h) * g.W + ww) * g.Cs + ic]);
      }
      As[kk][lp] = av;
      int oc = n0 + lp;
      Bs[kk][lp] = (oc < g.OC && k < g.Kp) ? bf16_to_f32(w[static_cast<int64_t>(oc) * g.Kp + k]) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][tm * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tn * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = __fmaf_rn(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int64_t m = m0 + tm * 4 + i;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int c = n0 + tn * 4 + j;
      if (c >= g.OC) continue;
      int32_t code = 0;
      float v = apply_epi(epi, acc[i][j], m, c, g.OC, &code);
      store_out(out, v, code, m, c);
    }
  }
}

// ---- convolution, fp32, the reference's exact arithmetic ---------------------------
// facc += x*w in the order ic -> kh -> kw with padded taps skipped
// (kernels.cpp:681-701), product and sum each rounded (no FMA).
__global__ void k_conv_f32_strict(const float* __restrict__ x, const float* __restrict__ w, ConvGeom g,
                                  EpiDev epi, OutDev out) {
  const int64_t M = static_cast<int64_t>(g.N) * g.OH * g.OW;
  int64_t total = M * g.OC;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int oc = static_cast<int>(i % g.OC);
    int64_t m = i / g.OC;
    int ow = static_cast<int>(m % g.OW);
    int64_t t = m / g.OW;
    int oh = static_cast<int>(t % g.OH);
    int n = static_cast<int>(t / g.OH);
    float facc = 0.0f;
    for (int ic = 0; ic < g.C; ++ic)
      for (int kh = 0; kh < g.KH; ++kh)
        for (int kw = 0; kw < g.KW; ++kw) {
          int h = oh * g.sh - g.ph + kh, ww = ow * g.sw - g.pw + kw;
          if (h < 0 || h >= g.H || ww < 0 || ww >= g.W) continue;
          float xv = x[((static_cast<int64_t>(n) * g.H + h) * g.W + ww) * g.Cs + ic];
          float wv = w[((static_cast<int64_t>(oc) * g.C + ic) * g.KH + kh) * g.KW + kw];
          facc = __fadd_rn(facc, __fmul_rn(xv, wv));
        }
    int32_t code = 0;
    float v = apply_epi(epi, facc, m, oc, g.OC, &code);
    store_out(out, v, code, m, oc);
  }
}

// ---- depthwise convolution (float; reference order kh -> kw) ---------------------
__global__ void k_dwconv(const void* __restrict__ x, int xfmt, const float* __restrict__ w, ConvGeom g,
                         int strict, EpiDev epi, OutDev out) {
  const int64_t M = static_cast<int64_t>(g.N) * g.OH * g.OW;
  int64_t total = M * g.C;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int c = static_cast<int>(i % g.C);
    int64_t m = i / g.C;
    int ow = static_cast<int>(m % g.OW);
    int64_t t = m / g.OW;
    int oh = static_cast<int>(t % g.OH);
    int n = static_cast<int>(t / g.OH);
    float facc = 0.0f;
    for (int kh = 0; kh < g.KH; ++kh)
      for (int kw = 0; kw < g.KW; ++kw) {
        int h = oh * g.sh - g.ph + kh, ww = ow * g.sw - g.pw + kw;
        if (h < 0 || h >= g.H || ww < 0 || ww >= g.W) continue;
        float xv = load_fmt(x, xfmt, ((static_cast<int64_t>(n) * g.H + h) * g.W + ww) * g.Cs + c);
        float wv = w[(static_cast<int64_t>(c) * g.KH + kh) * g.KW + kw];
        facc = strict ? __fadd_rn(facc, __fmul_rn(xv, wv)) : __fmaf_rn(xv, wv, facc);
      }
    int32_t code = 0;
    float v = apply_epi(epi, facc, m, c, g.C, &code);
    store_out(out, v, code, m, c);
  }
}

// ---- max pooling: max over valid taps, seeded with the first (harness kernel) ----
__global__ void k_maxpool(const void* __restrict__ x, int xfmt, ConvGeom g, OutDev out) {
  const int64_t M = static_cast<int64_t>(g.N) * g.OH * g.OW;
  int64_t total = M * g.C;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int c = static_cast<int>(i % g.C);
    int64_t m = i / g.C;
    int ow = static_cast<int>(m % g.OW);
    int64_t t = m / g.OW;
    int oh = static_cast<int>(t % g.OH);
    int n = static_cast<int>(t / g.OH);
    float acc = 0.f;
    bool seeded = false;
    for (int kh = 0; kh < g.KH; ++kh)
      for (int kw = 0; kw < g.KW; ++kw) {
        int h = oh * g.sh - g.ph + kh, ww = ow * g.sw - g.pw + kw;
        if (h < 0 || h >= g.H || ww < 0 || ww >= g.W) continue;
        float v = load_fmt(x, xfmt, ((static_cast<int64_t>(n) * g.H + h) * g.W + ww) * g.Cs + c);
        if (!seeded) {
          acc = v;
          seeded = true;
        } else {
          acc = acc < v ? v : acc;  // std::max(acc, v)
        }
      }
    store_out(out, acc, 0, m, c);
  }
}

// ---- sum over HW, sequential in row-major (h, w) order, seeded with the first ----
// reduce_impl (kernels.cpp:519-566) visits the input row-major, so for a fixed
// (n, c) the terms arrive in (h, w) order.
__global__ void k_sum_hw(const float* __restrict__ x, int N, int HW, int C, float* __restrict__ y) {
  int64_t total = static_cast<int64_t>(N) * C;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int c = static_cast<int>(i % C);
    int64_t n = i / C;
    const float* p = x + n * HW * C + c;
    float acc = p[0];
    for (int k = 1; k < HW; ++k) acc = __fadd_rn(acc, p[static_cast<int64_t>(k) * C]);
    y[i] = acc;
  }
}

// ---- dense ----------------------------------------------------------------------------
// One block per (row n, 256 outputs).  The data row (float32) gets its prologue
// (pre_mul, realize chain) applied once into shared memory.
//   mode 0: int8 codes, dp4a, int32 acc * acc_scale
//   mode 1: float32 strict, sequential k (kernels.cpp:618-623)
//   mode 2: bf16 weights, fp32 FMA accumulate
__global__ void k_dense(const float* __restrict__ x, int N, int K, int Kp, const void* __restrict__ w, int M,
                        int mode, float pre_mul, int quant, QDev q, float acc_scale, EpiDev epi, OutDev out) {
  extern __shared__ float srow[];
  int n = blockIdx.y;
  int8_t* scode = reinterpret_cast<int8_t*>(srow);
  for (int k = threadIdx.x; k < Kp; k += blockDim.x) {
    float v = k < K ? x[static_cast<int64_t>(n) * K + k] : 0.f;
    if (pre_mul != 0.f && k < K) v = __fmul_rn(v, pre_mul);
    if (mode == 0) scode[k] = k < K ? static_cast<int8_t>(quant ? quant_code(v, q) : static_cast<int32_t>(v)) : 0;
    else srow[k] = v;
  }
  __syncthreads();
  int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= M) return;
  float v;
  if (mode == 0) {
    const int8_t* wr = static_cast<const int8_t*>(w) + static_cast<int64_t>(j) * Kp;
    int acc = 0;
    for (int k = 0; k < Kp; k += 4)
      acc = __dp4a(*reinterpret_cast<const int32_t*>(scode + k), *reinterpret_cast<const int32_t*>(wr + k), acc);
    v = __fmul_rn(static_cast<float>(acc), acc_scale);
  } else if (mode == 1) {
    const float* wr = static_cast<const float*>(w) + static_cast<int64_t>(j) * K;
    float acc = 0.0f;
    for (int k = 0; k < K; ++k) acc = __fadd_rn(acc, __fmul_rn(srow[k], wr[k]));
    v = acc;
  } else {
    const uint16_t* wr = static_cast<const uint16_t*>(w) + static_cast<int64_t>(j) * Kp;
    float acc = 0.0f;
    for (int k = 0; k < K; ++k) acc = __fmaf_rn(srow[k], bf16_to_f32(wr[k]), acc);
    v = acc;
  }
  int32_t code = 0;
  v = apply_epi(epi, v, n, j, M, &code);
  store_out(out, v, code, n, j);
}

unsigned grid_stride_blocks(int64_t total) {
  int64_t b = (total + kThreads - 1) / kThreads;
  if (b > 148 * 32) b = 148 * 32;
  if (b < 1) b = 1;
  return static_cast<unsigned>(b);
}

}  // namespace

void launch_input_convert(const float* x, int N, int C, int H, int W, void* out, int fmt, int Cs,
                          float pre_mul, QDev q, cudaStream_t s) {
  int64_t total = static_cast<int64_t>(N) * H * W * Cs;
  k_input_convert<<<grid_stride_blocks(total), kThreads, 0, s>>>(x, N, C, H, W, out, fmt, Cs, pre_mul, q);
}

void launch_nhwc_to_nchw(const void* x, int fmt, int Cs, float c2, float* y, int N, int C, int H, int W,
                         cudaStream_t s) {
  int64_t total = static_cast<int64_t>(N) * C * H * W;
  k_nhwc_to_nchw<<<grid_stride_blocks(total), kThreads, 0, s>>>(x, fmt, Cs, c2, y, N, C, H, W);
}

void launch_weight_prep(const float* w, int O, int I, int KH, int KW, int Cs, const float* oc_scale,
                        float scalar, int fmt, int quant, QDev q, void* out, cudaStream_t s) {
  int64_t total = fmt == FMT_F32 ? static_cast<int64_t>(O) * I * KH * KW : static_cast<int64_t>(O) * KH * KW * Cs;
  k_weight_prep<<<grid_stride_blocks(total), kThreads, 0, s>>>(w, O, I, KH, KW, Cs, oc_scale, scalar, fmt, quant, q, out);
}

void launch_conv_i8_simt(const int8_t* x, const int8_t* w, const ConvGeom& g, float acc_scale,
                         const EpiDev& epi, const OutDev& out, cudaStream_t s) {
  int64_t M = static_cast<int64_t>(g.N) * g.OH * g.OW;
  dim3 grid(static_cast<unsigned>((M + 63) / 64), static_cast<unsigned>((g.OC + 63) / 64));
  k_conv_i8_simt<<<grid, 256, 0, s>>>(x, w, g, acc_scale, epi, out);
}

void launch_conv_bf16_simt(const uint16_t* x, const uint16_t* w, const ConvGeom& g, const EpiDev& epi,
                           const OutDev& out, cudaStream_t s) {
  int64_t M = static_cast<int64_t>(g.N) * g.OH * g.OW;
  dim3 grid(static_cast<unsigned>((M + 63) / 64), static_cast<unsigned>((g.OC + 63) / 64));
  k_conv_bf16_simt<<<grid, 256, 0, s>>>(x, w, g, epi, out);
}

void launch_conv_f32_strict(const float* x, const float* w, const ConvGeom& g, const EpiDev& epi,
                            const OutDev& out, cudaStream_t s) {
  int64_t total = static_cast<int64_t>(g.N) * g.OH * g.OW * g.OC;
  k_conv_f32_strict<<<grid_stride_blocks(total), kThreads, 0, s>>>(x, w, g, epi, out);
}

void launch_dwconv(const void* x, int xfmt, const float* w, const ConvGeom& g, int strict, const EpiDev& epi,
                   const OutDev& out, cudaStream_t s) {
  int64_t total = static_cast<int64_t>(g.N) * g.OH * g.OW * g.C;
  k_dwconv<<<grid_stride_blocks(total), kThreads, 0, s>>>(x, xfmt, w, g, strict, epi, out);
}

void launch_maxpool(const void* x, int xfmt, const ConvGeom& g, const OutDev& out, cudaStream_t s) {
  int64_t total = static_cast<int64_t>(g.N) * g.OH * g.OW * g.C;
  k_maxpool<<<grid_stride_blocks(total), kThreads, 0, s>>>(x, xfmt, g, out);
}

void launch_sum_hw(const float* x, int N, int HW, int C, float* y, cudaStream_t s) {
  int64_t total = static_cast<int64_t>(N) * C;
  k_sum_hw<<<grid_stride_blocks(total), kThreads, 0, s>>>(x, N, HW, C, y);
}

void launch_dense(const float* x, int N, int K, int Kp, const void* w, int M, int mode, float pre_mul,
                  int quant, QDev q, float acc_scale, const EpiDev& epi, const OutDev& out, cudaStream_t s) {
  dim3 grid(static_cast<unsigned>((M + 255) / 256), static_cast<unsigned>(N));
  size_t smem = mode == 0 ? static_cast<size_t>(Kp) : static_cast<size_t>(Kp) * sizeof(float);
  if (smem > 48 * 1024) cudaFuncSetAttribute(k_dense, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  k_dense<<<grid, 256, smem, s>>>(x, N, K, Kp, w, M, mode, pre_mul, quant, q, acc_scale, epi, out);
}

}  // namespace mrb200
