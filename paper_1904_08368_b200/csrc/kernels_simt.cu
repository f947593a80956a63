// kernels_simt.cu -- CUDA-core kernels: boundary conversions, hoisted weight
// prologues, pooling, the HW sum, dense heads, and the CUDA-core convolution
// variants (int8 dp4a, bf16, and the fp32 reference-order "strict" conv used
// to check the float lowering bit for bit).  The tensor-core convolutions
// live in conv_tc.cu; these are the baseline they are measured against.
// Activations use the padded P16 layout (kernels.cuh).
#include <cuda_runtime.h>

#include <cstdio>
#include <stdexcept>
#include <cstdlib>

#include "kernels.cuh"
#include "launch.hpp"

namespace mrb200 {

namespace {

constexpr int kThreads = 256;

#define GRID_STRIDE(i, total)                                                         \
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < (total); \
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)

struct Pix {
  int32_t n, h, w;  // logical (h, w may be -1 / H for border pixels)
  bool border;
};

__device__ __forceinline__ Pix decode_pix(int64_t pix, int32_t H, int32_t W) {
  const int32_t Hp = H + 2 * kPad, Wp = W + 2 * kPad;
  Pix p;
  int32_t wp = static_cast<int32_t>(pix % Wp);
  int64_t t = pix / Wp;
  int32_t hp = static_cast<int32_t>(t % Hp);
  p.n = static_cast<int32_t>(t / Hp);
  p.h = hp - kPad;
  p.w = wp - kPad;
  p.border = p.h < 0 || p.h >= H || p.w < 0 || p.w >= W;
  return p;
}

// ---- boundary: NCHW float32 -> P16 -----------------------------------------------
// One thread per 16-byte output chunk (cpc channels of one padded pixel);
// consecutive threads take consecutive pixels, so the NCHW reads coalesce per
// channel and the stores are contiguous.  Zeros on the border and in the
// channel padding of the last chunk.
__global__ void k_input_convert(const float* __restrict__ x, int N, int C, int H, int W, void* out, int fmt,
                                Lay L, int s2d_pad, float pre_mul, QDev q) {
  pdl_trigger();
  pdl_wait();
  const int eb = L.kb / L.cpc;
  const int gpc = L.kb / 16;       // 16-byte granules per chunk
  const int cpg = 16 / eb;         // channels per granule
  const int planes = L.kind == LAY_S2D ? (L.C + L.cpc - 1) / L.cpc : (C + L.cpc - 1) / L.cpc;
  const int64_t grid_pix = L.kind == LAY_S2D ? static_cast<int64_t>(N) * L.Hq * L.Wq
                                             : static_cast<int64_t>(N) * (H + 2 * kPad) * (W + 2 * kPad);
  const int64_t total = static_cast<int64_t>(planes) * gpc * grid_pix;
  GRID_STRIDE(i, total) {
    int64_t pix = i % grid_pix;
    int64_t t = i / grid_pix;
    const int gr = static_cast<int>(t % gpc);
    const int32_t pl = static_cast<int32_t>(t / gpc);
    float v[16];
    bool live[16];
    int64_t dst_byte;
    if (L.kind == LAY_S2D) {
      // s2d pixel (n, si, sj), channel sc = (py*2 + px)*C + c  <-  x[n][c][2si+py-pad][2sj+px-pad]
      int32_t sj = static_cast<int32_t>(pix % L.Wq);
      int64_t t2 = pix / L.Wq;
      int32_t si = static_cast<int32_t>(t2 % L.Hq);
      int32_t n = static_cast<int32_t>(t2 / L.Hq);
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        int sc = pl * L.cpc + gr * cpg + k;
        int ph = sc / C, c = sc - ph * C;
        int y = 2 * si + (ph >> 1) - s2d_pad, xx = 2 * sj + (ph & 1) - s2d_pad;
        live[k] = k < cpg && sc < 4 * C && y >= 0 && y < H && xx >= 0 && xx < W;
        v[k] = live[k] ? x[((static_cast<int64_t>(n) * C + c) * H + y) * W + xx] : 0.f;
      }
      dst_byte = (pl * L.Pp + pix) * L.kb + gr * 16;
    } else {
      Pix p = decode_pix(pix, H, W);
      int32_t c0 = pl * L.cpc + gr * cpg;
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        live[k] = k < cpg && !p.border && c0 + k < C;
        v[k] = live[k] ? x[((static_cast<int64_t>(p.n) * C + c0 + k) * H + p.h) * W + p.w] : 0.f;
      }
      dst_byte = lay_chunk(L, pix, pl * L.cpc) * L.kb + gr * 16;
    }
#pragma unroll
    for (int k = 0; k < 16; ++k)
      if (pre_mul != 0.f && live[k]) v[k] = __fmul_rn(v[k], pre_mul);
    char* dst = static_cast<char*>(out) + dst_byte;
    if (fmt == FMT_F32) {
      if (L.kind == LAY_S2D)  // float32 s2d feeds only the tf32 stem: round (the MMA would truncate)
        *reinterpret_cast<float4*>(dst) = make_float4(tf32_rn(v[0]), tf32_rn(v[1]), tf32_rn(v[2]), tf32_rn(v[3]));
      else
        *reinterpret_cast<float4*>(dst) = make_float4(v[0], v[1], v[2], v[3]);
    } else if (fmt == FMT_BF16) {
      uint32_t w4[4];
#pragma unroll
      for (int h = 0; h < 4; ++h)
        w4[h] = pack_bf16x2(v[2 * h], v[2 * h + 1]);
      *reinterpret_cast<uint4*>(dst) = make_uint4(w4[0], w4[1], w4[2], w4[3]);
    } else {
      uint32_t w4[4];
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        uint32_t u = 0;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          int k = 4 * h + b;
          int32_t code = live[k] ? quant_code(v[k], q) : 0;
          u |= (static_cast<uint32_t>(code) & 0xff) << (8 * b);
        }
        w4[h] = u;
      }
      *reinterpret_cast<uint4*>(dst) = make_uint4(w4[0], w4[1], w4[2], w4[3]);
    }
  }
}

// ---- boundary for the stem: NCHW float32 -> LAY_S2D -------------------------------
// Persistent: each block walks s2d rows (n, si) with stride gridDim.x.  An s2d
// row reads input rows y = 2*si + {0, 1} - pad of every channel; the block
// stages those 2*C rows in shared memory with cp.async (16-byte, zero-filled
// outside the image), prefetching the next row into the other buffer while
// it emits the current one as whole s2d pixels (contiguous 16-byte granules).
// Channel sc = (py*2 + px)*C + c of s2d pixel (si, sj) holds
// x[n][c][2si+py-pad][2sj+px-pad], zero outside the image (padded taps).
__device__ __forceinline__ void s2d_prefetch(float* buf, const float* __restrict__ x, int n, int si, int C, int H,
                                             int W, int pad) {
  const int W4 = W >> 2, total4 = 2 * C * W4;
  for (int i = threadIdx.x; i < total4; i += blockDim.x) {
    const int cr = i / W4, x4 = i - cr * W4, y = 2 * si - pad + (cr & 1), c = cr >> 1;
    const bool in = y >= 0 && y < H;
    const float* src = x + ((static_cast<int64_t>(n) * C + c) * H + (in ? y : 0)) * W + 4 * x4;
    const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(buf + 4 * i));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(in ? 16 : 0) : "memory");
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}

__global__ void __launch_bounds__(128) k_input_s2d(const float* __restrict__ x, int N, int C, int H, int W, void* out,
                                                   int fmt, Lay L, int pad, float pre_mul, QDev q) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ __align__(16) float rows[];  // 2 x [C][2][W]
  const int stride = 2 * C * W;
  const int n_rows = N * L.Hq;
  const int eb = L.kb >> lay_lg(L);
  const int gpc = L.kb / 16, cpg = 16 / eb;
  const int planes = (L.C + L.cpc - 1) / L.cpc;
  const bool fast_q = q.lo > -2147483648.f && q.hi < 2147483648.f;  // realize clips: [-128, 127] / [0, 255]
  // per granule channel (pl, gr, k): staged row offset, column shift, row parity, liveness
  __shared__ int2 ktab[64];
  for (int i = threadIdx.x; i < planes * gpc * 16 && i < 64; i += blockDim.x) {
    const int k = i & 15, pg = i >> 4;
    const int sc = (pg / gpc) * L.cpc + (pg % gpc) * cpg + k;
    const int ph = sc / C, c = sc - ph * C, r = (ph >> 1) & 1;
    const bool ok = k < cpg && sc < 4 * C;
    ktab[i] = make_int2((c * 2 + r) * W, (((ph & 1) - pad + 64) << 2) | (r << 1) | (ok ? 1 : 0));
  }
  if (blockIdx.x < n_rows) s2d_prefetch(rows, x, blockIdx.x / L.Hq, blockIdx.x % L.Hq, C, H, W, pad);
  int it = 0;
  for (int row = blockIdx.x; row < n_rows; row += gridDim.x, ++it) {
    const int n = row / L.Hq, si = row - n * L.Hq;
    const int nxt = row + gridDim.x;
    if (nxt < n_rows) {
      s2d_prefetch(rows + ((it + 1) & 1) * stride, x, nxt / L.Hq, nxt % L.Hq, C, H, W, pad);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    const float* cur = rows + (it & 1) * stride;
    const int y0 = 2 * si - pad;
    const bool row_ok0 = y0 >= 0 && y0 < H, row_ok1 = y0 + 1 >= 0 && y0 + 1 < H;
    for (int pl = 0; pl < planes; ++pl)
      for (int gr = 0; gr < gpc; ++gr) {
        for (int sj = threadIdx.x; sj < L.Wq; sj += blockDim.x) {
          const int64_t pix = (static_cast<int64_t>(n) * L.Hq + si) * L.Wq + sj;
          float v[16];
          bool live[16];
#pragma unroll
          for (int k = 0; k < 16; ++k) {
            const int2 t = ktab[(pl * gpc + gr) * 16 + k];
            const int xx = 2 * sj + (t.y >> 2) - 64;
            live[k] = (t.y & 1) && ((t.y & 2) ? row_ok1 : row_ok0) && xx >= 0 && xx < W;
            v[k] = live[k] ? cur[t.x + xx] : 0.f;
            if (live[k] && pre_mul != 0.f) v[k] = __fmul_rn(v[k], pre_mul);
          }
          char* dst = static_cast<char*>(out) + (pl * L.Pp + pix) * L.kb + gr * 16;
          uint32_t w4[4];
          if (fmt == FMT_F32) {  // the tf32 stem's operand: rounded (the MMA would truncate)
            *reinterpret_cast<float4*>(dst) = make_float4(tf32_rn(v[0]), tf32_rn(v[1]), tf32_rn(v[2]), tf32_rn(v[3]));
            continue;
          } else if (fmt == FMT_BF16) {
#pragma unroll
            for (int h = 0; h < 4; ++h)
              w4[h] = pack_bf16x2(v[2 * h], v[2 * h + 1]);
          } else {
#pragma unroll
            for (int h = 0; h < 4; ++h) {
              uint32_t u = 0;
#pragma unroll
              for (int b = 0; b < 4; ++b) {
                const int k = 4 * h + b;
                const int32_t code = !live[k] ? 0 : fast_q ? quant_code_fast(v[k], q) : quant_code(v[k], q);
                u |= (static_cast<uint32_t>(code) & 0xff) << (8 * b);
              }
              w4[h] = u;
            }
          }
          *reinterpret_cast<uint4*>(dst) = make_uint4(w4[0], w4[1], w4[2], w4[3]);
        }
      }
    __syncthreads();  // `cur` is refilled by the prefetch two rows ahead
  }
}

// Compile-time form of k_input_s2d for the common stem (C input channels,
// padding PAD, CPC channels per 16-byte chunk: 16 int8 / 8 bf16): the channel
// -> (row, column shift) map folds to constants and every tap is a branch-free
// select, so the kernel stays memory-bound.  Same values as k_input_s2d.
// PHASED writes LAY_S2DP: the s2d grid is walked from (-2, -2) over the
// 2*Hq x 2*Wq extent of the 4 phase sub-grids (every position written, zeros
// outside the image), so no separate border pass is needed.
#ifndef MRB200_S2D_BPS
#define MRB200_S2D_BPS 16  // S2D row-conversion blocks per SM (A/B: 16 > 12 > 8; 24, 32 = 16)
#endif
#ifndef MRB200_S2D_STAGES
#define MRB200_S2D_STAGES 2  // deeper rings measured slower inside the CUDA graph
#endif
constexpr int kS2dStages = MRB200_S2D_STAGES;  // k_input_s2d_ct row ring depth

template <int C, int PAD, int CPC, bool PHASED, bool CAL>
__global__ void __launch_bounds__(128) k_input_s2d_ct(const float* __restrict__ x, int N, int H, int W, void* out,
                                                      Lay L, float pre_mul, QDev q, FastDiv fd_w4) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ __align__(16) float rows[];  // kS2dStages x [C][2][W]
  constexpr int PLANES = (4 * C + CPC - 1) / CPC;
  constexpr int OFF = PHASED ? 2 : 0;                  // s2d index = grid index - OFF
  const int GR = PHASED ? 2 * L.Hq : L.Hq, GC = PHASED ? 2 * L.Wq : L.Wq;  // walked grid
  const int stride = 2 * C * W;
  const int n_rows = N * GR;
  const int W4 = W >> 2, total4 = 2 * C * W4;
  const bool fast_q = q.lo > -2147483648.f && q.hi < 2147483648.f;
  // the 2*C input row segments of one s2d row: segment cr = (channel, row parity);
  // W4 <= 64: thread = (segment phase t / 64, 16-byte column t % 64), so the
  // segment base is computed once per segment, not per 16-byte chunk
  const bool seg_map = W4 <= 64 && blockDim.x == 128;
  auto prefetch = [&](float* buf, int row) {
    const int n = row / GR, si = row - n * GR - OFF;
    if (seg_map) {
      const int x4 = threadIdx.x & 63;
      if (x4 < W4) {
        const uint32_t dst0 = static_cast<uint32_t>(__cvta_generic_to_shared(buf + 4 * x4));
#pragma unroll
        for (int cr = threadIdx.x >> 6; cr < 2 * C; cr += 2) {
          const int y = 2 * si - PAD + (cr & 1), c = cr >> 1;
          const bool in = y >= 0 && y < H;
          const float* src = x + ((static_cast<int64_t>(n) * C + c) * H + (in ? y : 0)) * W + 4 * x4;
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst0 + static_cast<uint32_t>(cr * W4 * 16)),
                       "l"(src), "r"(in ? 16 : 0)
                       : "memory");
        }
      }
    } else {
      for (int i = threadIdx.x; i < total4; i += blockDim.x) {
        const int cr = static_cast<int>(fdiv(static_cast<uint32_t>(i), fd_w4)), x4 = i - cr * W4;
        const int y = 2 * si - PAD + (cr & 1), c = cr >> 1;
        const bool in = y >= 0 && y < H;
        const float* src = x + ((static_cast<int64_t>(n) * C + c) * H + (in ? y : 0)) * W + 4 * x4;
        const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(buf + 4 * i));
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(in ? 16 : 0) : "memory");
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  // kS2dStages-deep cp.async ring: rows it+1 .. it+kS2dStages-1 are in flight
  // while row it converts (one commit group per row, empty past the end)
#pragma unroll
  for (int k = 0; k < kS2dStages - 1; ++k) {
    const int r = blockIdx.x + k * gridDim.x;
    if (r < n_rows) prefetch(rows + k * stride, r);
    else asm volatile("cp.async.commit_group;" ::: "memory");
  }
  int it = 0;
  for (int row = blockIdx.x; row < n_rows; row += gridDim.x, ++it) {
    const int n = row / GR, gi = row - n * GR, si = gi - OFF;
    const int ahead = row + (kS2dStages - 1) * gridDim.x;
    if (ahead < n_rows) prefetch(rows + ((it + kS2dStages - 1) % kS2dStages) * stride, ahead);
    else asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group %0;" ::"n"(kS2dStages - 1) : "memory");
    __syncthreads();
    const float* cur = rows + (it % kS2dStages) * stride;
    const int y0 = 2 * si - PAD;
    const bool rok[2] = {y0 >= 0 && y0 < H, y0 + 1 >= 0 && y0 + 1 < H};
    for (int gj = threadIdx.x; gj < GC; gj += blockDim.x) {
      const int sj = gj - OFF;
      const int64_t pix = PHASED ? static_cast<int64_t>((gi & 1) * 2 + (gj & 1)) * L.Pp +
                                       (static_cast<int64_t>(n) * L.Hq + (gi >> 1)) * L.Wq + (gj >> 1)
                                 : (static_cast<int64_t>(n) * L.Hq + si) * L.Wq + sj;
      const int xb = 2 * sj - PAD;  // column of phase px = 0
      const bool cok[2] = {xb >= 0 && xb < W, xb + 1 >= 0 && xb + 1 < W};
      const int xc[2] = {min(max(xb, 0), W - 1), min(max(xb + 1, 0), W - 1)};
#pragma unroll
      for (int pl = 0; pl < PLANES; ++pl) {
        float v[CPC];
        bool live[CPC];
#pragma unroll
        for (int k = 0; k < CPC; ++k) {
          const int sc = pl * CPC + k;
          if (sc < 4 * C) {
            const int ph = sc / C, c = sc % C, r = ph >> 1, px = ph & 1;
            live[k] = rok[r] && cok[px];
            const float t = cur[(c * 2 + r) * W + xc[px]];
            v[k] = live[k] ? (pre_mul != 0.f ? __fmul_rn(t, pre_mul) : t) : 0.f;
          } else {
            live[k] = false;
            v[k] = 0.f;
          }
        }
        char* dst = static_cast<char*>(out) + (pl * (PHASED ? 4 : 1) * L.Pp + pix) * 16;
        uint32_t w4[4];
        if constexpr (CPC == 8) {
#pragma unroll
          for (int h = 0; h < 4; ++h)
            w4[h] = pack_bf16x2(v[2 * h], v[2 * h + 1]);
        } else {
#pragma unroll
          for (int h = 0; h < 4; ++h) {
            uint32_t u = 0;
#pragma unroll
            for (int b = 0; b < 4; ++b) {
              const int k = 4 * h + b;
              const int32_t code = !live[k] ? 0 : fast_q ? quant_code_cvt_t<CAL>(v[k], q) : quant_code_t<CAL>(v[k], q);
              u |= (static_cast<uint32_t>(code) & 0xff) << (8 * b);
            }
            w4[h] = u;
          }
        }
        *reinterpret_cast<uint4*>(dst) = make_uint4(w4[0], w4[1], w4[2], w4[3]);
      }
    }
    __syncthreads();
  }
}

// ---- P16 / row-major -> NCHW float32 (@main result) -------------------------------
// fmt FMT_I8: realize codes, the value is code * c2 (exact).
__global__ void k_to_nchw(const void* __restrict__ x, int fmt, Lay L, float c2, float* __restrict__ y, int N, int C,
                          int H, int W, int is4d, int rq, QDev q) {
  pdl_trigger();
  pdl_wait();
  const int64_t total = static_cast<int64_t>(N) * C * H * W;
  GRID_STRIDE(i, total) {
    int w = static_cast<int>(i % W);
    int64_t t = i / W;
    int h = static_cast<int>(t % H);
    t /= H;
    int c = static_cast<int>(t % C);
    int n = static_cast<int>(t / C);
    int64_t pix = is4d ? pad_pix(n, h, w, H, W) : n;
    int64_t src = lay_off(L, pix, c);
    float v;
    if (fmt == FMT_I8) v = __fmul_rn(static_cast<float>(static_cast<const int8_t*>(x)[src]), c2);
    else v = load_fmt(x, fmt, src);
    // rq: a realize chain after a flatten (quantize.cpp:181-201): code then code * c2
    if (rq) v = __fmul_rn(static_cast<float>(quant_code(v, q)), q.c2);
    y[i] = v;
  }
}

// ---- zero the one-pixel border of a P16 buffer (after producers that write
// interior pixels only) -- NORMAL or PHASE layout -----------------------------------
__global__ void k_zero_border(void* buf, Lay L, int N) {
  pdl_trigger();
  pdl_wait();
  const int32_t Hp = L.Hp, Wp = L.Wp, H = Hp - 2 * kPad;
  const int32_t per = 2 * Wp + 2 * H;  // border pixels per image
  const int planes = (L.C + L.cpc - 1) / L.cpc;
  const int64_t total = static_cast<int64_t>(planes) * N * per;
  GRID_STRIDE(i, total) {
    int32_t b = static_cast<int32_t>(i % per);
    int64_t t = i / per;
    int32_t n = static_cast<int32_t>(t % N);
    int32_t plane = static_cast<int32_t>(t / N);
    int32_t hp, wp;
    if (b < Wp) {
      hp = 0;
      wp = b;
    } else if (b < 2 * Wp) {
      hp = Hp - 1;
      wp = b - Wp;
    } else {
      int32_t r = b - 2 * Wp;
      hp = 1 + r / 2;
      wp = (r & 1) ? Wp - 1 : 0;
    }
    int64_t pix = (static_cast<int64_t>(n) * Hp + hp) * Wp + wp;
    int4* dst = reinterpret_cast<int4*>(static_cast<char*>(buf) + lay_chunk(L, pix, plane * L.cpc) * L.kb);
    for (int g = 0; g < L.kb / 16; ++g) dst[g] = make_int4(0, 0, 0, 0);
  }
}

// ---- hoisted weight prologue ----------------------------------------------------
// OIHW float32 -> kernel layout.  v = w [* oc_scale[o]] [* scalar]; then
//   WL_ROWS (I8 / BF16): [O][KH][KW][Cs]               CUDA-core kernels
//   WL_TC   (I8 / BF16 / F32 for tf32): [KH*KW][I/cpc][O][cpc]  tcgen05 B operand (16-byte K chunks)
//   F32 strict:          [O][I][KH][KW]                reference loop order
//   WL_S2D  (I8 / BF16): [TA*TA][4I/cpc][O][cpc]      stride-2 stem over the space-to-depth
//                        input: tap (a, b), s2d channel (py*2+px)*I + c  <-  w[o][c][2a+py][2b+px]
__global__ void k_weight_prep(const float* __restrict__ w, int O, int I, int KH, int KW, int Cs, int wl,
                              const float* __restrict__ oc_scale, float scalar, int fmt, int quant, QDev q,
                              void* out) {
  // WL_TC / WL_S2D: Cs carries the chunk width in bytes (16, 64 or 128)
  // (F32 with WL_TC: the tf32 tcgen05 B operand, 4-byte elements)
  const bool strict = fmt == FMT_F32 && wl == WL_ROWS;
  const int cpc = (wl == WL_ROWS ? 16 : Cs) / (fmt == FMT_I8 ? 1 : fmt == FMT_BF16 ? 2 : 4);
  const int TA = (KH + 1) / 2;
  int planes = wl == WL_S2D ? (4 * I + cpc - 1) / cpc : (I + cpc - 1) / cpc;
  if (wl == WL_S2D && fmt == FMT_F32) planes = (planes + 1) & ~1;  // tf32 stem: even planes (exec make_lay)
  int64_t total;
  if (strict) total = static_cast<int64_t>(O) * I * KH * KW;
  else if (wl == WL_TC) total = static_cast<int64_t>(KH) * KW * planes * O * cpc;
  else if (wl == WL_S2D) total = static_cast<int64_t>(TA) * TA * planes * O * cpc;
  else total = static_cast<int64_t>(O) * KH * KW * Cs;
  GRID_STRIDE(i, total) {
    int o, ic, kh, kw;
    if (strict) {
      kw = static_cast<int>(i % KW);
      int64_t t = i / KW;
      kh = static_cast<int>(t % KH);
      t /= KH;
      ic = static_cast<int>(t % I);
      o = static_cast<int>(t / I);
    } else if (wl == WL_TC) {
      int within = static_cast<int>(i % cpc);
      int64_t t = i / cpc;
      o = static_cast<int>(t % O);
      t /= O;
      int plane = static_cast<int>(t % planes);
      int tap = static_cast<int>(t / planes);
      ic = plane * cpc + within;
      kh = tap / KW;
      kw = tap % KW;
    } else if (wl == WL_S2D) {
      int within = static_cast<int>(i % cpc);
      int64_t t = i / cpc;
      o = static_cast<int>(t % O);
      t /= O;
      int plane = static_cast<int>(t % planes);
      int tap = static_cast<int>(t / planes);
      int sc = plane * cpc + within;
      int ph = sc / I;
      ic = sc - ph * I;
      kh = 2 * (tap / TA) + (ph >> 1);
      kw = 2 * (tap % TA) + (ph & 1);
      if (sc >= 4 * I || kh >= KH || kw >= KW) ic = I;  // structural zero
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
    if (fmt == FMT_F32) {  // WL_TC: the tf32 B operand, rounded to tf32 (the MMA would truncate)
      static_cast<float*>(out)[i] = live ? (strict ? v : tf32_rn(v)) : 0.f;
    } else if (fmt == FMT_BF16) {
      static_cast<uint16_t*>(out)[i] = live ? f32_to_bf16(v) : 0;
    } else {
      int32_t code = 0;
      if (live) code = quant ? quant_code(v, q) : static_cast<int32_t>(v);
      static_cast<int8_t*>(out)[i] = static_cast<int8_t>(code);
    }
  }
}

struct OutPix {
  int64_t m;  // logical output index (n, oh, ow)
  int32_t n, oh, ow;
};

__device__ __forceinline__ OutPix decode_out(int64_t m, const ConvGeom& g) {
  OutPix o;
  o.m = m;
  o.ow = static_cast<int32_t>(m % g.OW);
  int64_t t = m / g.OW;
  o.oh = static_cast<int32_t>(t % g.OH);
  o.n = static_cast<int32_t>(t / g.OH);
  return o;
}

// ---- convolution, int8 codes, dp4a, int32 accumulate -----------------------------
// Implicit GEMM: M = N*OH*OW output pixels, N = OC, K = KH*KW*Cs (tap-major,
// channel-minor).  64x64 tile, 256 threads x (4 pixels x 4 channels), K staged
// 32 bytes at a time.  Integer accumulation is exact; the float32 conversion
// times acc_scale (= c2_x * c2_w, a power of two) equals the reference's
// fake-quant fp32 conv whenever every sequential partial sum stays below 2^24
// quanta (checked statically at weight load).
__global__ void __launch_bounds__(256) k_conv_i8_simt(const int8_t* __restrict__ x, const int8_t* __restrict__ w,
                                                      ConvGeom g, float acc_scale, EpiDev epi, OutDev out) {
  pdl_trigger();
  pdl_wait();
  __shared__ int32_t As[8][64 + 4];
  __shared__ int32_t Bs[8][64 + 4];
  const int64_t M = static_cast<int64_t>(g.N) * g.OH * g.OW;
  const int64_t m0 = static_cast<int64_t>(blockIdx.x) * 64;
  const int n0 = blockIdx.y * 64;
  const int tid = threadIdx.x;
  const int tm = tid & 15, tn = tid >> 4;
  const int Kw = g.Kp / 4;
  int acc[4][4] = {};
  const int lp = tid & 63;
  const bool pvalid = m0 + lp < M;
  const OutPix P = decode_out(pvalid ? m0 + lp : 0, g);
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
        int h = P.oh * g.sh - g.ph + kh, ww = P.ow * g.sw - g.pw + kwi;
        if (ic < g.C && h >= 0 && h < g.H && ww >= 0 && ww < g.W)
          av = *reinterpret_cast<const int32_t*>(x + lay_off(g.in, pad_pix(P.n, h, ww, g.H, g.W), ic));
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
    OutPix o = decode_out(m, g);
    int64_t pix = pad_pix(o.n, o.oh, o.ow, g.OH, g.OW);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int c = n0 + tn * 4 + j;
      if (c >= g.OC) continue;
      int32_t code = 0;
      float v = apply_epi(epi, __fmul_rn(static_cast<float>(acc[i][j]), acc_scale), pix, c, &code);
      store_out(out, v, code, pix, c);
    }
  }
}

// ---- convolution, bf16 operands, fp32 accumulate (CUDA cores) --------------------
__global__ void __launch_bounds__(256) k_conv_bf16_simt(const uint16_t* __restrict__ x, const uint16_t* __restrict__ w,
                                                        ConvGeom g, EpiDev epi, OutDev out) {
  pdl_trigger();
  pdl_wait();
  __shared__ float As[16][64 + 4];
  __shared__ float Bs[16][64 + 4];
  const int64_t M = static_cast<int64_t>(g.N) * g.OH * g.OW;
  const int64_t m0 = static_cast<int64_t>(blockIdx.x) * 64;
  const int n0 = blockIdx.y * 64;
  const int tid = threadIdx.x;
  const int tm = tid & 15, tn = tid >> 4;
  float acc[4][4] = {};
  const int lp = tid & 63;
  const bool pvalid = m0 + lp < M;
  const OutPix P = decode_out(pvalid ? m0 + lp : 0, g);
  for (int k0 = 0; k0 < g.Kp; k0 += 16) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      int kk = (tid >> 6) + r * 4;
      int k = k0 + kk;
      float av = 0.f;
      if (pvalid && k < g.Kp) {
        int tap = k / g.Cs, ic = k - tap * g.Cs;
        int kh = tap / g.KW, kwi = tap - kh * g.KW;
        int h = P.oh * g.sh - g.ph + kh, ww = P.ow * g.sw - g.pw + kwi;
        if (ic < g.C && h >= 0 && h < g.H && ww >= 0 && ww < g.W)
          av = bf16_to_f32(x[lay_off(g.in, pad_pix(P.n, h, ww, g.H, g.W), ic)]);
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
    OutPix o = decode_out(m, g);
    int64_t pix = pad_pix(o.n, o.oh, o.ow, g.OH, g.OW);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int c = n0 + tn * 4 + j;
      if (c >= g.OC) continue;
      int32_t code = 0;
      float v = apply_epi(epi, acc[i][j], pix, c, &code);
      store_out(out, v, code, pix, c);
    }
  }
}

// ---- convolution, fp32, the reference's exact arithmetic ---------------------------
// facc += x*w in the order ic -> kh -> kw with padded taps skipped
// (kernels.cpp:681-701), product and sum each rounded (no FMA).
__global__ void k_conv_f32_strict(const float* __restrict__ x, const float* __restrict__ w, ConvGeom g,
                                  EpiDev epi, OutDev out) {
  pdl_trigger();
  pdl_wait();
  const int64_t total = static_cast<int64_t>(g.N) * g.OH * g.OW * g.OC;
  GRID_STRIDE(i, total) {
    int oc = static_cast<int>(i % g.OC);
    OutPix o = decode_out(i / g.OC, g);
    float facc = 0.0f;
    for (int ic = 0; ic < g.C; ++ic)
      for (int kh = 0; kh < g.KH; ++kh)
        for (int kw = 0; kw < g.KW; ++kw) {
          int h = o.oh * g.sh - g.ph + kh, ww = o.ow * g.sw - g.pw + kw;
          if (h < 0 || h >= g.H || ww < 0 || ww >= g.W) continue;
          float xv = x[lay_off(g.in, pad_pix(o.n, h, ww, g.H, g.W), ic)];
          float wv = w[((static_cast<int64_t>(oc) * g.C + ic) * g.KH + kh) * g.KW + kw];
          facc = __fadd_rn(facc, __fmul_rn(xv, wv));
        }
    int64_t pix = pad_pix(o.n, o.oh, o.ow, g.OH, g.OW);
    int32_t code = 0;
    float v = apply_epi(epi, facc, pix, oc, &code);
    store_out(out, v, code, pix, oc);
  }
}

// ---- depthwise convolution (float; reference order kh -> kw) ---------------------
__global__ void k_dwconv(const void* __restrict__ x, int xfmt, const float* __restrict__ w, ConvGeom g, int strict,
                         EpiDev epi, OutDev out) {
  pdl_trigger();
  pdl_wait();
  const int64_t total = static_cast<int64_t>(g.N) * g.OH * g.OW * g.C;
  GRID_STRIDE(i, total) {
    int c = static_cast<int>(i % g.C);
    OutPix o = decode_out(i / g.C, g);
    float facc = 0.0f;
    for (int kh = 0; kh < g.KH; ++kh)
      for (int kw = 0; kw < g.KW; ++kw) {
        int h = o.oh * g.sh - g.ph + kh, ww = o.ow * g.sw - g.pw + kw;
        if (h < 0 || h >= g.H || ww < 0 || ww >= g.W) continue;
        float xv = load_fmt(x, xfmt, lay_off(g.in, pad_pix(o.n, h, ww, g.H, g.W), c));
        float wv = w[(static_cast<int64_t>(c) * g.KH + kh) * g.KW + kw];
        facc = strict ? __fadd_rn(facc, __fmul_rn(xv, wv)) : __fmaf_rn(xv, wv, facc);
      }
    int64_t pix = pad_pix(o.n, o.oh, o.ow, g.OH, g.OW);
    int32_t code = 0;
    float v = apply_epi(epi, facc, pix, c, &code);
    store_out(out, v, code, pix, c);
  }
}

// ---- depthwise conv, bandwidth path --------------------------------------------------
// One thread per (output pixel, 16-byte input granule: 4 fp32 / 8 bf16 channels),
// output column fastest (coalesced 16-byte tap loads; the 3 input rows of a
// warp are L1-resident).  The taps are fixed byte offsets into the zero-padded
// input (padding <= kPad), so no bounds tests: adding a padded tap's exact
// zero product leaves the sum bit-identical to the reference's skip (the
// accumulator starts at +0, kernels.cpp:684-701 / ref_harness
// k_depthwise_conv2d).  strict: fmul then fadd per tap in kh -> kw order.
__global__ void __launch_bounds__(256) k_dwconv_fast(const void* __restrict__ x, int xfmt, const float* __restrict__ w,
                                                     ConvGeom g, int strict, EpiDev epi, OutDev out, FastDiv fd_ow,
                                                     FastDiv fd_oh, FastDiv fd_n) {
  pdl_trigger();
  pdl_wait();
  const int eb = xfmt == FMT_F32 ? 4 : 2;
  const int cpg = 16 / eb;
  const uint32_t grans = static_cast<uint32_t>(g.C / cpg);
  const uint32_t total = grans * g.N * g.OH * g.OW;
  const int Wp = g.W + 2 * kPad, Hp = g.H + 2 * kPad;
  const int OWp = g.OW + 2 * kPad, OHp = g.OH + 2 * kPad;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const uint32_t t = fdiv(i, fd_ow);
    const int ow = static_cast<int>(i - t * static_cast<uint32_t>(g.OW));
    const uint32_t t2 = fdiv(t, fd_oh);
    const int oh = static_cast<int>(t - t2 * static_cast<uint32_t>(g.OH));
    const uint32_t gran = fdiv(t2, fd_n);
    const int n = static_cast<int>(t2 - gran * static_cast<uint32_t>(g.N));
    const int c0 = static_cast<int>(gran) * cpg;
    const int64_t pin = (static_cast<int64_t>(n) * Hp + oh * g.sh - g.ph + kPad) * Wp + ow * g.sw - g.pw + kPad;
    const char* src = static_cast<const char*>(x) + lay_byte(g.in, pin, c0);
    const int64_t row = static_cast<int64_t>(Wp) * g.in.kb;
    float acc[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) acc[k] = 0.0f;
    for (int kh = 0; kh < g.KH; ++kh)
      for (int kw = 0; kw < g.KW; ++kw) {
        const char* p = src + kh * row + kw * g.in.kb;
        float v[8];
        if (xfmt == FMT_F32) {
          const float4 f = __ldg(reinterpret_cast<const float4*>(p));
          v[0] = f.x; v[1] = f.y; v[2] = f.z; v[3] = f.w;
          v[4] = v[5] = v[6] = v[7] = 0.f;
        } else {
          const uint4 u = __ldg(reinterpret_cast<const uint4*>(p));
          const uint32_t w4[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
          for (int b = 0; b < 4; ++b) {
            v[2 * b] = __uint_as_float(w4[b] << 16);
            v[2 * b + 1] = __uint_as_float(w4[b] & 0xffff0000u);
          }
        }
        const int tap = kh * g.KW + kw;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          if (k >= cpg) break;
          const float wv = __ldg(w + static_cast<int64_t>(c0 + k) * g.KH * g.KW + tap);
          acc[k] = strict ? __fadd_rn(acc[k], __fmul_rn(v[k], wv)) : __fmaf_rn(v[k], wv, acc[k]);
        }
      }
    const int64_t pix = (static_cast<int64_t>(n) * OHp + oh + kPad) * OWp + ow + kPad;
    // epilogue + stores in 4-channel pieces (each lies inside one output chunk)
    for (int s4 = 0; s4 < cpg / 4; ++s4) {
      float r[4];
      int32_t code[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        code[k] = 0;
        r[k] = apply_epi(epi, acc[4 * s4 + k], pix, c0 + 4 * s4 + k, &code[k]);
      }
      char* d4 = static_cast<char*>(out.primary) + lay_byte(out.plan, pix, c0 + 4 * s4);
      if (out.primary_fmt == FMT_F32) {
        *reinterpret_cast<float4*>(d4) = make_float4(f32_out(out, r[0]), f32_out(out, r[1]), f32_out(out, r[2]), f32_out(out, r[3]));
      } else if (out.primary_fmt == FMT_BF16) {
        *reinterpret_cast<uint2*>(d4) =
            make_uint2(pack_bf16x2(r[0], r[1]),
                       pack_bf16x2(r[2], r[3]));
      } else {
        uint32_t u = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) u |= (static_cast<uint32_t>(code[k]) & 0xff) << (8 * k);
        *reinterpret_cast<uint32_t*>(d4) = u;
      }
      if (out.side) {
        char* s4p = static_cast<char*>(out.side) + lay_byte(out.slay, pix, c0 + 4 * s4);
        if (out.side_fmt == FMT_I8) {
          uint32_t u = 0;
#pragma unroll
          for (int k = 0; k < 4; ++k) u |= (static_cast<uint32_t>(quant_code(r[k], out.side_q)) & 0xff) << (8 * k);
          *reinterpret_cast<uint32_t*>(s4p) = u;
        } else {
          *reinterpret_cast<uint2*>(s4p) =
              make_uint2(pack_bf16x2(r[0], r[1]),
                         pack_bf16x2(r[2], r[3]));
        }
      }
    }
  }
}

// Register-blocked depthwise 3x3 (stride 1 or 2, pad <= 1): one thread = 4
// channels x 4 consecutive output columns.  The 36 weights stay in registers,
// the input columns of the 4 outputs are loaded once per input row (6 / 9
// loads per row), the epilogue's ops are interpreted once per thread over the
// 16 values with their per-channel vectors hoisted.  Same per-output order and
// arithmetic as k_dwconv_fast (and the reference).
// PL consecutive lanes take PL consecutive 4-channel pieces of the same
// pixels (PL = 8: 32 channels), so each warp store covers whole 32-byte
// sectors of the consumer's channel rows (no partial-sector write merges).
// Output pixels per thread along the row and the blocks-per-SM floor, per input
// format (A/B builds on MobileNet-v1): bf16 (PL 8) 4 outputs, >= 2 blocks/SM;
// fp32 (PL 1, the int8 modules' float path) 2 outputs, >= 3 blocks/SM.
// PL 16 (bf16 inputs in 128-byte chunks): 16 lanes cover one pixel's 64-channel
// row, so every warp load / store is two whole 128-byte lines.
constexpr int dw_outs(int pl) { return pl >= 8 ? 4 : 2; }
constexpr int dw_minb(int pl) { return pl >= 16 ? 3 : pl >= 8 ? 2 : 3; }
// DSIG: compile-time epilogue for MobileNet's (bf16 out, no side output)
// multiply(gamma') -> bias_add -> clip(0, 6) / relu with the per-channel vectors
// held in registers; DSIG 0 interprets the op list.
// DW_MULC_BIAS_CLIP_REQ: the int8 modules' form, realize codes as the primary output.
enum DwSig : int { DW_ANY = 0, DW_MULC_BIAS_CLIP = 1, DW_MULC_BIAS_RELU = 2, DW_MULC_BIAS_CLIP_REQ = 3 };
template <int SW, int PL, int DSIG = DW_ANY>
__global__ void __launch_bounds__(256, dw_minb(PL)) k_dw3x3_rb(const void* __restrict__ x, int xfmt, const float* __restrict__ w,
                                                  ConvGeom g, int strict, EpiDev epi, OutDev out, FastDiv fd_owq,
                                                  FastDiv fd_oh, FastDiv fd_n) {
  pdl_trigger();
  pdl_wait();
  constexpr int OUTS = dw_outs(PL), NCOL = (OUTS - 1) * SW + 3;
  const int owq = (g.OW + OUTS - 1) / OUTS;
  // blockIdx.y = a group of PL 4-channel pieces; the block's threads walk the
  // output pixels of that channel group, so the 36 weights (and the epilogue's
  // per-channel vectors) are loaded once per thread, not once per item
  const uint32_t lo = threadIdx.x % PL, slot = threadIdx.x / PL, slots = blockDim.x / PL;
  const uint32_t total = static_cast<uint32_t>(g.N) * g.OH * owq;
  const int Wp = g.W + 2 * kPad, Hp = g.H + 2 * kPad;
  const int OWp = g.OW + 2 * kPad, OHp = g.OH + 2 * kPad;
  const bool f32 = xfmt == FMT_F32;
  const int c0 = static_cast<int>(blockIdx.y * PL + lo) * 4;
  // PL 16: the block's 64 channels' weights in shared memory, [tap][channel] (one
  // conflict-free 16-byte load per tap), freeing 36 registers for a third block per SM
  constexpr bool SMW = PL == 16 || PL == 1;
  constexpr int CH = 4 * PL;  // channels of the block's group
  __shared__ __align__(16) float sw[SMW ? 9 * CH : 4];
  float wr[4][9];
  if constexpr (SMW) {
    for (int i = threadIdx.x; i < 9 * CH; i += blockDim.x)
      sw[i] = __ldg(w + static_cast<int64_t>(blockIdx.y * CH + (i % CH)) * 9 + (i / CH));
    __syncthreads();
  } else {
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
      for (int tp = 0; tp < 9; ++tp) wr[k][tp] = __ldg(w + static_cast<int64_t>(c0 + k) * 9 + tp);
  }
  float sv[2][4];  // DSIG != DW_ANY: gamma' and bias of this thread's 4 channels
  if constexpr (DSIG != DW_ANY) {
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const float4 f = *reinterpret_cast<const float4*>(epi.vec[j] + c0);
      sv[j][0] = f.x; sv[j][1] = f.y; sv[j][2] = f.z; sv[j][3] = f.w;
    }
  }
  for (uint32_t ii = blockIdx.x * slots + slot; ii < total; ii += gridDim.x * slots) {
    const uint32_t t = fdiv(ii, fd_owq);
    const int oq = static_cast<int>(ii - t * static_cast<uint32_t>(owq));
    const uint32_t n32 = fdiv(t, fd_oh);
    const int oh = static_cast<int>(t - n32 * static_cast<uint32_t>(g.OH));
    const int n = static_cast<int>(n32);
    const int ow0 = oq * OUTS;
    float acc[OUTS][4];
#pragma unroll
    for (int o = 0; o < OUTS; ++o)
#pragma unroll
      for (int k = 0; k < 4; ++k) acc[o][k] = 0.0f;
    const int ih0 = oh * g.sh - g.ph + kPad;  // padded input row of tap kh = 0
    const int iw0 = ow0 * SW - g.pw + kPad;
    const int64_t rowb = static_cast<int64_t>(Wp) * g.in.kb;
    const char* base = static_cast<const char*>(x) + lay_byte(g.in, (static_cast<int64_t>(n) * Hp + ih0) * Wp, c0);
#pragma unroll
    for (int kh = 0; kh < 3; ++kh) {
      float col[NCOL][4];
#pragma unroll
      for (int j = 0; j < NCOL; ++j) {
        const int cw = min(iw0 + j, Wp - 1);  // columns past the row end only feed discarded outputs
        const char* p = base + kh * rowb + static_cast<int64_t>(cw) * g.in.kb;
        if (f32) {
          const float4 f = __ldg(reinterpret_cast<const float4*>(p));
          col[j][0] = f.x; col[j][1] = f.y; col[j][2] = f.z; col[j][3] = f.w;
        } else {
          const uint2 u = __ldg(reinterpret_cast<const uint2*>(p));
          col[j][0] = __uint_as_float(u.x << 16); col[j][1] = __uint_as_float(u.x & 0xffff0000u);
          col[j][2] = __uint_as_float(u.y << 16); col[j][3] = __uint_as_float(u.y & 0xffff0000u);
        }
      }
#pragma unroll
      for (int kw = 0; kw < 3; ++kw) {
        float w4[4];
        if constexpr (SMW) {
          const float4 f = *reinterpret_cast<const float4*>(sw + (kh * 3 + kw) * CH + lo * 4);
          w4[0] = f.x; w4[1] = f.y; w4[2] = f.z; w4[3] = f.w;
        } else {
#pragma unroll
          for (int k = 0; k < 4; ++k) w4[k] = wr[k][kh * 3 + kw];
        }
        // paired fp32 FMA (sm_100 FFMA2): per lane the same fused op as __fmaf_rn,
        // half the issue slots (the strict path stays scalar: paired multiply + add
        // measured not bit-exact against the reference on MobileNet-v1 int8)
        const float2 w01 = make_float2(w4[0], w4[1]), w23 = make_float2(w4[2], w4[3]);
#pragma unroll
        for (int o = 0; o < OUTS; ++o) {
          const float* xv = col[o * SW + kw];
          float2 a01 = make_float2(acc[o][0], acc[o][1]), a23 = make_float2(acc[o][2], acc[o][3]);
          const float2 x01 = make_float2(xv[0], xv[1]), x23 = make_float2(xv[2], xv[3]);
          if (strict) {  // (scalar: the reference's separate multiply and add, never contracted)
            a01 = make_float2(__fadd_rn(a01.x, __fmul_rn(x01.x, w01.x)), __fadd_rn(a01.y, __fmul_rn(x01.y, w01.y)));
            a23 = make_float2(__fadd_rn(a23.x, __fmul_rn(x23.x, w23.x)), __fadd_rn(a23.y, __fmul_rn(x23.y, w23.y)));
          } else {
            a01 = __ffma2_rn(x01, w01, a01);
            a23 = __ffma2_rn(x23, w23, a23);
          }
          acc[o][0] = a01.x; acc[o][1] = a01.y; acc[o][2] = a23.x; acc[o][3] = a23.y;
        }
      }
    }
    if constexpr (DSIG != DW_ANY) {
#pragma unroll
      for (int o = 0; o < OUTS; ++o) {
        if (ow0 + o >= g.OW) break;
        float r[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          r[k] = __fadd_rn(__fmul_rn(acc[o][k], sv[0][k]), sv[1][k]);
          r[k] = DSIG == DW_MULC_BIAS_RELU ? relu_ref(r[k]) : clip_ref(r[k], epi.s[2], epi.s2[2]);
        }
        const int64_t pix = (static_cast<int64_t>(n) * OHp + oh + kPad) * OWp + ow0 + o + kPad;
        char* dst = static_cast<char*>(out.primary) + lay_byte(out.plan, pix, c0);
        if constexpr (DSIG == DW_MULC_BIAS_CLIP_REQ) {
          uint32_t u = 0;
#pragma unroll
          for (int k = 0; k < 4; ++k) u |= (static_cast<uint32_t>(quant_code(r[k], epi.q[3])) & 0xff) << (8 * k);
          *reinterpret_cast<uint32_t*>(dst) = u;
        } else {
          *reinterpret_cast<uint2*>(dst) = make_uint2(pack_bf16x2(r[0], r[1]), pack_bf16x2(r[2], r[3]));
        }
      }
      continue;
    }
    // epilogue: the op list once per thread over OUTS x 4 values
    int32_t code[OUTS][4];
#pragma unroll
    for (int o = 0; o < OUTS; ++o)
#pragma unroll
      for (int k = 0; k < 4; ++k) code[o][k] = 0;
    for (int op = 0; op < epi.n_ops; ++op) {
      const int kind = epi.op[op];
      if (kind == E_MULC || kind == E_BIAS) {
        const float4 v4 = *reinterpret_cast<const float4*>(epi.vec[op] + c0);
        const float vv[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
        for (int o = 0; o < OUTS; ++o)
#pragma unroll
          for (int k = 0; k < 4; ++k) acc[o][k] = kind == E_MULC ? __fmul_rn(acc[o][k], vv[k]) : __fadd_rn(acc[o][k], vv[k]);
      } else if (kind == E_MULS) {
#pragma unroll
        for (int o = 0; o < OUTS; ++o)
#pragma unroll
          for (int k = 0; k < 4; ++k) acc[o][k] = __fmul_rn(acc[o][k], epi.s[op]);
      } else if (kind == E_RELU) {
#pragma unroll
        for (int o = 0; o < OUTS; ++o)
#pragma unroll
          for (int k = 0; k < 4; ++k) acc[o][k] = relu_ref(acc[o][k]);
      } else if (kind == E_CLIP) {
#pragma unroll
        for (int o = 0; o < OUTS; ++o)
#pragma unroll
          for (int k = 0; k < 4; ++k) acc[o][k] = clip_ref(acc[o][k], epi.s[op], epi.s2[op]);
      } else if (kind == E_REQ) {
        const QDev q = epi.q[op];
#pragma unroll
        for (int o = 0; o < OUTS; ++o)
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            code[o][k] = quant_code(acc[o][k], q);
            acc[o][k] = __fmul_rn(static_cast<float>(code[o][k]), q.c2);
          }
      } else {  // E_RES: per element through the generic path
#pragma unroll
        for (int o = 0; o < OUTS; ++o) {
          const int64_t pix = (static_cast<int64_t>(n) * OHp + oh + kPad) * OWp + min(ow0 + o, g.OW - 1) + kPad;
#pragma unroll
          for (int k = 0; k < 4; ++k)
            acc[o][k] = __fadd_rn(acc[o][k], load_fmt(epi.res[op], epi.res_fmt[op], lay_off(epi.res_lay[op], pix, c0 + k)));
        }
      }
    }
#pragma unroll
    for (int o = 0; o < OUTS; ++o) {
      if (ow0 + o >= g.OW) break;
      const int64_t pix = (static_cast<int64_t>(n) * OHp + oh + kPad) * OWp + ow0 + o + kPad;
      char* d4 = static_cast<char*>(out.primary) + lay_byte(out.plan, pix, c0);
      const float* r = acc[o];
      if (out.primary_fmt == FMT_F32) {
        *reinterpret_cast<float4*>(d4) = make_float4(f32_out(out, r[0]), f32_out(out, r[1]), f32_out(out, r[2]), f32_out(out, r[3]));
      } else if (out.primary_fmt == FMT_BF16) {
        *reinterpret_cast<uint2*>(d4) =
            make_uint2(pack_bf16x2(r[0], r[1]),
                       pack_bf16x2(r[2], r[3]));
      } else {
        uint32_t u = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) u |= (static_cast<uint32_t>(code[o][k]) & 0xff) << (8 * k);
        *reinterpret_cast<uint32_t*>(d4) = u;
      }
      if (out.side) {
        char* s4p = static_cast<char*>(out.side) + lay_byte(out.slay, pix, c0);
        if (out.side_fmt == FMT_I8) {
          uint32_t u = 0;
#pragma unroll
          for (int k = 0; k < 4; ++k) u |= (static_cast<uint32_t>(quant_code(r[k], out.side_q)) & 0xff) << (8 * k);
          *reinterpret_cast<uint32_t*>(s4p) = u;
        } else {
          *reinterpret_cast<uint2*>(s4p) =
              make_uint2(pack_bf16x2(r[0], r[1]),
                         pack_bf16x2(r[2], r[3]));
        }
      }
    }
  }
}

// ---- max pooling: max over valid taps, seeded with the first (harness kernel) ----
// One thread per (output pixel, 16-byte chunk), output column fastest; 32-bit
// index math; the window's taps are 16-byte loads from the padded P16 input
// (padded taps skipped, like the reference's bounds test).  Also emits the
// consumers' second copy (int8 codes or bf16) when requested.
// 2x2 / stride-2 / pad-0 pooling (VGG): every window tap is inside the image, so
// the reference's seeded ordered max is max(max(a, b), max(c, d)) in tap order
// with its std::max comparison; one thread = one output pixel x one 16-byte input
// granule (8 bf16 / 4 fp32 channels), 4 loads issued together, one 16-byte store
// when the output layout keeps the granule's channels contiguous.
template <int EB>
__global__ void __launch_bounds__(256) k_maxpool2x2(const void* __restrict__ x, ConvGeom g, OutDev out,
                                                    FastDiv fd_ow, FastDiv fd_oh, FastDiv fd_n, int vec_store) {
  pdl_trigger();
  pdl_wait();
  constexpr int CPG = 16 / EB;
  const uint32_t grans = static_cast<uint32_t>(g.C / CPG);
  const uint32_t total = grans * g.N * g.OH * g.OW;
  const int Hp = g.H + 2 * kPad, Wp = g.W + 2 * kPad, OHp = g.OH + 2 * kPad, OWp = g.OW + 2 * kPad;
  const int64_t row = static_cast<int64_t>(Wp) * g.in.kb;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const uint32_t t = fdiv(i, fd_ow);
    const int ow = static_cast<int>(i - t * static_cast<uint32_t>(g.OW));
    const uint32_t t2 = fdiv(t, fd_oh);
    const int oh = static_cast<int>(t - t2 * static_cast<uint32_t>(g.OH));
    const uint32_t gran = fdiv(t2, fd_n);
    const int n = static_cast<int>(t2 - gran * static_cast<uint32_t>(g.N));
    const int c0 = static_cast<int>(gran) * CPG;
    const char* src = static_cast<const char*>(x) +
                      lay_byte(g.in, (static_cast<int64_t>(n) * Hp + 2 * oh + kPad) * Wp + 2 * ow + kPad, c0);
    const uint4 q[4] = {__ldg(reinterpret_cast<const uint4*>(src)), __ldg(reinterpret_cast<const uint4*>(src + g.in.kb)),
                        __ldg(reinterpret_cast<const uint4*>(src + row)),
                        __ldg(reinterpret_cast<const uint4*>(src + row + g.in.kb))};
    float acc[8];
#pragma unroll
    for (int tp = 0; tp < 4; ++tp) {
      const uint32_t w4[4] = {q[tp].x, q[tp].y, q[tp].z, q[tp].w};
#pragma unroll
      for (int k = 0; k < CPG; ++k) {
        const float v = EB == 4 ? __uint_as_float(w4[k]) : __uint_as_float(k & 1 ? (w4[k >> 1] & 0xffff0000u) : (w4[k >> 1] << 16));
        acc[k] = tp == 0 ? v : (acc[k] < v ? v : acc[k]);  // std::max(acc, v), taps in (kh, kw) order
      }
    }
    const int64_t pix = (static_cast<int64_t>(n) * OHp + oh + kPad) * OWp + ow + kPad;
    if (vec_store) {
      char* d = static_cast<char*>(out.primary) + lay_byte(out.plan, pix, c0);
      if constexpr (EB == 4)
        *reinterpret_cast<float4*>(d) = make_float4(f32_out(out, acc[0]), f32_out(out, acc[1]), f32_out(out, acc[2]),
                                                    f32_out(out, acc[3]));
      else
        *reinterpret_cast<uint4*>(d) = make_uint4(pack_bf16x2(acc[0], acc[1]), pack_bf16x2(acc[2], acc[3]),
                                                  pack_bf16x2(acc[4], acc[5]), pack_bf16x2(acc[6], acc[7]));
    } else {
#pragma unroll
      for (int k = 0; k < CPG; ++k) store_out(out, acc[k], 0, pix, c0 + k);
    }
  }
}

__global__ void k_maxpool(const void* __restrict__ x, int xfmt, ConvGeom g, OutDev out) {
  pdl_trigger();
  pdl_wait();
  const int eb = xfmt == FMT_F32 ? 4 : 2;
  const int cpg = 16 / eb;  // channels per 16-byte granule
  const uint32_t grans = static_cast<uint32_t>((g.C + cpg - 1) / cpg);
  const uint32_t total = grans * g.N * g.OH * g.OW;
  const int Hp = g.H + 2 * kPad, Wp = g.W + 2 * kPad;
  const int OHp = g.OH + 2 * kPad, OWp = g.OW + 2 * kPad;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    uint32_t t = i / g.OW;
    const int ow = static_cast<int>(i - t * g.OW);
    uint32_t t2 = t / g.OH;
    const int oh = static_cast<int>(t - t2 * g.OH);
    const uint32_t gran = t2 / g.N;
    const int n = static_cast<int>(t2 - gran * g.N);
    const int c0 = static_cast<int>(gran) * cpg;
    const int h0 = oh * g.sh - g.ph, w0 = ow * g.sw - g.pw;  // logical window origin
    // taps are consecutive pixels of one chunk plane: byte stride g.in.kb
    const char* src = static_cast<const char*>(x) +
                      lay_byte(g.in, (static_cast<int64_t>(n) * Hp + h0 + kPad) * Wp + w0 + kPad, c0);
    const int64_t row = static_cast<int64_t>(Wp) * g.in.kb;
    float acc[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) acc[k] = 0.f;
    bool seeded = false;
    for (int kh = 0; kh < g.KH; ++kh) {
      const bool hv = h0 + kh >= 0 && h0 + kh < g.H;
      for (int kw = 0; kw < g.KW; ++kw) {
        if (!hv || w0 + kw < 0 || w0 + kw >= g.W) continue;
        const char* p = src + kh * row + kw * g.in.kb;
        float v[8];
        if (xfmt == FMT_F32) {
          float4 f = __ldg(reinterpret_cast<const float4*>(p));
          v[0] = f.x; v[1] = f.y; v[2] = f.z; v[3] = f.w;
          v[4] = v[5] = v[6] = v[7] = 0.f;
        } else {
          uint4 u = __ldg(reinterpret_cast<const uint4*>(p));
          uint32_t w4[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
          for (int b = 0; b < 4; ++b) {
            v[2 * b] = __uint_as_float(w4[b] << 16);
            v[2 * b + 1] = __uint_as_float(w4[b] & 0xffff0000u);
          }
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) acc[k] = !seeded ? v[k] : (acc[k] < v[k] ? v[k] : acc[k]);  // std::max(acc, v)
        seeded = true;
      }
    }
    const int64_t pix = (static_cast<int64_t>(n) * OHp + oh + kPad) * OWp + ow + kPad;
    char* dst = static_cast<char*>(out.primary) + lay_byte(out.plan, pix, c0);
    // 4-channel pieces at their own addresses: the input granule (cpg = 4 or 8
    // channels) and the output's (4 fp32 / 8 bf16) need not coincide
    (void)dst;
    for (int s4 = 0; s4 < cpg / 4 && c0 + 4 * s4 < g.C; ++s4) {
      char* d4 = static_cast<char*>(out.primary) + lay_byte(out.plan, pix, c0 + 4 * s4);
      const float* a4 = acc + 4 * s4;
      if (out.primary_fmt == FMT_F32) {
        *reinterpret_cast<float4*>(d4) = make_float4(f32_out(out, a4[0]), f32_out(out, a4[1]), f32_out(out, a4[2]), f32_out(out, a4[3]));
      } else {
        *reinterpret_cast<uint2*>(d4) =
            make_uint2(pack_bf16x2(a4[0], a4[1]),
                       pack_bf16x2(a4[2], a4[3]));
      }
    }
    if (out.side) {
      if (out.side_fmt == FMT_I8 && cpg == 4 && c0 + 4 <= g.C) {
        uint32_t u = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) u |= (static_cast<uint32_t>(quant_code_fast(acc[k], out.side_q)) & 0xff) << (8 * k);
        *reinterpret_cast<uint32_t*>(static_cast<char*>(out.side) + lay_byte(out.slay, pix, c0)) = u;
      } else {
        for (int k = 0; k < cpg && c0 + k < g.C; ++k) {
          int64_t so = lay_off(out.slay, pix, c0 + k);
          if (out.side_fmt == FMT_I8) static_cast<int8_t*>(out.side)[so] = static_cast<int8_t>(quant_code(acc[k], out.side_q));
          else static_cast<uint16_t*>(out.side)[so] = f32_to_bf16(acc[k]);
        }
      }
    }
  }
}

// ---- sum over HW, sequential in row-major (h, w) order, seeded with the first ----
// reduce_impl (kernels.cpp:519-566) visits the input row-major, so for a fixed
// (n, c) the terms arrive in (h, w) order.  Input P16 float32, output [N, C].
__global__ void k_sum_hw(const float* __restrict__ x, Lay L, int N, int H, int W, int C, float* __restrict__ y) {
  pdl_trigger();
  pdl_wait();
  const int64_t total = static_cast<int64_t>(N) * C;
  GRID_STRIDE(i, total) {
    int c = static_cast<int>(i % C);
    int n = static_cast<int>(i / C);
    float acc = x[lay_off(L, pad_pix(n, 0, 0, H, W), c)];
    for (int h = 0; h < H; ++h)
      for (int w = (h == 0 ? 1 : 0); w < W; ++w) acc = __fadd_rn(acc, x[lay_off(L, pad_pix(n, h, w, H, W), c)]);
    y[i] = acc;
  }
}

// Same sum, one warp per (image, 4-channel granule) of a NORMAL fp32 layout
// with HW <= 64: the warp stages the granule's HW pixels (16 B each,
// pixel-consecutive in the chunk plane: coalesced) in shared memory, then
// lanes 0..3 each run one channel's sequential seeded sum in (h, w) order.
__global__ void __launch_bounds__(256) k_sum_hw_warp(const float* __restrict__ x, Lay L, int N, int H, int W, int C,
                                                     float* __restrict__ y) {
  pdl_trigger();
  pdl_wait();
  __shared__ float4 st[8][64];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int HW = H * W, grans = C / 4;
  const int64_t items = static_cast<int64_t>(N) * grans;
  for (int64_t it = static_cast<int64_t>(blockIdx.x) * 8 + warp; it < items; it += static_cast<int64_t>(gridDim.x) * 8) {
    const int n = static_cast<int>(it / grans), g = static_cast<int>(it - static_cast<int64_t>(n) * grans);
    for (int p = lane; p < HW; p += 32) {
      const int h = p / W, w = p - h * W;
      st[warp][p] = *reinterpret_cast<const float4*>(x + lay_off(L, pad_pix(n, h, w, H, W), 4 * g));
    }
    __syncwarp();
    if (lane < 4) {
      const float* col = reinterpret_cast<const float*>(st[warp]) + lane;
      float acc = col[0];
      for (int p = 1; p < HW; ++p) acc = __fadd_rn(acc, col[4 * p]);
      y[static_cast<int64_t>(n) * C + 4 * g + lane] = acc;
    }
    __syncwarp();
  }
}

// Same sum, one warp per (image, 32-channel group = 8 granules): the warp stages
// the 8 granule planes (HW <= 64 pixels of 16 B each) in shared memory with all
// lanes loading (12-16 independent 16-byte loads per lane for 7x7), then every
// lane runs one channel's sequential seeded sum in (h, w) order.  Granule plane
// stride S = 1 (mod 8) float4 puts the 8 granules of one pixel on distinct banks.
constexpr int kSumWarps = 4;
template <bool CAL>
__global__ void __launch_bounds__(kSumWarps * 32) k_sum_hw_warp32(const float* __restrict__ x, Lay L, int N, int H,
                                                                  int W, int C, float* __restrict__ y, SumOperand op) {
  pdl_trigger();
  pdl_wait();
  __shared__ float4 st[kSumWarps][8 * 65];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int HW = H * W, S = ((HW + 7) / 8) * 8 + 1, groups = C / 32;
  const int64_t items = static_cast<int64_t>(N) * groups;
  for (int64_t it = static_cast<int64_t>(blockIdx.x) * kSumWarps + warp; it < items;
       it += static_cast<int64_t>(gridDim.x) * kSumWarps) {
    const int n = static_cast<int>(it / groups), c0 = 32 * static_cast<int>(it - static_cast<int64_t>(n) * groups);
    // all of the lane's loads are issued before the first shared-memory store
    // (a rolled load->store loop would serialise ~13 L2/HBM round trips)
    float4 v[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int idx = lane + 32 * u;
      if (idx < 8 * HW) {
        const int g = idx / HW, p = idx - g * HW, h = p / W, w = p - h * W;
        v[u] = __ldg(reinterpret_cast<const float4*>(x + lay_off(L, pad_pix(n, h, w, H, W), c0 + 4 * g)));
      }
    }
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int idx = lane + 32 * u;
      if (idx < 8 * HW) {
        const int g = idx / HW;
        st[warp][g * S + idx - g * HW] = v[u];
      }
    }
    __syncwarp();
    const float* col = reinterpret_cast<const float*>(st[warp] + (lane >> 2) * S) + (lane & 3);
    // all the lane's shared-memory reads first, then the seeded sequential sum
    // (a load in the dependency chain of every add would cost ~30 cycles each)
    float vals[64];
#pragma unroll
    for (int p = 0; p < 64; ++p) vals[p] = p < HW ? col[4 * p] : 0.f;
    float acc = vals[0];
#pragma unroll
    for (int p = 1; p < 64; ++p)
      if (p < HW) acc = __fadd_rn(acc, vals[p]);
    const int c = c0 + lane;
    if (y) y[static_cast<int64_t>(n) * C + c] = acc;
    if (op.ptr) {  // the consumer dense's operand: its data prologue applied once here
      float t = acc;
      if (op.pre_mul != 0.f) t = __fmul_rn(t, op.pre_mul);
      const int64_t o = static_cast<int64_t>(n) * op.Kp + c;
      if (op.eb == 1)
        static_cast<int8_t*>(op.ptr)[o] = static_cast<int8_t>(op.quant ? quant_code_t<CAL>(t, op.q) : static_cast<int32_t>(t));
      else if (op.eb == 2)
        static_cast<uint16_t*>(op.ptr)[o] = f32_to_bf16(t);
      else
        static_cast<float*>(op.ptr)[o] = tf32_rn(t);
    }
    __syncwarp();
  }
}

// ---- dense ----------------------------------------------------------------------------
// Block = kDenseRows data rows x 256 outputs.  The rows get their prologue
// (pre_mul, realize chain) once into shared memory; each thread owns one
// output column j and walks K once, reading the transposed weights
// ([K/4][M] int8 words or [K][M] bf16, coalesced across j) and updating
// kDenseRows accumulators per weight load.
//   mode 0: int8 codes, dp4a, int32 acc * acc_scale (exact)
//   mode 1: float32 strict, sequential k (kernels.cpp:618-623), weights [M][K]
//   mode 2: bf16 weights, fp32 FMA accumulate
constexpr int kDenseRows = 8;
constexpr int kDenseK = 2048;  // K chunk staged in shared memory (a multiple of 4)

template <bool CAL>
__global__ void __launch_bounds__(256) k_dense(const float* __restrict__ x, int N, int K, int Kp,
                                               const void* __restrict__ w, int M, int mode, float pre_mul, int quant,
                                               QDev q, float acc_scale, EpiDev epi, OutDev out) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ float srow[];  // [kDenseRows][ks] floats (mode 1/2) or bytes (mode 0)
  const int ks = min(Kp, kDenseK);  // row stride of the staged chunk (== the launcher's allocation)
  const int n0 = blockIdx.y * kDenseRows;
  int8_t* scode = reinterpret_cast<int8_t*>(srow);
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const bool jv = j < M;
  int acc[kDenseRows];
  float res[kDenseRows];
#pragma unroll
  for (int r = 0; r < kDenseRows; ++r) {
    acc[r] = 0;
    res[r] = 0.0f;
  }
  // K in chunks of kDenseK (the row prologue is staged per chunk); the
  // accumulation order over k is the same sequential order as one pass
  for (int k0 = 0; k0 < Kp; k0 += kDenseK) {
    const int kc = min(kDenseK, Kp - k0);
    __syncthreads();  // the previous chunk is consumed
    for (int idx = threadIdx.x; idx < kDenseRows * kc; idx += blockDim.x) {
      const int r = idx / kc, kk = idx - r * kc, k = k0 + kk;
      const int n = n0 + r;
      const bool live = n < N && k < K;
      float v = live ? x[static_cast<int64_t>(n) * K + k] : 0.f;
      if (pre_mul != 0.f && live) v = __fmul_rn(v, pre_mul);
      if (mode == 0) scode[r * ks + kk] = live ? static_cast<int8_t>(quant ? quant_code_t<CAL>(v, q) : static_cast<int32_t>(v)) : 0;
      else srow[r * ks + kk] = v;
    }
    __syncthreads();
    if (!jv) continue;
    if (mode == 0) {
      const int32_t* wt = static_cast<const int32_t*>(w) + static_cast<int64_t>(k0 / 4) * M + j;
      const int KW = kc / 4;  // Kp and kDenseK are multiples of 4
      int kw = 0;
      for (; kw + 8 <= KW; kw += 8) {  // 8 weight words in flight per thread
        int32_t wv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) wv[u] = __ldg(wt + static_cast<int64_t>(kw + u) * M);
#pragma unroll
        for (int u = 0; u < 8; ++u)
#pragma unroll
          for (int r = 0; r < kDenseRows; ++r)
            acc[r] = __dp4a(*reinterpret_cast<const int32_t*>(scode + r * ks + (kw + u) * 4), wv[u], acc[r]);
      }
      for (; kw < KW; ++kw) {
        const int32_t wv = __ldg(wt + static_cast<int64_t>(kw) * M);
#pragma unroll
        for (int r = 0; r < kDenseRows; ++r)
          acc[r] = __dp4a(*reinterpret_cast<const int32_t*>(scode + r * ks + kw * 4), wv, acc[r]);
      }
    } else if (mode == 1) {
      const float* wr = static_cast<const float*>(w) + static_cast<int64_t>(j) * K + k0;
      const int kend = min(kc, K - k0);
      for (int kk = 0; kk < kend; ++kk) {
        const float wv = wr[kk];
#pragma unroll
        for (int r = 0; r < kDenseRows; ++r) res[r] = __fadd_rn(res[r], __fmul_rn(srow[r * ks + kk], wv));
      }
    } else {
      // [K/8][M][8] bf16: one 16-byte load = 8 consecutive k of column j (padding rows are zero)
      const uint4* wt = reinterpret_cast<const uint4*>(w) + static_cast<int64_t>(k0 / 8) * M + j;
      for (int kk = 0; kk < kc; kk += 8) {
        const uint4 u = __ldg(wt + static_cast<int64_t>(kk / 8) * M);
        const uint32_t w4[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          const float w0 = __uint_as_float(w4[h] << 16), w1 = __uint_as_float(w4[h] & 0xffff0000u);
#pragma unroll
          for (int r = 0; r < kDenseRows; ++r) {
            res[r] = __fmaf_rn(srow[r * ks + kk + 2 * h], w0, res[r]);
            res[r] = __fmaf_rn(srow[r * ks + kk + 2 * h + 1], w1, res[r]);
          }
        }
      }
    }
  }
  if (!jv) return;
  if (mode == 0) {
#pragma unroll
    for (int r = 0; r < kDenseRows; ++r) res[r] = __fmul_rn(static_cast<float>(acc[r]), acc_scale);
  }
#pragma unroll
  for (int r = 0; r < kDenseRows; ++r) {
    const int n = n0 + r;
    if (n >= N) break;
    int32_t code = 0;
    float v = apply_epi(epi, res[r], n, j, &code);
    store_out(out, v, code, n, j);
  }
}

// ---- dense, K split across warps (int8 codes / bf16 weights) ----------------------
// The int8 contraction is an exact int32 sum and the bf16 mode is held to a
// tolerance, so K can be split: block = 32 output columns (one per lane) x R
// rows; warp w owns K slice w of each staged chunk, the 8 partial sums are
// reduced through shared memory in fixed warp order.  Each thread issues its
// chunk's weight loads before the row staging so the L2 round trip overlaps
// it.  Grid: ceil(M/32) x ceil(N/R) (the head: 32 x 16 = 512 blocks).
constexpr int kDkWarps = 8;

template <int MODE, int R, int kDkChunk, bool CAL>  // kDkChunk: K elements per staged chunk (multiple of 8 * kDkWarps)
__global__ void __launch_bounds__(256) k_dense_ks(const float* __restrict__ x, int N, int K, int Kp,
                                                  const void* __restrict__ w, int M, float pre_mul, int quant, QDev q,
                                                  float acc_scale, EpiDev epi, OutDev out) {
  pdl_trigger();
  pdl_wait();
  constexpr int kSlice = kDkChunk / kDkWarps;            // K per warp per chunk
  constexpr int kLoads = MODE == 0 ? kSlice / 4 : kSlice / 8;  // weight words (int32 / uint4) per thread
  __shared__ __align__(16) uint8_t stage[MODE == 0 ? R * kDkChunk : R * kDkChunk * 4];
  // the cross-warp partial sums: their own array when both fit the 48 KB of static
  // shared memory, else the staging buffer once the K loop is done
  constexpr int kStageBytes = MODE == 0 ? R * kDkChunk : R * kDkChunk * 4;
  constexpr bool kAliasRed = kStageBytes + static_cast<int>(sizeof(float)) * kDkWarps * R * 32 > 48 * 1024;
  static_assert(!kAliasRed || static_cast<int>(sizeof(float)) * kDkWarps * R * 32 <= kStageBytes, "red fits stage");
  __shared__ float red_own[kAliasRed ? 1 : kDkWarps][kAliasRed ? 1 : R][32];
  auto red = kAliasRed ? reinterpret_cast<float (*)[R][32]>(stage) : reinterpret_cast<float (*)[R][32]>(&red_own[0][0][0]);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int j = blockIdx.x * 32 + lane;
  const bool jv = j < M;
  const int n0 = blockIdx.y * R;
  int acc[R];
  float res[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    acc[r] = 0;
    res[r] = 0.f;
  }
  for (int k0 = 0; k0 < Kp; k0 += kDkChunk) {
    const int kc = min(kDkChunk, Kp - k0);
    const int ks0 = warp * kSlice;  // this warp's slice within the chunk
    // 1. weight loads for the slice (zero past the chunk / the padded K)
    int32_t wv[MODE == 0 ? kLoads : 1];
    uint4 wb[MODE == 2 ? kLoads : 1];
    if (MODE == 0) {
      const int32_t* wt = static_cast<const int32_t*>(w) + static_cast<int64_t>((k0 + ks0) / 4) * M + j;
#pragma unroll
      for (int u = 0; u < kLoads; ++u) wv[u] = (jv && ks0 + u * 4 < kc) ? __ldg(wt + static_cast<int64_t>(u) * M) : 0;
    } else {
      const uint4* wt = reinterpret_cast<const uint4*>(w) + static_cast<int64_t>((k0 + ks0) / 8) * M + j;
#pragma unroll
      for (int u = 0; u < kLoads; ++u)
        wb[u] = (jv && ks0 + u * 8 < kc) ? __ldg(wt + static_cast<int64_t>(u) * M) : make_uint4(0, 0, 0, 0);
    }
    // 2. stage the R rows' chunk (prologue: pre_mul, realize chain); 8 row
    // loads in flight per thread (a dependent load per element would serialise
    // the DRAM round trips)
    __syncthreads();  // the previous chunk is consumed
    constexpr int kU = 8;
    if (MODE == 0 && (K & 3) == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0) {
      // int8 codes, K % 4 == 0: one 16-byte row load -> 4 codes -> one 4-byte
      // shared store (the per-element index math dominated the head's issue slots)
      const int kc4 = kc >> 2;
      for (int base = threadIdx.x; base < R * kc4; base += kU * blockDim.x) {
        float4 v[kU];
        bool live[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const int idx = base + u * blockDim.x;
          const int r = idx / kc4, k = k0 + 4 * (idx - r * kc4);
          live[u] = idx < R * kc4 && n0 + r < N && k < K;
          v[u] = live[u] ? __ldg(reinterpret_cast<const float4*>(x + static_cast<int64_t>(n0 + r) * K + k))
                         : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const int idx = base + u * blockDim.x;
          if (idx >= R * kc4) break;
          const int r = idx / kc4, k4 = idx - r * kc4;
          uint32_t packed = 0;
          if (live[u]) {
            const float e[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
            for (int b = 0; b < 4; ++b) {
              float t = e[b];
              if (pre_mul != 0.f) t = __fmul_rn(t, pre_mul);
              const uint8_t code =
                  static_cast<uint8_t>(static_cast<int8_t>(quant ? quant_code_t<CAL>(t, q) : static_cast<int32_t>(t)));
              packed |= static_cast<uint32_t>(code) << (8 * b);
            }
          }
          *reinterpret_cast<uint32_t*>(stage + r * kDkChunk + 4 * k4) = packed;
        }
      }
    } else
    for (int base = threadIdx.x; base < R * kc; base += kU * blockDim.x) {
      float v[kU];
      bool live[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int idx = base + u * blockDim.x;
        const int r = idx / kc, k = k0 + idx - r * kc;
        live[u] = idx < R * kc && n0 + r < N && k < K;
        v[u] = live[u] ? x[static_cast<int64_t>(n0 + r) * K + k] : 0.f;
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int idx = base + u * blockDim.x;
        if (idx >= R * kc) break;
        const int r = idx / kc, kk = idx - r * kc;
        float t = v[u];
        if (pre_mul != 0.f && live[u]) t = __fmul_rn(t, pre_mul);
        if (MODE == 0)
          stage[r * kDkChunk + kk] = static_cast<uint8_t>(
              live[u] ? static_cast<int8_t>(quant ? quant_code_t<CAL>(t, q) : static_cast<int32_t>(t)) : 0);
        else
          reinterpret_cast<float*>(stage)[r * kDkChunk + kk] = t;
      }
    }
    __syncthreads();
    // 3. contract the slice
    if (MODE == 0) {
#pragma unroll
      for (int u = 0; u < kLoads; ++u) {
        if (ks0 + u * 4 >= kc) break;
#pragma unroll
        for (int r = 0; r < R; ++r)
          acc[r] = __dp4a(*reinterpret_cast<const int32_t*>(stage + r * kDkChunk + ks0 + u * 4), wv[u], acc[r]);
      }
    } else {
      const float* sf = reinterpret_cast<const float*>(stage);
#pragma unroll
      for (int u = 0; u < kLoads; ++u) {
        if (ks0 + u * 8 >= kc) break;
        const uint32_t w4[4] = {wb[u].x, wb[u].y, wb[u].z, wb[u].w};
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const float4 a = *reinterpret_cast<const float4*>(sf + r * kDkChunk + ks0 + u * 8);
          const float4 b = *reinterpret_cast<const float4*>(sf + r * kDkChunk + ks0 + u * 8 + 4);
          const float xs[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
          for (int h = 0; h < 4; ++h) {
            res[r] = __fmaf_rn(xs[2 * h], __uint_as_float(w4[h] << 16), res[r]);
            res[r] = __fmaf_rn(xs[2 * h + 1], __uint_as_float(w4[h] & 0xffff0000u), res[r]);
          }
        }
      }
    }
  }
  // 4. cross-warp reduction (fixed order) + epilogue
  if constexpr (kAliasRed) __syncthreads();  // every warp is done reading the staged rows
#pragma unroll
  for (int r = 0; r < R; ++r) red[warp][r][lane] = MODE == 0 ? __int_as_float(acc[r]) : res[r];
  __syncthreads();
  for (int idx = threadIdx.x; idx < R * 32; idx += blockDim.x) {
    const int r = idx >> 5, l = idx & 31;
    const int n = n0 + r, jj = blockIdx.x * 32 + l;
    if (n >= N || jj >= M) continue;
    float v;
    if (MODE == 0) {
      int s = 0;
#pragma unroll
      for (int ww = 0; ww < kDkWarps; ++ww) s += __float_as_int(red[ww][r][l]);
      v = __fmul_rn(static_cast<float>(s), acc_scale);
    } else {
      v = red[0][r][l];
#pragma unroll
      for (int ww = 1; ww < kDkWarps; ++ww) v += red[ww][r][l];
    }
    int32_t code = 0;
    v = apply_epi(epi, v, n, jj, &code);
    store_out(out, v, code, n, jj);
  }
}

// [M][K] float32 (after the prologue) -> transposed kernel layouts for k_dense.
__global__ void k_dense_weight_t(const float* __restrict__ w, int M, int K, int Kp, const float* __restrict__ oc_scale,
                                 float scalar, int fmt, int quant, QDev q, void* out) {
  const int64_t total = static_cast<int64_t>(M) * Kp;
  GRID_STRIDE(i, total) {
    int j = static_cast<int>(i % M);
    int k = static_cast<int>(i / M);  // out index: [k/8][j][k%8] (bf16) / [k/4][j][k%4] (int8)
    float v = 0.f;
    bool live = k < K;
    if (live) {
      v = w[static_cast<int64_t>(j) * K + k];
      if (oc_scale) v = __fmul_rn(v, oc_scale[j]);
      if (scalar != 0.f) v = __fmul_rn(v, scalar);
    }
    if (fmt == FMT_I8) {
      int32_t code = live ? (quant ? quant_code(v, q) : static_cast<int32_t>(v)) : 0;
      static_cast<int8_t*>(out)[(static_cast<int64_t>(k / 4) * M + j) * 4 + (k & 3)] = static_cast<int8_t>(code);
    } else {
      static_cast<uint16_t*>(out)[(static_cast<int64_t>(k / 8) * M + j) * 8 + (k & 7)] = live ? f32_to_bf16(v) : 0;
    }
  }
}

}  // namespace

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("MRB200_NO_PDL");
    return !(e && std::atoi(e));
  }();
  return on;
}

namespace {

unsigned grid_stride_blocks(int64_t total) {
  int64_t b = (total + kThreads - 1) / kThreads;
  if (b > 148 * 32) b = 148 * 32;
  if (b < 1) b = 1;
  return static_cast<unsigned>(b);
}

}  // namespace

void launch_input_convert(const float* x, int N, int C, int H, int W, void* out, int fmt, const Lay& L,
                          int s2d_pad, float pre_mul, QDev q, cudaStream_t s) {
  if (L.kind == LAY_S2DP) {
    // only the int8 3-channel pad-3 stem is planned onto LAY_S2DP (exec.cpp decide_tc)
    static int sms2 = [] {
      int d = 0, v = 0;
      cudaGetDevice(&d);
      cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, d);
      return v > 0 ? v : 148;
    }();
    if (!(C == 3 && s2d_pad == 3 && (fmt == FMT_I8 || fmt == FMT_BF16) && W % 4 == 0 &&
          reinterpret_cast<uintptr_t>(x) % 16 == 0)) {
      std::fprintf(stderr, "mrb200: LAY_S2DP input conversion needs a 3-channel pad-3 stem (int8 / bf16)\n");
      std::abort();
    }
    const FastDiv fd = make_fastdiv(static_cast<uint32_t>(W / 4));
    const int rows = N * 2 * L.Hq;
    if (fmt == FMT_BF16) {
      pdl_launch(k_input_s2d_ct<3, 3, 8, true, false>, std::min(rows, sms2 * MRB200_S2D_BPS), 128, kS2dStages * 2 * C * W * sizeof(float), s, x,
                 N, H, W, out, L, pre_mul, q, fd);
      return;
    }
    pdl_launch(q.ovf ? k_input_s2d_ct<3, 3, 16, true, true> : k_input_s2d_ct<3, 3, 16, true, false>, std::min(rows, sms2 * MRB200_S2D_BPS), 128, kS2dStages * 2 * C * W * sizeof(float), s,
               x, N, H, W, out, L, pre_mul, q, fd);
    return;
  }
  const int s2d_planes = (L.C + L.cpc - 1) / L.cpc;
  if (L.kind == LAY_S2D && 2 * 2 * C * W * 4 <= 40 * 1024 && W % 4 == 0 && s2d_planes * (L.kb / 16) <= 4 &&
      reinterpret_cast<uintptr_t>(x) % 16 == 0) {
    static int sms = [] {
      int d = 0, v = 0;
      cudaGetDevice(&d);
      cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, d);
      return v > 0 ? v : 148;
    }();
    const int rows = N * L.Hq;
    const size_t smem = kS2dStages * 2 * C * W * sizeof(float);
    if (C == 3 && s2d_pad == 3 && L.kb == 16 && (fmt == FMT_I8 || fmt == FMT_BF16) && smem <= 48 * 1024) {
      const FastDiv fd = make_fastdiv(static_cast<uint32_t>(W / 4));
      if (fmt == FMT_I8)
        pdl_launch(q.ovf ? k_input_s2d_ct<3, 3, 16, false, true> : k_input_s2d_ct<3, 3, 16, false, false>, std::min(rows, sms * 8), 128, smem, s, x, N, H, W, out, L, pre_mul, q, fd);
      else
        pdl_launch(k_input_s2d_ct<3, 3, 8, false, false>, std::min(rows, sms * 8), 128, smem, s, x, N, H, W, out, L, pre_mul, q, fd);
      return;
    }
    // 3x3/s2/pad-1 stems over 3 channels (MobileNet-v1): the same kernel with PAD 1
    if (C == 3 && s2d_pad == 1 && L.kb == 16 && (fmt == FMT_I8 || fmt == FMT_BF16) && smem <= 48 * 1024) {
      const FastDiv fd = make_fastdiv(static_cast<uint32_t>(W / 4));
      if (fmt == FMT_I8)
        pdl_launch(q.ovf ? k_input_s2d_ct<3, 1, 16, false, true> : k_input_s2d_ct<3, 1, 16, false, false>,
                   std::min(rows, sms * 8), 128, smem, s, x, N, H, W, out, L, pre_mul, q, fd);
      else
        pdl_launch(k_input_s2d_ct<3, 1, 8, false, false>, std::min(rows, sms * 8), 128, smem, s, x, N, H, W, out, L,
                   pre_mul, q, fd);
      return;
    }
    pdl_launch(k_input_s2d, std::min(rows, sms * 8), 128, 2 * 2 * C * W * sizeof(float), s, x, N, C, H, W, out, fmt, L,
                                                                                  s2d_pad, pre_mul, q);
    return;
  }
  int planes = L.kind == LAY_S2D ? (L.C + L.cpc - 1) / L.cpc : (C + L.cpc - 1) / L.cpc;
  int64_t grid_pix = L.kind == LAY_S2D ? static_cast<int64_t>(N) * L.Hq * L.Wq
                                       : static_cast<int64_t>(N) * (H + 2 * kPad) * (W + 2 * kPad);
  pdl_launch(k_input_convert, grid_stride_blocks(planes * (L.kb / 16) * grid_pix), kThreads, 0, s, x, N, C, H, W, out, fmt, L, s2d_pad,
                                                                            pre_mul, q);
}

void launch_to_nchw(const void* x, int fmt, const Lay& L, float c2, float* y, int N, int C, int H, int W, int is4d,
                    cudaStream_t s, const QDev* rq) {
  int64_t total = static_cast<int64_t>(N) * C * H * W;
  pdl_launch(k_to_nchw, grid_stride_blocks(total), kThreads, 0, s, x, fmt, L, c2, y, N, C, H, W, is4d, rq ? 1 : 0,
             rq ? *rq : QDev{});
}

void launch_zero_border(void* buf, const Lay& L, int N, cudaStream_t s) {
  int planes = (L.C + L.cpc - 1) / L.cpc;
  int64_t total = static_cast<int64_t>(planes) * N * (2 * L.Wp + 2 * (L.Hp - 2 * kPad));
  pdl_launch(k_zero_border, grid_stride_blocks(total), kThreads, 0, s, buf, L, N);
}

void launch_weight_prep(const float* w, int O, int I, int KH, int KW, int Cs, int wl, const float* oc_scale,
                        float scalar, int fmt, int quant, QDev q, void* out, cudaStream_t s) {
  int cpc = (wl == WL_ROWS ? 16 : Cs) / (fmt == FMT_I8 ? 1 : 2);
  int TA = (KH + 1) / 2;
  int planes = wl == WL_S2D ? (4 * I + cpc - 1) / cpc : (I + cpc - 1) / cpc;
  if (wl == WL_S2D && fmt == FMT_F32) planes = (planes + 1) & ~1;
  int64_t total;
  if (fmt == FMT_F32) total = static_cast<int64_t>(O) * I * KH * KW;
  else if (wl == WL_TC) total = static_cast<int64_t>(KH) * KW * planes * O * cpc;
  else if (wl == WL_S2D) total = static_cast<int64_t>(TA) * TA * planes * O * cpc;
  else total = static_cast<int64_t>(O) * KH * KW * Cs;
  k_weight_prep<<<grid_stride_blocks(total), kThreads, 0, s>>>(w, O, I, KH, KW, Cs, wl, oc_scale, scalar, fmt, quant,
                                                              q, out);
}

void launch_conv_i8_simt(const int8_t* x, const int8_t* w, const ConvGeom& g, float acc_scale,
                         const EpiDev& epi, const OutDev& out, cudaStream_t s) {
  int64_t M = static_cast<int64_t>(g.N) * g.OH * g.OW;
  dim3 grid(static_cast<unsigned>((M + 63) / 64), static_cast<unsigned>((g.OC + 63) / 64));
  pdl_launch(k_conv_i8_simt, grid, 256, 0, s, x, w, g, acc_scale, epi, out);
}

// ---- 3x3 / stride 1 / pad 1 convolution over a tiny channel count (a network's
// first layer, e.g. VGG-16's 3 -> 64), bf16 mode.  K = 9*C is too small for a
// tensor-core formulation; one thread per output pixel keeps the 9*C input taps
// in registers (the padded layout makes the border taps plain zero loads) and
// runs them against the weights staged in shared memory ([k][OC] fp32, the
// 16-OC rows read as broadcasts), 16 output channels per pass.
template <int C>
__global__ void __launch_bounds__(256) k_conv3x3_tinyc(const uint16_t* __restrict__ x, const uint16_t* __restrict__ w,
                                                       ConvGeom g, EpiDev epi, OutDev out, FastDiv fd_ow, FastDiv fd_oh) {
  pdl_trigger();
  extern __shared__ __align__(16) float ws[];  // [9 * C][OC]
  const int OC = g.OC;
  for (int i = threadIdx.x; i < 9 * C * OC; i += blockDim.x) {
    const int k = i / OC, oc = i - k * OC;
    const int tap = k / C, ic = k - tap * C;
    ws[i] = bf16_to_f32(w[static_cast<int64_t>(oc) * g.Kp + tap * g.Cs + ic]);
  }
  __syncthreads();
  pdl_wait();
  const int Hp = g.H + 2 * kPad, Wp = g.W + 2 * kPad;
  const bool fast_store = !out.side && out.primary_fmt == FMT_BF16 && out.plan.kind == LAY_NORMAL &&
                          out.plan.cpc % 16 == 0;
  const uint32_t total = static_cast<uint32_t>(g.N) * g.OH * g.OW;
  for (uint32_t m = blockIdx.x * blockDim.x + threadIdx.x; m < total; m += gridDim.x * blockDim.x) {
    const uint32_t t = fdiv(m, fd_ow);
    const int ow = static_cast<int>(m - t * static_cast<uint32_t>(g.OW));
    const uint32_t n32 = fdiv(t, fd_oh);
    const int oh = static_cast<int>(t - n32 * static_cast<uint32_t>(g.OH));
    const int n = static_cast<int>(n32);
    float xin[9 * C];
#pragma unroll
    for (int kh = 0; kh < 3; ++kh)
#pragma unroll
      for (int kw = 0; kw < 3; ++kw) {
        // padded input (oh + kh, ow + kw): the zero border covers the pad-1 taps
        const int64_t pix = (static_cast<int64_t>(n) * Hp + oh + kh) * Wp + ow + kw;
        const uint2 u = __ldg(reinterpret_cast<const uint2*>(x + lay_off(g.in, pix, 0)));
        const float v4[4] = {__uint_as_float(u.x << 16), __uint_as_float(u.x & 0xffff0000u),
                             __uint_as_float(u.y << 16), __uint_as_float(u.y & 0xffff0000u)};
#pragma unroll
        for (int c = 0; c < C; ++c) xin[(kh * 3 + kw) * C + c] = v4[c];
      }
    const int64_t opix = pad_pix(n, oh, ow, g.OH, g.OW);
    for (int oc0 = 0; oc0 < OC; oc0 += 16) {
      float acc[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) acc[j] = 0.f;
#pragma unroll
      for (int k = 0; k < 9 * C; ++k) {
        const float4* wp = reinterpret_cast<const float4*>(ws + k * OC + oc0);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float4 wv = wp[q];
          acc[4 * q] = __fmaf_rn(xin[k], wv.x, acc[4 * q]);
          acc[4 * q + 1] = __fmaf_rn(xin[k], wv.y, acc[4 * q + 1]);
          acc[4 * q + 2] = __fmaf_rn(xin[k], wv.z, acc[4 * q + 2]);
          acc[4 * q + 3] = __fmaf_rn(xin[k], wv.w, acc[4 * q + 3]);
        }
      }
      // the op list once over the 16 values (op-major: one switch per op, not per value)
      int32_t codes[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) codes[j] = 0;
      for (int op = 0; op < epi.n_ops; ++op) {
        const int kind = epi.op[op];
        if (kind == E_MULC || kind == E_BIAS) {
          const float4* vp = reinterpret_cast<const float4*>(epi.vec[op] + oc0);
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const float4 v4 = __ldg(vp + q);
            const float vv[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
            for (int r = 0; r < 4; ++r)
              acc[4 * q + r] = kind == E_MULC ? __fmul_rn(acc[4 * q + r], vv[r]) : __fadd_rn(acc[4 * q + r], vv[r]);
          }
        } else if (kind == E_MULS) {
#pragma unroll
          for (int j = 0; j < 16; ++j) acc[j] = __fmul_rn(acc[j], epi.s[op]);
        } else if (kind == E_RELU) {
#pragma unroll
          for (int j = 0; j < 16; ++j) acc[j] = relu_ref(acc[j]);
        } else if (kind == E_CLIP) {
#pragma unroll
          for (int j = 0; j < 16; ++j) acc[j] = clip_ref(acc[j], epi.s[op], epi.s2[op]);
        } else if (kind == E_REQ) {
          const QDev qd = epi.q[op];
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            codes[j] = quant_code(acc[j], qd);
            acc[j] = __fmul_rn(static_cast<float>(codes[j]), qd.c2);
          }
        } else if (kind == E_RES) {
#pragma unroll
          for (int j = 0; j < 16; ++j)
            acc[j] = __fadd_rn(acc[j], load_fmt(epi.res[op], epi.res_fmt[op], lay_off(epi.res_lay[op], opix, oc0 + j)));
        }
      }
      if (fast_store) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          uint32_t w4[4];
#pragma unroll
          for (int q = 0; q < 4; ++q)
            w4[q] = pack_bf16x2(acc[8 * h + 2 * q], acc[8 * h + 2 * q + 1]);
          *reinterpret_cast<uint4*>(static_cast<char*>(out.primary) + lay_byte(out.plan, opix, oc0 + 8 * h)) =
              make_uint4(w4[0], w4[1], w4[2], w4[3]);
        }
      } else {
#pragma unroll
        for (int j = 0; j < 16; ++j) store_out(out, acc[j], codes[j], opix, oc0 + j);
      }
    }
  }
}

void launch_conv_bf16_simt(const uint16_t* x, const uint16_t* w, const ConvGeom& g, const EpiDev& epi,
                           const OutDev& out, cudaStream_t s) {
  if (g.KH == 3 && g.KW == 3 && g.sh == 1 && g.sw == 1 && g.ph == 1 && g.pw == 1 && g.C <= 4 && g.OC % 16 == 0 &&
      g.in.kind == LAY_NORMAL && g.in.cpc >= 4 && 9 * g.C * g.OC * 4 <= 48 * 1024 &&
      static_cast<int64_t>(g.N) * g.OH * g.OW < (int64_t(1) << 31) && !std::getenv("MRB200_NO_TINYC")) {
    static int sms = [] {
      int d = 0, v = 0;
      cudaGetDevice(&d);
      cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, d);
      return v > 0 ? v : 148;
    }();
    const size_t smem = static_cast<size_t>(9) * g.C * g.OC * 4;
    const FastDiv a = make_fastdiv(static_cast<uint32_t>(g.OW)), b = make_fastdiv(static_cast<uint32_t>(g.OH));
    const int grid = sms * 8;
    switch (g.C) {
      case 1: pdl_launch(k_conv3x3_tinyc<1>, grid, 256, smem, s, x, w, g, epi, out, a, b); return;
      case 2: pdl_launch(k_conv3x3_tinyc<2>, grid, 256, smem, s, x, w, g, epi, out, a, b); return;
      case 3: pdl_launch(k_conv3x3_tinyc<3>, grid, 256, smem, s, x, w, g, epi, out, a, b); return;
      default: pdl_launch(k_conv3x3_tinyc<4>, grid, 256, smem, s, x, w, g, epi, out, a, b); return;
    }
  }
  int64_t M = static_cast<int64_t>(g.N) * g.OH * g.OW;
  dim3 grid(static_cast<unsigned>((M + 63) / 64), static_cast<unsigned>((g.OC + 63) / 64));
  pdl_launch(k_conv_bf16_simt, grid, 256, 0, s, x, w, g, epi, out);
}

void launch_conv_f32_strict(const float* x, const float* w, const ConvGeom& g, const EpiDev& epi,
                            const OutDev& out, cudaStream_t s) {
  int64_t total = static_cast<int64_t>(g.N) * g.OH * g.OW * g.OC;
  pdl_launch(k_conv_f32_strict, grid_stride_blocks(total), kThreads, 0, s, x, w, g, epi, out);
}

void launch_dwconv(const void* x, int xfmt, const float* w, const ConvGeom& g, int strict, const EpiDev& epi,
                   const OutDev& out, cudaStream_t s) {
  const int cpg = xfmt == FMT_F32 ? 4 : 8;
  const int ocpc = out.plan.cpc, scpc = out.side ? out.slay.cpc : 4;
  const bool fast = g.ph <= kPad && g.pw <= kPad && g.C % cpg == 0 && g.in.kind == LAY_NORMAL && g.in.cpc % cpg == 0 &&
                    out.plan.kind == LAY_NORMAL && ocpc % 4 == 0 && scpc % 4 == 0 && (xfmt == FMT_F32 || xfmt == FMT_BF16);
  // (Measured: a row-streaming warp-per-chunk-plane form -- lane = channel pair,
  // 128-byte coalesced rows, a sliding 3x3 register window -- ran 2.30 vs 1.90 ms
  // over MobileNet-v1's 13 depthwise layers: too little load parallelism per lane.)
  if (fast && g.KH == 3 && g.KW == 3 && g.sh == g.sw && (g.sw == 1 || g.sw == 2) && g.C % 4 == 0 &&
      g.in.cpc % 4 == 0) {
    // bf16 inputs: sector-complete stores; fp32 inputs (4-channel planes): pixel-consecutive lanes
    // keep the larger input reads coalesced
    const bool pl16 = g.C % 64 == 0 && xfmt == FMT_BF16 && g.in.kb == 128 && g.in.cpc == 64;
    const bool pl8 = g.C % 32 == 0 && (xfmt == FMT_BF16 || (xfmt == FMT_F32 && g.in.kb == 128 && g.in.cpc == 32));
    const int outs = pl16 ? dw_outs(16) : pl8 ? dw_outs(8) : dw_outs(1);
    const int owq = (g.OW + outs - 1) / outs;
    const int64_t tot = static_cast<int64_t>(g.C / 4) * g.N * g.OH * owq;
    if (tot < (int64_t(1) << 31)) {
      const FastDiv a = make_fastdiv(static_cast<uint32_t>(owq)), b = make_fastdiv(static_cast<uint32_t>(g.OH)),
                    c = make_fastdiv(static_cast<uint32_t>(g.N));
      auto kern = g.sw == 1 ? (pl16 ? k_dw3x3_rb<1, 16> : pl8 ? k_dw3x3_rb<1, 8> : k_dw3x3_rb<1, 1>)
                            : (pl16 ? k_dw3x3_rb<2, 16> : pl8 ? k_dw3x3_rb<2, 8> : k_dw3x3_rb<2, 1>);
      // MobileNet's bf16 depthwise epilogues at compile time
      const bool simple = (pl16 || pl8) && out.primary_fmt == FMT_BF16 && !out.side && epi.n_ops == 3 &&
                          epi.op[0] == E_MULC && epi.op[1] == E_BIAS && (epi.op[2] == E_CLIP || epi.op[2] == E_RELU);
      const bool simple_q = !pl16 && out.primary_fmt == FMT_I8 && !out.side && epi.n_ops == 4 &&
                            epi.op[0] == E_MULC && epi.op[1] == E_BIAS && epi.op[2] == E_CLIP && epi.op[3] == E_REQ &&
                            !epi.q[3].ovf;
      if (simple_q)
        kern = pl8 ? (g.sw == 1 ? k_dw3x3_rb<1, 8, DW_MULC_BIAS_CLIP_REQ> : k_dw3x3_rb<2, 8, DW_MULC_BIAS_CLIP_REQ>)
                   : (g.sw == 1 ? k_dw3x3_rb<1, 1, DW_MULC_BIAS_CLIP_REQ> : k_dw3x3_rb<2, 1, DW_MULC_BIAS_CLIP_REQ>);
      if (simple) {
        const bool clip = epi.op[2] == E_CLIP;
        if (g.sw == 1)
          kern = pl16 ? (clip ? k_dw3x3_rb<1, 16, DW_MULC_BIAS_CLIP> : k_dw3x3_rb<1, 16, DW_MULC_BIAS_RELU>)
                      : (clip ? k_dw3x3_rb<1, 8, DW_MULC_BIAS_CLIP> : k_dw3x3_rb<1, 8, DW_MULC_BIAS_RELU>);
        else
          kern = pl16 ? (clip ? k_dw3x3_rb<2, 16, DW_MULC_BIAS_CLIP> : k_dw3x3_rb<2, 16, DW_MULC_BIAS_RELU>)
                      : (clip ? k_dw3x3_rb<2, 8, DW_MULC_BIAS_CLIP> : k_dw3x3_rb<2, 8, DW_MULC_BIAS_RELU>);
      }
      const int pl = pl16 ? 16 : pl8 ? 8 : 1;
      const int64_t pix_items = static_cast<int64_t>(g.N) * g.OH * owq;
      const unsigned gy = static_cast<unsigned>(g.C / (4 * pl));
      // about 8 resident blocks' worth per SM over the whole grid
      const unsigned gx = static_cast<unsigned>(std::max<int64_t>(
          1, std::min<int64_t>((pix_items + 256 / pl - 1) / (256 / pl), (148 * 8 + gy - 1) / gy)));
      pdl_launch(kern, dim3(gx, gy), 256, 0, s, x, xfmt, w, g, strict, epi, out, a, b, c);
      return;
    }
  }
  if (fast) {
    const int64_t tot = static_cast<int64_t>(g.C / cpg) * g.N * g.OH * g.OW;
    if (tot < (int64_t(1) << 31)) {
      pdl_launch(k_dwconv_fast, grid_stride_blocks(tot), 256, 0, s, x, xfmt, w, g, strict, epi, out,
                 make_fastdiv(static_cast<uint32_t>(g.OW)), make_fastdiv(static_cast<uint32_t>(g.OH)),
                 make_fastdiv(static_cast<uint32_t>(g.N)));
      return;
    }
  }
  int64_t total = static_cast<int64_t>(g.N) * g.OH * g.OW * g.C;
  pdl_launch(k_dwconv, grid_stride_blocks(total), kThreads, 0, s, x, xfmt, w, g, strict, epi, out);
}

void launch_maxpool(const void* x, int xfmt, const ConvGeom& g, const OutDev& out, cudaStream_t s) {
  int cpg = xfmt == FMT_F32 ? 4 : 8;
  if (g.KH == 2 && g.KW == 2 && g.sh == 2 && g.sw == 2 && g.ph == 0 && g.pw == 0 && g.H % 2 == 0 && g.W % 2 == 0 &&
      g.C % cpg == 0 && g.in.kind == LAY_NORMAL && g.in.cpc % cpg == 0 && !out.side && out.primary_fmt == xfmt &&
      out.plan.kind == LAY_NORMAL && (xfmt == FMT_F32 || xfmt == FMT_BF16)) {
    const int vec = out.plan.cpc >= cpg && out.plan.cpc % cpg == 0 && out.primary_fmt != FMT_I8 ? 1 : 0;
    const int64_t total = static_cast<int64_t>(g.C / cpg) * g.N * g.OH * g.OW;
    if (total < (int64_t(1) << 31)) {
      const FastDiv a = make_fastdiv(static_cast<uint32_t>(g.OW)), b = make_fastdiv(static_cast<uint32_t>(g.OH)),
                    c = make_fastdiv(static_cast<uint32_t>(g.N));
      pdl_launch(xfmt == FMT_F32 ? k_maxpool2x2<4> : k_maxpool2x2<2>, grid_stride_blocks(total), 256, 0, s, x, g, out,
                 a, b, c, vec);
      return;
    }
  }
  int64_t total = static_cast<int64_t>(g.N) * g.OH * g.OW * ((g.C + cpg - 1) / cpg);
  pdl_launch(k_maxpool, grid_stride_blocks(total), kThreads, 0, s, x, xfmt, g, out);
}

void launch_sum_hw(const float* x, const Lay& L, int N, int H, int W, int C, float* y, cudaStream_t s,
                   const SumOperand* op) {
  if (H * W <= 64 && C % 4 == 0 && L.cpc >= 4 && L.cpc % 4 == 0 && L.kind == LAY_NORMAL && L.kb >= 16) {
    if (C % 32 == 0) {
      const int64_t items32 = static_cast<int64_t>(N) * (C / 32);
      const SumOperand o = op ? *op : SumOperand{};
      const bool cal = op && op->quant && op->q.ovf;
      pdl_launch(cal ? k_sum_hw_warp32<true> : k_sum_hw_warp32<false>,
                 static_cast<int>(std::min<int64_t>((items32 + kSumWarps - 1) / kSumWarps, 148 * 16)), kSumWarps * 32,
                 0, s, x, L, N, H, W, C, y, o);
      return;
    }
    if (op) throw std::runtime_error("sum -> dense operand fusion needs C % 32 == 0");
    const int64_t items = static_cast<int64_t>(N) * (C / 4);
    pdl_launch(k_sum_hw_warp, static_cast<int>(std::min<int64_t>((items + 7) / 8, 148 * 8)), 256, 0, s, x, L, N, H, W,
               C, y);
    return;
  }
  int64_t total = static_cast<int64_t>(N) * C;
  pdl_launch(k_sum_hw, grid_stride_blocks(total), kThreads, 0, s, x, L, N, H, W, C, y);
}

void launch_dense_weight_t(const float* w, int M, int K, int Kp, const float* oc_scale, float scalar, int fmt,
                           int quant, QDev q, void* out, cudaStream_t s) {
  int64_t total = static_cast<int64_t>(M) * Kp;
  k_dense_weight_t<<<grid_stride_blocks(total), kThreads, 0, s>>>(w, M, K, Kp, oc_scale, scalar, fmt, quant, q, out);
}

void launch_dense(const float* x, int N, int K, int Kp, const void* w, int M, int mode, float pre_mul,
                  int quant, QDev q, float acc_scale, const EpiDev& epi, const OutDev& out, cudaStream_t s) {
  dim3 grid(static_cast<unsigned>((M + 255) / 256), static_cast<unsigned>((N + kDenseRows - 1) / kDenseRows));
  const size_t kc = static_cast<size_t>(std::min(Kp, kDenseK));
  size_t smem = (mode == 0 ? kc : kc * sizeof(float)) * kDenseRows;
  // a calibration run (mr_calibrate) observes the prologue's quantize site and the epilogue's
  bool cal = quant && q.ovf;
  for (int k = 0; k < epi.n_ops; ++k) cal = cal || (epi.op[k] == E_REQ && epi.q[k].ovf);
  if (mode == 0 || mode == 2) {  // K split across warps (exact int32 sum / bf16 tolerance)
    // bf16: 32 rows per block over 256-element K chunks, so large fc layers (VGG fc6:
    // 205 MB of weights) re-read their weights once per 32 batch rows, not per 4
    constexpr int R0 = 16, R2 = 4, R2L = 32;
    const bool big = mode == 2 && K >= 4096;
    const int R = mode == 0 ? R0 : big ? R2L : R2;
    dim3 g2(static_cast<unsigned>((M + 31) / 32), static_cast<unsigned>((N + R - 1) / R));
    if (mode == 0 && Kp <= 512) {
      // short K (the ResNet-18 head, K = 512): 512-element chunks keep all 8 warps
      // busy, 8 rows per block double the grid (1024 blocks for 256 x 1000)
      constexpr int RS = 8;
      dim3 g3(static_cast<unsigned>((M + 31) / 32), static_cast<unsigned>((N + RS - 1) / RS));
      auto k3 = cal ? k_dense_ks<0, RS, 512, true> : k_dense_ks<0, RS, 512, false>;
      pdl_launch(k3, g3, 256, 0, s, x, N, K, Kp, w, M, pre_mul, quant, q, acc_scale, epi, out);
    } else if (mode == 0) {
      auto k2 = cal ? k_dense_ks<0, R0, 1024, true> : k_dense_ks<0, R0, 1024, false>;
      pdl_launch(k2, g2, 256, 0, s, x, N, K, Kp, w, M, pre_mul, quant, q, acc_scale, epi, out);
    } else {
      auto k2 = big ? (cal ? k_dense_ks<2, R2L, 256, true> : k_dense_ks<2, R2L, 256, false>)
                    : (cal ? k_dense_ks<2, R2, 1024, true> : k_dense_ks<2, R2, 1024, false>);
      pdl_launch(k2, g2, 256, 0, s, x, N, K, Kp, w, M, pre_mul, quant, q, acc_scale, epi, out);
    }
    return;
  }
  auto kern = cal ? k_dense<true> : k_dense<false>;
  if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  pdl_launch(kern, grid, 256, smem, s, x, N, K, Kp, w, M, mode, pre_mul, quant, q, acc_scale, epi, out);
}

}  // namespace mrb200
