/* mr_oracle.c -- TEST INFRASTRUCTURE ONLY: C restatement of the reference's
 * float32 kernels (kernels.cpp).  See mr_oracle.h.  Built with
 * -O2 -ffp-contract=off (no FMA contraction, as the reference build), so
 * `acc += x * w` rounds the product and the sum separately like the
 * reference's float arithmetic. */
#include "mr_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>

/* ---- a minimal pthreads parallel-for over independent output rows ---------
 * (threading only splits independent output elements; each element's
 * arithmetic order is the reference's sequential order). */
static int g_threads = 1;
void mro_set_threads(int n) { g_threads = n < 1 ? 1 : (n > 256 ? 256 : n); }

typedef void (*row_fn)(void* ctx, int64_t i);
typedef struct { row_fn fn; void* ctx; int64_t lo, hi; } pf_job;

static void* pf_run(void* p) {
  pf_job* j = (pf_job*)p;
  for (int64_t i = j->lo; i < j->hi; ++i) j->fn(j->ctx, i);
  return NULL;
}

static void parallel_for(int64_t n, row_fn fn, void* ctx) {
  int t = g_threads;
  if (t > n) t = (int)(n > 0 ? n : 1);
  pthread_t th[256];
  pf_job jobs[256];
  for (int k = 0; k < t; ++k) {
    jobs[k].fn = fn;
    jobs[k].ctx = ctx;
    jobs[k].lo = n * k / t;
    jobs[k].hi = n * (k + 1) / t;
  }
  int started = 0;
  for (int k = 1; k < t; ++k)
    if (pthread_create(&th[k], NULL, pf_run, &jobs[k]) == 0) ++started; else pf_run(&jobs[k]);
  pf_run(&jobs[0]);
  for (int k = 1; k <= started; ++k) pthread_join(th[k], NULL);
}

/* kernels.cpp:94-131.  The float32 branch evaluates the kernel on the two
 * float operands promoted to double and rounds the double result once to
 * float (static_cast<float>(k.on_float(...))). */
void mro_binary_f32(int op, const float* a, const int64_t* as, const float* b, const int64_t* bs,
                    float* out, const int64_t* od, int nd) {
  int64_t n = 1;
  for (int d = 0; d < nd; ++d) n *= od[d];
  for (int64_t i = 0; i < n; ++i) {
    int64_t r = i, ia = 0, ib = 0;
    for (int d = nd - 1; d >= 0; --d) {
      int64_t c = r % od[d];
      r /= od[d];
      ia += c * as[d];
      ib += c * bs[d];
    }
    double x = (double)a[ia], y = (double)b[ib], z;
    switch (op) {
      case MRO_ADD: z = x + y; break;          /* kernels.cpp:160-165 */
      case MRO_SUBTRACT: z = x - y; break;     /* kernels.cpp:167-172 */
      case MRO_MULTIPLY: z = x * y; break;     /* kernels.cpp:174-179 */
      default: z = x / y; break;               /* kernels.cpp:181-188 */
    }
    out[i] = (float)z;
  }
}

void mro_relu_f32(const float* x, float* y, int64_t n) {
  for (int64_t i = 0; i < n; ++i) y[i] = x[i] > 0 ? x[i] : 0.0f;
}

void mro_round_f32(const float* x, float* y, int64_t n) {
  for (int64_t i = 0; i < n; ++i) y[i] = nearbyintf(x[i]);  /* FE_TONEAREST: half to even */
}

/* float bounds: static_cast<float>(a_min / a_max), std::min(std::max(x, lo), hi) */
void mro_clip_f32(const float* x, float* y, int64_t n, double lo, double hi) {
  const float flo = (float)lo, fhi = (float)hi;
  for (int64_t i = 0; i < n; ++i) {
    float t = x[i] < flo ? flo : x[i];  /* std::max(x, lo) returns x unless x < lo */
    y[i] = fhi < t ? fhi : t;           /* std::min(t, hi) returns t unless hi < t */
  }
}

static int64_t checked_trunc(double v) { /* kernels.cpp:320-326 */
  if (!(v > -9.2e18 && v < 9.2e18)) return v > 0 ? INT64_MAX : INT64_MIN;
  return (int64_t)v;
}

static int64_t wrap_int(int64_t v, int bits, int is_signed) { /* kernels.cpp:41-51 */
  if (bits >= 64) return v;
  const uint64_t mask = ((uint64_t)1 << bits) - 1;
  uint64_t u = (uint64_t)v & mask;
  if (is_signed && (u & ((uint64_t)1 << (bits - 1)))) u |= ~mask;
  return (int64_t)u;
}

void mro_cast_f32_to_int(const float* x, int64_t* y, int64_t n, int bits, int is_signed) {
  for (int64_t i = 0; i < n; ++i) y[i] = wrap_int(checked_trunc((double)x[i]), bits, is_signed);
}

void mro_cast_int_to_f32(const int64_t* x, float* y, int64_t n) {
  for (int64_t i = 0; i < n; ++i) y[i] = (float)(double)x[i];  /* get_double then static_cast<float> */
}

void mro_simq_f32(const float* x, float* y, int64_t n, double scale, int bits, int sign) {
  const double two_pow = ldexp(1.0, bits - sign);
  const double lo = sign ? -ldexp(1.0, bits - 1) : 0.0;
  const double hi = sign ? ldexp(1.0, bits - 1) - 1 : ldexp(1.0, bits) - 1;
  const float fscale = (float)scale, ftwo = (float)two_pow, flo = (float)lo, fhi = (float)hi;
  for (int64_t i = 0; i < n; ++i) {
    float t = x[i] / fscale * ftwo;
    float r = nearbyintf(t);
    float c = r < flo ? flo : r;  /* std::max(r, lo) */
    c = fhi < c ? fhi : c;        /* std::min(c, hi) */
    y[i] = c * fscale / ftwo;
  }
}

typedef struct {
  const float *x, *w;
  float* y;
  int64_t N, C, H, W, OC, KH, KW, sh, sw, ph, pw, OH, OW;
} conv_ctx;

static void conv_row(void* p, int64_t row) {  /* row = n * OC + oc */
  const conv_ctx* a = (const conv_ctx*)p;
  const int64_t n = row / a->OC, oc = row % a->OC, C = a->C, H = a->H, W = a->W;
  for (int64_t oh = 0; oh < a->OH; ++oh)
    for (int64_t ow = 0; ow < a->OW; ++ow) {
      float acc = 0.0f;
      for (int64_t ic = 0; ic < C; ++ic)
        for (int64_t kh = 0; kh < a->KH; ++kh)
          for (int64_t kw = 0; kw < a->KW; ++kw) {
            const int64_t h = oh * a->sh - a->ph + kh, ww = ow * a->sw - a->pw + kw;
            if (h < 0 || h >= H || ww < 0 || ww >= W) continue;
            acc += a->x[((n * C + ic) * H + h) * W + ww] * a->w[((oc * C + ic) * a->KH + kh) * a->KW + kw];
          }
      a->y[(row * a->OH + oh) * a->OW + ow] = acc;
    }
}

void mro_conv2d_f32(const float* x, const float* w, float* y, int64_t N, int64_t C, int64_t H,
                    int64_t W, int64_t OC, int64_t KH, int64_t KW, int64_t sh, int64_t sw,
                    int64_t ph, int64_t pw) {
  conv_ctx a = {x, w, y, N, C, H, W, OC, KH, KW, sh, sw, ph, pw,
                (H - KH + 2 * ph) / sh + 1, (W - KW + 2 * pw) / sw + 1};
  parallel_for(N * OC, conv_row, &a);
}

void mro_dense_f32(const float* x, const float* w, float* y, int64_t n, int64_t k, int64_t m) {
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < m; ++j) {
      float acc = 0.0f;
      for (int64_t kk = 0; kk < k; ++kk) acc += x[i * k + kk] * w[j * k + kk];
      y[i * m + j] = acc;
    }
}

void mro_bias_add_f32(const float* x, const float* b, float* y, const int64_t* dims, int nd,
                      int axis) {
  int64_t n = 1, inner = 1;
  for (int d = 0; d < nd; ++d) n *= dims[d];
  for (int d = axis + 1; d < nd; ++d) inner *= dims[d];
  for (int64_t i = 0; i < n; ++i) y[i] = x[i] + b[(i / inner) % dims[axis]];
}

void mro_sum_f32(const float* x, float* y, const int64_t* dims, int nd, const int* reduced) {
  int64_t n = 1, on = 1;
  int64_t ostr[16];
  for (int d = 0; d < nd; ++d) n *= dims[d];
  for (int d = nd - 1; d >= 0; --d) {
    ostr[d] = reduced[d] ? 0 : on;  /* keepdims only changes the output shape */
    if (!reduced[d]) on *= dims[d];
  }
  for (int64_t o = 0; o < on; ++o) y[o] = 0.0f;
  unsigned char* seeded = (unsigned char*)calloc((size_t)on, 1);
  for (int64_t i = 0; i < n; ++i) {
    int64_t r = i, oi = 0;
    for (int d = nd - 1; d >= 0; --d) {
      oi += (r % dims[d]) * ostr[d];
      r /= dims[d];
    }
    if (!seeded[oi]) {
      y[oi] = x[i];
      seeded[oi] = 1;
    } else {
      y[oi] += x[i];
    }
  }
  free(seeded);
}

void mro_max_pool2d_f32(const float* x, float* y, int64_t N, int64_t C, int64_t H, int64_t W,
                        int64_t KH, int64_t KW, int64_t sh, int64_t sw, int64_t ph, int64_t pw) {
  const int64_t OH = (H - KH + 2 * ph) / sh + 1, OW = (W - KW + 2 * pw) / sw + 1;
  for (int64_t n = 0; n < N; ++n)
    for (int64_t c = 0; c < C; ++c)
      for (int64_t oh = 0; oh < OH; ++oh)
        for (int64_t ow = 0; ow < OW; ++ow) {
          float acc = 0.0f;
          int seeded = 0;
          for (int64_t kh = 0; kh < KH; ++kh)
            for (int64_t kw = 0; kw < KW; ++kw) {
              const int64_t h = oh * sh - ph + kh, ww = ow * sw - pw + kw;
              if (h < 0 || h >= H || ww < 0 || ww >= W) continue;
              const float v = x[((n * C + c) * H + h) * W + ww];
              if (!seeded) {
                acc = v;
                seeded = 1;
              } else {
                acc = acc < v ? v : acc;  /* std::max(acc, v) */
              }
            }
          y[((n * C + c) * OH + oh) * OW + ow] = acc;
        }
}

void mro_dwconv2d_f32(const float* x, const float* w, float* y, int64_t N, int64_t C, int64_t H, int64_t W,
                      int64_t KH, int64_t KW, int64_t sh, int64_t sw, int64_t ph, int64_t pw) {
  const int64_t OH = (H - KH + 2 * ph) / sh + 1, OW = (W - KW + 2 * pw) / sw + 1;
  for (int64_t n = 0; n < N; ++n)
    for (int64_t c = 0; c < C; ++c)
      for (int64_t oh = 0; oh < OH; ++oh)
        for (int64_t ow = 0; ow < OW; ++ow) {
          float acc = 0.0f;
          for (int64_t kh = 0; kh < KH; ++kh)
            for (int64_t kw = 0; kw < KW; ++kw) {
              const int64_t h = oh * sh - ph + kh, ww = ow * sw - pw + kw;
              if (h < 0 || h >= H || ww < 0 || ww >= W) continue;
              acc += x[((n * C + c) * H + h) * W + ww] * w[(c * KH + kh) * KW + kw];
            }
          y[((n * C + c) * OH + oh) * OW + ow] = acc;
        }
}
