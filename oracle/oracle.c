/* TEST INFRASTRUCTURE — NOT PRODUCT CODE.  See oracle.h for what this is,
 * which reference code each function restates, and how it is pinned. */
#include "oracle.h"

#include <math.h>
#include <string.h>

/* ---- std::mt19937_64 (the engine random_tensor uses, vm.cpp:40) ---------- */
typedef struct {
  uint64_t s[312];
  int i;
} mt64;

static void mt64_seed(mt64* g, uint64_t seed) {
  g->s[0] = seed;
  for (int k = 1; k < 312; ++k)
    g->s[k] = 6364136223846793005ULL * (g->s[k - 1] ^ (g->s[k - 1] >> 62)) + (uint64_t)k;
  g->i = 312;
}

static uint64_t mt64_next(mt64* g) {
  if (g->i >= 312) {
    for (int k = 0; k < 312; ++k) {
      uint64_t y = (g->s[k] & 0xFFFFFFFF80000000ULL) | (g->s[(k + 1) % 312] & 0x7FFFFFFFULL);
      uint64_t v = g->s[(k + 156) % 312] ^ (y >> 1);
      if (y & 1) v ^= 0xB5026F5AA96619E9ULL;
      g->s[k] = v;
    }
    g->i = 0;
  }
  uint64_t y = g->s[g->i++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

/* ---- scalar semantics ------------------------------------------------------ */
int64_t orc_wrap_int(int64_t v, int bits, int is_signed) {
  if (bits >= 64) return v;
  uint64_t mask = (1ULL << bits) - 1;
  uint64_t u = (uint64_t)v & mask;
  if (is_signed && (u >> (bits - 1)) & 1) u |= ~mask;
  return (int64_t)u;
}

int64_t orc_float_to_int(double f) {
  if (isnan(f)) return 0;
  if (f >= 9223372036854775808.0) return INT64_MAX;
  if (f <= -9223372036854775808.0) return INT64_MIN;
  return (int64_t)trunc(f);
}

/* binary16 RNE: scale |x| so one unit == one binary16 ulp (exact, power-of-two
 * scaling), round to nearest even with rint, then assemble the fields. */
uint16_t orc_f64_to_f16_bits(double x) {
  uint16_t sign = signbit(x) ? 0x8000 : 0;
  if (isnan(x)) return sign | 0x7e00;
  double a = fabs(x);
  if (isinf(a)) return sign | 0x7c00;
  if (a == 0.0) return sign;
  int e2;
  frexp(a, &e2);
  int msb = e2 - 1; /* a in [2^msb, 2^(msb+1)) */
  if (msb > 15) return sign | 0x7c00;
  int ulp = msb < -14 ? -24 : msb - 10;
  double q = rint(ldexp(a, -ulp)); /* default FE_TONEAREST: ties to even */
  if (msb < -14) return sign | (uint16_t)q; /* 1024 == smallest normal, 0x400 */
  if (q >= 2048.0) {
    q = 1024.0;
    msb += 1;
  }
  if (msb > 15) return sign | 0x7c00;
  return sign | (uint16_t)(((msb + 15) << 10) | ((int)q - 1024));
}

double orc_f16_bits_to_f64(uint16_t b) {
  double s = (b & 0x8000) ? -1.0 : 1.0;
  int e = (b >> 10) & 0x1f, f = b & 0x3ff;
  if (e == 0x1f) return f ? NAN : s * INFINITY;
  if (e == 0) return s * ldexp((double)f, -24);
  return s * ldexp((double)(f | 0x400), e - 25);
}

void orc_random_fill(int dtype, uint64_t seed, int64_t n, void* out) {
  mt64 g;
  mt64_seed(&g, seed);
  switch (dtype) {
    case ORC_F16:
      for (int64_t i = 0; i < n; ++i)
        ((uint16_t*)out)[i] = orc_f64_to_f16_bits((double)(mt64_next(&g) >> 11) * 0x1.0p-53);
      return;
    case ORC_F32:
      for (int64_t i = 0; i < n; ++i)
        ((float*)out)[i] = (float)((double)(mt64_next(&g) >> 11) * 0x1.0p-53);
      return;
    default: {
      static const int bits[] = {8, 8, 16, 16, 32, 32};
      static const int sgn[] = {0, 1, 0, 1, 0, 1};
      int b = bits[dtype];
      uint64_t span = 1ULL << b;
      int64_t lo = sgn[dtype] ? -(INT64_C(1) << (b - 1)) : 0;
      int bytes = b / 8;
      for (int64_t i = 0; i < n; ++i) {
        uint64_t v = (uint64_t)(lo + (int64_t)(mt64_next(&g) % span));
        memcpy((uint8_t*)out + i * bytes, &v, (size_t)bytes); /* little-endian */
      }
    }
  }
}

static int32_t wrap32(int64_t v) { return (int32_t)(uint32_t)(uint64_t)v; }

/* fp32 accumulate-form step: t = round_f32(a*b); acc = round_f32(acc + t),
 * both computed in binary64 first exactly as vm.cpp:154-164,486-488. */
static float fstep(float acc, uint16_t a, uint16_t b) {
  float t = (float)(orc_f16_bits_to_f64(a) * orc_f16_bits_to_f64(b));
  return (float)((double)acc + (double)t);
}

/* ---- int8 profile ----------------------------------------------------------- */
void orc_matmul_u8i8(int64_t M, int64_t N, int64_t K, const uint8_t* A,
                     const int8_t* B, const int32_t* seed, int32_t* C, int64_t m_lo,
                     int64_t m_hi) {
  (void)M;
  for (int64_t m = m_lo; m < m_hi; ++m)
    for (int64_t n = 0; n < N; ++n) {
      const uint8_t* a = A + m * K;
      const int8_t* b = B + n * K;
      int64_t acc = seed ? seed[m * N + n] : 0;
      for (int64_t k = 0; k < K; ++k) acc += (int32_t)a[k] * (int32_t)b[k];
      C[m * N + n] = wrap32(acc);
    }
}

void orc_conv2d_nhwc_u8i8(int64_t N, int64_t Hp, int64_t Wp, int64_t C, int64_t K,
                          int64_t R, int64_t S, int64_t st, const uint8_t* x,
                          const int8_t* w, const int32_t* seed, int32_t* out,
                          int64_t n_lo, int64_t n_hi) {
  (void)N;
  int64_t OH = (Hp - R) / st + 1, OW = (Wp - S) / st + 1;
  for (int64_t n = n_lo; n < n_hi; ++n)
    for (int64_t oh = 0; oh < OH; ++oh)
      for (int64_t ow = 0; ow < OW; ++ow)
        for (int64_t k = 0; k < K; ++k) {
          int64_t o = ((n * OH + oh) * OW + ow) * K + k;
          int64_t acc = seed ? seed[o] : 0;
          for (int64_t r = 0; r < R; ++r)
            for (int64_t s = 0; s < S; ++s) {
              const uint8_t* px = x + ((n * Hp + oh * st + r) * Wp + ow * st + s) * C;
              const int8_t* pw = w + ((k * R + r) * S + s) * C;
              for (int64_t c = 0; c < C; ++c) acc += (int32_t)px[c] * (int32_t)pw[c];
            }
          out[o] = wrap32(acc);
        }
}

void orc_conv2d_blocked_u8i8(int64_t C, int64_t H, int64_t K, int64_t R, int64_t st,
                             int64_t cb, int64_t kb, const uint8_t* data,
                             const int8_t* kernel, const int32_t* seed, int32_t* out,
                             int64_t oh_lo, int64_t oh_hi) {
  int64_t CO = C / cb, KO = K / kb, OH = (H - R) / st + 1, OW = OH, W = H;
  for (int64_t ko = 0; ko < KO; ++ko)
    for (int64_t oh = oh_lo; oh < oh_hi; ++oh)
      for (int64_t ow = 0; ow < OW; ++ow)
        for (int64_t ki = 0; ki < kb; ++ki) {
          int64_t o = ((ko * OH + oh) * OW + ow) * kb + ki;
          int64_t acc = seed ? seed[o] : 0;
          for (int64_t co = 0; co < CO; ++co)
            for (int64_t r = 0; r < R; ++r)
              for (int64_t s = 0; s < R; ++s)
                for (int64_t ci = 0; ci < cb; ++ci) {
                  int64_t di = ((co * H + oh * st + r) * W + ow * st + s) * cb + ci;
                  int64_t wi = ((((ko * CO + co) * R + r) * R + s) * kb + ki) * cb + ci;
                  acc += (int32_t)data[di] * (int32_t)kernel[wi];
                }
          out[o] = wrap32(acc);
        }
}

void orc_requant_i8(int64_t n, const int32_t* c, float s, int8_t* q) {
  for (int64_t i = 0; i < n; ++i) {
    float cf = (float)c[i];                    /* cast<fp32>: RNE */
    float p = (float)((double)cf * (double)s); /* fp32 Mul: exact in f64, one RNE */
    q[i] = (int8_t)orc_wrap_int(orc_float_to_int((double)p), 8, 1);
  }
}

/* ---- fp16 profile ------------------------------------------------------------ */
void orc_matmul_f16(int64_t M, int64_t N, int64_t K, const uint16_t* A,
                    const uint16_t* B, const float* seed, float* C, int64_t m_lo,
                    int64_t m_hi) {
  (void)M;
  for (int64_t m = m_lo; m < m_hi; ++m)
    for (int64_t n = 0; n < N; ++n) {
      float acc = seed ? seed[m * N + n] : 0.0f;
      for (int64_t k = 0; k < K; ++k) acc = fstep(acc, A[m * K + k], B[k * N + n]);
      C[m * N + n] = acc;
    }
}

void orc_conv2d_nhwc_f16(int64_t N, int64_t Hp, int64_t Wp, int64_t C, int64_t K,
                         int64_t R, int64_t S, int64_t st, const uint16_t* x,
                         const uint16_t* w, const float* seed, float* out,
                         int64_t n_lo, int64_t n_hi) {
  (void)N;
  int64_t OH = (Hp - R) / st + 1, OW = (Wp - S) / st + 1;
  for (int64_t n = n_lo; n < n_hi; ++n)
    for (int64_t oh = 0; oh < OH; ++oh)
      for (int64_t ow = 0; ow < OW; ++ow)
        for (int64_t k = 0; k < K; ++k) {
          int64_t o = ((n * OH + oh) * OW + ow) * K + k;
          float acc = seed ? seed[o] : 0.0f;
          for (int64_t r = 0; r < R; ++r)
            for (int64_t s = 0; s < S; ++s) {
              const uint16_t* px = x + ((n * Hp + oh * st + r) * Wp + ow * st + s) * C;
              const uint16_t* pw = w + ((k * R + r) * S + s) * C;
              for (int64_t c = 0; c < C; ++c) acc = fstep(acc, px[c], pw[c]);
            }
          out[o] = acc;
        }
}

void orc_conv2d_blocked_f16(int64_t C, int64_t H, int64_t K, int64_t R, int64_t st,
                            int64_t cb, int64_t kb, const uint16_t* data,
                            const uint16_t* kernel, const float* seed, float* out,
                            int64_t oh_lo, int64_t oh_hi) {
  int64_t CO = C / cb, KO = K / kb, OH = (H - R) / st + 1, OW = OH, W = H;
  for (int64_t ko = 0; ko < KO; ++ko)
    for (int64_t oh = oh_lo; oh < oh_hi; ++oh)
      for (int64_t ow = 0; ow < OW; ++ow)
        for (int64_t ki = 0; ki < kb; ++ki) {
          int64_t o = ((ko * OH + oh) * OW + ow) * kb + ki;
          float acc = seed ? seed[o] : 0.0f;
          for (int64_t co = 0; co < CO; ++co)
            for (int64_t r = 0; r < R; ++r)
              for (int64_t s = 0; s < R; ++s)
                for (int64_t ci = 0; ci < cb; ++ci) {
                  int64_t di = ((co * H + oh * st + r) * W + ow * st + s) * cb + ci;
                  int64_t wi = ((((ko * CO + co) * R + r) * R + s) * kb + ki) * cb + ci;
                  acc = fstep(acc, data[di], kernel[wi]);
                }
          out[o] = acc;
        }
}

void orc_cast_f16(int64_t n, const float* c, uint16_t* h) {
  for (int64_t i = 0; i < n; ++i) h[i] = orc_f64_to_f16_bits((double)c[i]);
}
