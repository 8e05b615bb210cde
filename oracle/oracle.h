/* TEST INFRASTRUCTURE — NOT PRODUCT CODE.
 *
 * C restatement of the reference's (tzc, /root/reference/proj) arithmetic on
 * the tensorized Conv2D/Matmul path, used only by tests/, bench.py's
 * cpu_baseline leg and __graft_entry__.smoke() as the checker.
 *
 * Parity of this restatement is PINNED two ways (tests/test_oracle.py):
 *   - against the reference itself, compiled unmodified into
 *     oracle/_ref/libtzc_ref.so (eval_reference / random_inputs on the same
 *     op text and seeds), and
 *   - against the golden vectors the reference's own tests freeze
 *     (proj/tests/test_vm.cpp:49-137, proj/tests/test_dtype.cpp:74-163,
 *     proj/python/tests/test_smoke.py:31-40), committed under tests/golden/.
 */
#ifndef TZC_ORACLE_H
#define TZC_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* TNSR dtype codes, proj/src/vm.cpp:694-704. */
enum { ORC_U8 = 0, ORC_I8, ORC_U16, ORC_I16, ORC_U32, ORC_I32, ORC_F16, ORC_F32 };

/* random_tensor (proj/src/vm.cpp:38-57): mt19937_64(seed); ints uniform over
 * the full declared range via lo + rng() % span; floats (rng()>>11)*2^-53 in
 * [0,1) rounded to the format. Output packed at declared width. */
void orc_random_fill(int dtype, uint64_t seed, int64_t n, void* out);

/* Bit-exact binary16 RNE from binary64 (proj/src/dtype.cpp:53-101). */
uint16_t orc_f64_to_f16_bits(double x);
double orc_f16_bits_to_f64(uint16_t bits);
int64_t orc_wrap_int(int64_t v, int bits, int is_signed); /* dtype.cpp:40-48 */
int64_t orc_float_to_int(double f);                       /* vm.cpp:79-84 */

/* ---- int8 profile (u8 data x i8 weight -> i32, wrap mod 2^32) ------------ */
/* C[m,n] = seed[m,n] + sum_k A[m,k]*B[n,k]; rows [m_lo, m_hi) only.
 * matmul_tdsl int8 layout (proj/src/workloads.cpp:41-63). seed may be NULL. */
void orc_matmul_u8i8(int64_t M, int64_t N, int64_t K, const uint8_t* A,
                     const int8_t* B, const int32_t* seed, int32_t* C,
                     int64_t m_lo, int64_t m_hi);

/* Batched NHWC valid conv over a pre-padded input:
 * out[n,oh,ow,k] = seed + sum_{r,s,c} x[n,oh*st+r,ow*st+s,c] * w[k,r,s,c].
 * Images [n_lo, n_hi) only. */
void orc_conv2d_nhwc_u8i8(int64_t N, int64_t Hp, int64_t Wp, int64_t C, int64_t K,
                          int64_t R, int64_t S, int64_t st, const uint8_t* x,
                          const int8_t* w, const int32_t* seed, int32_t* out,
                          int64_t n_lo, int64_t n_hi);

/* conv2d_tdsl channel-blocked layout (proj/src/workloads.cpp:65-92):
 * data[C/cb,H,W,cb], kernel[K/kb,C/cb,R,R,kb,cb], out[K/kb,OH,OW,kb].
 * Output rows oh in [oh_lo, oh_hi) only. */
void orc_conv2d_blocked_u8i8(int64_t C, int64_t H, int64_t K, int64_t R,
                             int64_t st, int64_t cb, int64_t kb, const uint8_t* data,
                             const int8_t* kernel, const int32_t* seed, int32_t* out,
                             int64_t oh_lo, int64_t oh_hi);

/* Q[i] = cast<i8>(cast<fp32>(C[i]) * s): fp32 RNE, mul RNE, trunc toward
 * zero with int64 saturation, wrap mod 256 (vm.cpp:79-84,136-164). */
void orc_requant_i8(int64_t n, const int32_t* c, float s, int8_t* q);

/* ---- fp16 profile (fp16 x fp16 -> fp32; each op rounded, reduction loops
 * in declared order, last fastest; vm.cpp:482-495) ------------------------- */
/* matmul_tdsl fp16 layout: B is [K, N]. */
void orc_matmul_f16(int64_t M, int64_t N, int64_t K, const uint16_t* A,
                    const uint16_t* B, const float* seed, float* C, int64_t m_lo,
                    int64_t m_hi);
void orc_conv2d_nhwc_f16(int64_t N, int64_t Hp, int64_t Wp, int64_t C, int64_t K,
                         int64_t R, int64_t S, int64_t st, const uint16_t* x,
                         const uint16_t* w, const float* seed, float* out,
                         int64_t n_lo, int64_t n_hi);
void orc_conv2d_blocked_f16(int64_t C, int64_t H, int64_t K, int64_t R, int64_t st,
                            int64_t cb, int64_t kb, const uint16_t* data,
                            const uint16_t* kernel, const float* seed, float* out,
                            int64_t oh_lo, int64_t oh_hi);
/* H[i] = cast<fp16>(C[i]) (binary16 RNE of the fp32 value). */
void orc_cast_f16(int64_t n, const float* c, uint16_t* h);

#ifdef __cplusplus
}
#endif
#endif
