// gcx_device.cuh — bit-exact device arithmetic for the CGX codec on sm_100a.
//
// Everything here reproduces the reference's FP64/integer semantics
// (/root/reference/proj/src/codec.cpp:24-95, include/gcomm/util.hpp:14-29)
// WITHOUT the XU-pipe conversion instructions (F2F/I2F/F2I), which the first
// ncu capture showed saturating the XU pipe at 193% of peak.  Conversions are
// rebuilt from integer/FP64 pipe operations; each trick is exact and checked
// bit-for-bit against the oracle by tests/test_gpu_codec.py.
#pragma once

#include <cstdint>

namespace gcx_dev {

// |v| as an exact double: float exponent rebias in the integer pipes.  Zero
// and subnormals (exponent field 0) take the slow conversion.
__device__ __forceinline__ double f32abs_to_f64(uint32_t u_abs) {
  double d = __hiloint2double(int((u_abs >> 3) + 0x38000000u), int(u_abs << 29));
  if (u_abs < 0x00800000u) d = u_abs == 0 ? 0.0 : double(__uint_as_float(u_abs));
  return d;
}

// Same, branch-free (zero/subnormal via (2^52 + m) - 2^52 = m, times 2^-149),
// for dependency chains where a branch would sit on the critical path.
__device__ __forceinline__ double f32abs_to_f64_nb(uint32_t u_abs) {
  const double dn = __hiloint2double(int((u_abs >> 3) + 0x38000000u), int(u_abs << 29));
  const double ds = __dmul_rn(__dsub_rn(__hiloint2double(0x43300000, int(u_abs)), 4503599627370496.0),
                              0x1p-149);
  return u_abs < 0x00800000u ? ds : dn;
}

// RN-even double -> float for a non-negative finite q below 2^128; results
// below the normal float range take the slow conversion.
__device__ __forceinline__ float f64pos_to_f32_rn(double q) {
  const unsigned long long D = __double_as_longlong(q);
  if (D < 0x3810000000000000ull) return __double2float_rn(q);
  const unsigned long long R = D + 0x0FFFFFFFull + ((D >> 29) & 1ull);
  return __uint_as_float(uint32_t(R >> 29) - (896u << 23));
}

// small non-negative integer (< 2^31) as an exact double
__device__ __forceinline__ double u32_to_f64(uint32_t k) {
  return __dsub_rn(__hiloint2double(0x43300000, int(k)), 4503599627370496.0);
}

// ---------------------------------------------------------------------------
// mix64 (util.hpp:14-19) on (lo, hi) 32-bit halves.  The reference form
// compiles to ~27 ops per call, ~2/3 of them on the ALU pipe (SHF/LOP3/
// IADD3).  Here the high-word right shifts are done as IMAD.HI with an opaque
// power-of-two multiplier so they issue on the FMA pipe instead, balancing
// the two pipes.  `Opq` carries the multipliers in registers ptxas cannot
// constant-fold back into shifts.
// ---------------------------------------------------------------------------
struct Opq {
  uint32_t m30, m27, m31;  // 2^(32-k): hi >> k == mulhi(hi, 2^(32-k))
};

__device__ __forceinline__ Opq make_opq() {
  Opq o{4u, 32u, 2u};
  asm volatile("" : "+r"(o.m30), "+r"(o.m27), "+r"(o.m31));
  return o;
}

// z ^= z >> k  with hi >> k on the FMA pipe
__device__ __forceinline__ void xorshift(uint32_t& lo, uint32_t& hi, uint32_t k, uint32_t mk) {
  const uint32_t f = __funnelshift_r(lo, hi, k);  // (z >> k).lo  [ALU]
  const uint32_t t = __umulhi(hi, mk);            // (z >> k).hi  [FMA]
  lo ^= f;
  hi ^= t;
}

// z *= C (mod 2^64): 3 FMA-pipe ops
__device__ __forceinline__ void mul64c(uint32_t& lo, uint32_t& hi, uint32_t cl, uint32_t ch) {
  const unsigned long long w = (unsigned long long)lo * cl;
  uint32_t nhi = uint32_t(w >> 32);
  nhi += lo * ch;
  nhi += hi * cl;
  lo = uint32_t(w);
  hi = nhi;
}

__device__ __forceinline__ void mix64_split(uint32_t& lo, uint32_t& hi, const Opq& o) {
  // z += 0x9e3779b97f4a7c15
  asm("add.cc.u32 %0, %0, 0x7f4a7c15;\n\taddc.u32 %1, %1, 0x9e3779b9;" : "+r"(lo), "+r"(hi));
  xorshift(lo, hi, 30, o.m30);
  mul64c(lo, hi, 0x1ce4e5b9u, 0xbf58476du);
  xorshift(lo, hi, 27, o.m27);
  mul64c(lo, hi, 0x133111ebu, 0x94d049bbu);
  xorshift(lo, hi, 31, o.m31);
}

// Variant "ALU shifts, 3-IMAD multiplies": z *= C as mul.wide + two chained
// mad.lo (3 FMA-pipe ops, no separate add), all shifts on the ALU pipe.
__device__ __forceinline__ void mul64c_mad(uint32_t& lo, uint32_t& hi, uint32_t cl, uint32_t ch) {
  unsigned long long w;
  asm("mul.wide.u32 %0, %1, %2;" : "=l"(w) : "r"(lo), "r"(cl));
  uint32_t t, nhi;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(t) : "r"(lo), "r"(ch), "r"(uint32_t(w >> 32)));
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(nhi) : "r"(hi), "r"(cl), "r"(t));
  lo = uint32_t(w);
  hi = nhi;
}

__device__ __forceinline__ void xorshift_alu(uint32_t& lo, uint32_t& hi, uint32_t k) {
  const uint32_t f = __funnelshift_r(lo, hi, k);
  const uint32_t t = hi >> k;
  lo ^= f;
  hi ^= t;
}

__device__ __forceinline__ void mix64_alu(uint32_t& lo, uint32_t& hi) {
  asm("add.cc.u32 %0, %0, 0x7f4a7c15;\n\taddc.u32 %1, %1, 0x9e3779b9;" : "+r"(lo), "+r"(hi));
  xorshift_alu(lo, hi, 30);
  mul64c_mad(lo, hi, 0x1ce4e5b9u, 0xbf58476du);
  xorshift_alu(lo, hi, 27);
  mul64c_mad(lo, hi, 0x133111ebu, 0x94d049bbu);
  xorshift_alu(lo, hi, 31);
}

__device__ __forceinline__ void draw_key_alu(uint32_t i_lo, uint32_t i_hi, uint32_t b_lo,
                                             uint32_t b_hi, uint32_t s_lo, uint32_t s_hi,
                                             uint32_t& h_lo, uint32_t& h_hi) {
  uint32_t lo = i_lo, hi = i_hi;
  mix64_alu(lo, hi);
  lo ^= b_lo;
  hi ^= b_hi;
  mix64_alu(lo, hi);
  lo ^= s_lo;
  hi ^= s_hi;
  mix64_alu(lo, hi);
  h_lo = lo;
  h_hi = hi;
}

// Variant "opaque shifts": the shift amounts live in registers ptxas cannot
// constant-fold, so every 64-bit right shift stays a funnel SHF (half rate on
// B200) instead of being rewritten as IMAD.HI by a power of two (quarter rate
// on B200; scripts/piperate.cu measures both).
struct Shk {
  uint32_t k30, k27, k31;
};

__device__ __forceinline__ Shk make_shk() {
  Shk k{30u, 27u, 31u};
  asm volatile("" : "+r"(k.k30), "+r"(k.k27), "+r"(k.k31));
  return k;
}

__device__ __forceinline__ void xorshift_shf(uint32_t& lo, uint32_t& hi, uint32_t k) {
  const uint32_t f = __funnelshift_r(lo, hi, k);
  const uint32_t t = __funnelshift_r(hi, 0u, k);
  lo ^= f;
  hi ^= t;
}

__device__ __forceinline__ void mix64_shf(uint32_t& lo, uint32_t& hi, const Shk& k) {
  asm("add.cc.u32 %0, %0, 0x7f4a7c15;\n\taddc.u32 %1, %1, 0x9e3779b9;" : "+r"(lo), "+r"(hi));
  xorshift_shf(lo, hi, k.k30);
  mul64c(lo, hi, 0x1ce4e5b9u, 0xbf58476du);
  xorshift_shf(lo, hi, k.k27);
  mul64c(lo, hi, 0x133111ebu, 0x94d049bbu);
  xorshift_shf(lo, hi, k.k31);
}

__device__ __forceinline__ void draw_key_shf(uint32_t i_lo, uint32_t i_hi, uint32_t b_lo,
                                             uint32_t b_hi, uint32_t s_lo, uint32_t s_hi,
                                             const Shk& k, uint32_t& h_lo, uint32_t& h_hi) {
  uint32_t lo = i_lo, hi = i_hi;
  mix64_shf(lo, hi, k);
  lo ^= b_lo;
  hi ^= b_hi;
  mix64_shf(lo, hi, k);
  lo ^= s_lo;
  hi ^= s_hi;
  mix64_shf(lo, hi, k);
  h_lo = lo;
  h_hi = hi;
}

// h = mix64(seed ^ mix64(b ^ mix64(i)))  (uniform01's key, util.hpp:26-29)
__device__ __forceinline__ void draw_key(uint32_t i_lo, uint32_t i_hi, uint32_t b_lo, uint32_t b_hi,
                                         uint32_t s_lo, uint32_t s_hi, const Opq& o,
                                         uint32_t& h_lo, uint32_t& h_hi) {
  uint32_t lo = i_lo, hi = i_hi;
  mix64_split(lo, hi, o);
  lo ^= b_lo;
  hi ^= b_hi;
  mix64_split(lo, hi, o);
  lo ^= s_lo;
  hi ^= s_hi;
  mix64_split(lo, hi, o);
  h_lo = lo;
  h_hi = hi;
}

// Top word of the uniform01 key only: the final `z ^= z >> 31` of the outer
// mix64 is applied to the high word alone (the low word is needed only when
// the 32-bit comparison in quantize_field32 is ambiguous, and that path
// recomputes the whole key).  HV selects where the high-word right shifts
// issue: 0 = funnel SHF with opaque amounts (ALU pipe), 1 = plain shifts
// (ptxas's choice), 2 = IMAD.HI by an opaque power of two (FMA pipe).
#ifndef GCX_HASH_HV
#define GCX_HASH_HV 0
#endif
template <int HV>
__device__ __forceinline__ uint32_t shr_hi(uint32_t hi, uint32_t k, uint32_t mk) {
  if (HV == 0) return __funnelshift_r(hi, 0u, k);
  if (HV == 1) return hi >> k;
  return __umulhi(hi, mk);
}

struct HashK {
  uint32_t k30, k27, k31, m30, m27, m31;
};

__device__ __forceinline__ HashK make_hashk() {
  HashK h{30u, 27u, 31u, 4u, 32u, 2u};
  asm volatile("" : "+r"(h.k30), "+r"(h.k27), "+r"(h.k31), "+r"(h.m30), "+r"(h.m27), "+r"(h.m31));
  return h;
}

template <int HV>
__device__ __forceinline__ void xorshift_v(uint32_t& lo, uint32_t& hi, uint32_t k, uint32_t mk) {
  const uint32_t f = __funnelshift_r(lo, hi, k);
  const uint32_t t = shr_hi<HV>(hi, k, mk);
  lo ^= f;
  hi ^= t;
}

template <int HV>
__device__ __forceinline__ void mix64_v(uint32_t& lo, uint32_t& hi, const HashK& k) {
  asm("add.cc.u32 %0, %0, 0x7f4a7c15;\n\taddc.u32 %1, %1, 0x9e3779b9;" : "+r"(lo), "+r"(hi));
  xorshift_v<HV>(lo, hi, HV == 1 ? 30u : k.k30, k.m30);
  mul64c(lo, hi, 0x1ce4e5b9u, 0xbf58476du);
  xorshift_v<HV>(lo, hi, HV == 1 ? 27u : k.k27, k.m27);
  mul64c(lo, hi, 0x133111ebu, 0x94d049bbu);
  xorshift_v<HV>(lo, hi, HV == 1 ? 31u : k.k31, k.m31);
}

// The seed-independent part of the key: T(i) = mix64(b ^ mix64(i)).
template <int HV = GCX_HASH_HV>
__device__ __forceinline__ void draw_prefix(uint32_t i, uint32_t b, const HashK& k, uint32_t& lo,
                                            uint32_t& hi) {
  lo = i;
  hi = 0u;
  mix64_v<HV>(lo, hi, k);
  lo ^= b;
  mix64_v<HV>(lo, hi, k);
}

// Top word of mix64(seed ^ T): the final `z ^= z >> 31` is applied to the
// high word alone.
template <int HV = GCX_HASH_HV>
__device__ __forceinline__ uint32_t key_hi_from_prefix(uint32_t lo, uint32_t hi, uint32_t s_lo,
                                                       uint32_t s_hi, const HashK& k) {
  lo ^= s_lo;
  hi ^= s_hi;
  asm("add.cc.u32 %0, %0, 0x7f4a7c15;\n\taddc.u32 %1, %1, 0x9e3779b9;" : "+r"(lo), "+r"(hi));
  xorshift_v<HV>(lo, hi, HV == 1 ? 30u : k.k30, k.m30);
  mul64c(lo, hi, 0x1ce4e5b9u, 0xbf58476du);
  xorshift_v<HV>(lo, hi, HV == 1 ? 27u : k.k27, k.m27);
  // hi word of z * 0x94d049bb133111eb, then hi ^= hi >> 31
  const uint32_t h = __umulhi(lo, 0x133111ebu) + lo * 0x94d049bbu + hi * 0x133111ebu;
  return h ^ shr_hi<HV>(h, HV == 1 ? 31u : k.k31, k.m31);
}

// top word of the uniform01 key of (seed, b, i); the low word is needed only
// when the 32-bit comparison in quantize_field32 ties, and that path
// recomputes the whole key
template <int HV = GCX_HASH_HV>
__device__ __forceinline__ uint32_t draw_key_hi(uint32_t i, uint32_t b, uint32_t s_lo,
                                                uint32_t s_hi, const HashK& k) {
  uint32_t lo, hi;
  draw_prefix<HV>(i, b, k, lo, hi);
  return key_hi_from_prefix<HV>(lo, hi, s_lo, s_hi, k);
}

// |v| (normal, non-zero float bits) as an exact double: exponent rebias only.
__device__ __forceinline__ double f32normal_to_f64(uint32_t u_abs) {
  return __hiloint2double(int((u_abs >> 3) + 0x38000000u), int(u_abs << 29));
}

// ---------------------------------------------------------------------------
// Fast exact form of one element of codec::quantize (codec.cpp:50-64) for
// normal non-zero |v| (the caller checks and falls back otherwise):
//   a  = RN(|v|/norm)       (q0/r/a correction as in quantize_field)
//   X  = RN(a * s * 2^32)   = RN(a*s) * 2^32 exactly (power-of-two scaling)
//   T  = RZ(X + 2^52)       = 2^52 + floor(X): x < 2^20, so the low word of T
//                              is fl = floor(frac(x) * 2^32) and the high
//                              word's low 20 bits are level = trunc(x)
//   uniform01 < p  <=>  k53 < frac(x)*2^53 with k53 = h >> 11; decided by the
//   top key word alone unless hh == fl: hh < fl -> up, hh > fl -> not up.
// `mn` accumulates min(hh ^ fl): zero flags an ambiguous element, which the
// caller recomputes with the full key.  Returns level' | sign << BITS.
// ---------------------------------------------------------------------------
template <uint32_t BITS>
__device__ __forceinline__ uint32_t quantize_field32(uint32_t u, double av, double nd, double y,
                                                     uint32_t hh, uint32_t& mn) {
  constexpr uint32_t S = (1u << BITS) - 1;
  constexpr double S2 = double(S) * 4294967296.0;
  const double q0 = __dmul_rn(av, y);
  const double r = __fma_rn(-nd, q0, av);
  const double a = __fma_rn(r, y, q0);
  const double X = __dmul_rn(a, S2);
  const double T = __dadd_rz(X, 4503599627370496.0);
  const uint32_t fl = uint32_t(__double2loint(T));
  const uint32_t lv = uint32_t(__double2hiint(T)) & 0xFFFFFu;
  mn = min(mn, hh ^ fl);
  const uint32_t l = min(lv + (hh < fl ? 1u : 0u), S);
  return l | ((u >> 31) << BITS);
}

// reference form, for the microbenchmark and as documentation
__device__ __forceinline__ uint64_t mix64_ref(uint64_t z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

// ---------------------------------------------------------------------------
// One element of codec::quantize (codec.cpp:50-64), branch-free so two
// elements interleave.  nd = (double)norm, y = RN(1/norm), sd = s.
// Returns the (bits+1)-bit field level | sign << bits.
//   a  = RN(|v|/norm)   : q0 = |v|*y; r = fma(-nd, q0, |v|) (exact);
//                         a = fma(r, y, q0)  (correctly rounded, see header)
//   x  = RN(a*s); level = trunc(x) via RZ(x + 2^52); p = x - level (exact)
//   up = uniform01 < p  <=>  (k53 >> 1) < (k53 odd ? p*2^52 - 1/2 : p*2^52)
//        with k53 = h >> 11; both sides exact doubles
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t quantize_field(uint32_t u, double nd, double y, double sd,
                                                   uint32_t s, int bits, uint32_t h_lo,
                                                   uint32_t h_hi) {
  const double av = f32abs_to_f64(u & 0x7FFFFFFFu);
  const double q0 = __dmul_rn(av, y);
  const double r = __fma_rn(-nd, q0, av);
  const double a = __fma_rn(r, y, q0);
  const double x = __dmul_rn(a, sd);
  const double t = __dadd_rz(x, 4503599627370496.0);  // 2^52 + trunc(x)
  uint32_t level = uint32_t(__double2loint(t));
  const double lv = __dsub_rn(t, 4503599627370496.0);
  const double p = __dsub_rn(x, lv);
  const double Q = __dmul_rn(p, 4503599627370496.0);
  // kd = (h >> 12) as an exact double
  const uint32_t k_lo = __funnelshift_r(h_lo, h_hi, 12);
  const uint32_t k_hi = (h_hi >> 12) | 0x43300000u;
  const double kd = __dsub_rn(__hiloint2double(int(k_hi), int(k_lo)), 4503599627370496.0);
  const double thr = (h_lo & 0x800u) ? __dsub_rn(Q, 0.5) : Q;
  const uint32_t up = kd < thr ? 1u : 0u;
  level = level >= s ? s : level + up;
  return level | ((u >> 31) << bits);
}

// codec.cpp:84-93: level 0 -> +0.0f; else RN32(RN64(RN64(norm*l)/s)), signed.
// norm_d = (double)norm, ys = RN(1/s), sd = s.
__device__ __forceinline__ float dequant_field(double norm_d, uint32_t level, uint32_t sign,
                                               double sd, double ys) {
  const double nl = __dmul_rn(norm_d, u32_to_f64(level));  // exact: <= 32 significant bits
  const double q0 = __dmul_rn(nl, ys);
  const double r = __fma_rn(-sd, q0, nl);
  const double q = __fma_rn(r, ys, q0);
  const float mag = level == 0 ? 0.0f : f64pos_to_f32_rn(q);
  return (sign && level) ? -mag : mag;
}

// finalize's average (collectives.cpp:223-227): v / (float)N, exactly.
// N a power of two: multiplying by the exact reciprocal is the same real
// number, hence the same rounding; otherwise IEEE division.
__device__ __forceinline__ float apply_divisor(float v, float divisor, float recip, bool pow2) {
  if (divisor == 1.0f) return v;
  return pow2 ? __fmul_rn(v, recip) : __fdiv_rn(v, divisor);
}

}  // namespace gcx_dev
