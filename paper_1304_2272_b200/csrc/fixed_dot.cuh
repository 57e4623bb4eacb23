// Integer-only arithmetic shared by the int8 TRSM epilogue and the standalone reductions.
//
// Why integers: on sm_100a the FP64 pipe is throttled while the SM's tensor core runs
// tcgen05.mma (tools/epi_contention.cu: a dependent DFMA chain goes from 23 to 158 cycles per
// step, independent DFMAs from 2 to 16 cycles per warp instruction; inside the TRSM kernel ncu
// shows DFMA stalled on "math" at ~1/100 of the idle rate).  The FP32/INT32 pipes are not
// affected, so the epilogue that runs next to the MMAs issues no FP64 instruction at all:
//   * Xbar from the exact int32 slice products: one 128-bit integer, rounded once to double;
//   * the canonical per-block dot (below): exact 128-bit fixed-point sum, rounded once.
// (The code also avoids bit tests the compiler would turn into FP64 compares.)
//
// Canonical block dot of u, v over one GG_DOT_BLOCK-row block (every reduction of the GLS sweep
// -- S_BL, S_BR, b_B of each SNP and gram(XLbar), b_T of the prepare -- is a sum of these, so a
// SNP column equal to a covariate column gives bitwise-equal entries and an exactly singular S):
//   E_u = max_i fx_exp(u_i)  (|u_i| < 2^E_u; zeros and subnormals count as 2^-1021);
//   U_i = trunc(u_i * 2^(58 - E_u))  (|U_i| < 2^58, truncation toward zero), same for v;
//   dot = RN( (sum_i U_i V_i) * 2^(E_u + E_v - 116) )  with the sum exact.
// The sum is exact, so the value is independent of summation order and symmetric in u, v.
// It is formed from 29-bit halves U = Uh 2^29 + Ul with four 32 x 32 -> 64-bit multiply-adds
// per term (IMAD.WIDE), each partial sum of <= 32 terms staying below 2^63.
#pragma once

#include <stdint.h>

namespace gg {

constexpr unsigned long long FX_FRAC = (1ull << 52) - 1;

// smallest k with |x| < 2^k for normal x; -1021 for zeros and subnormals
__device__ __forceinline__ int fx_exp(double x) {
  const int be = (__double2hiint(x) >> 20) & 0x7ff;
  return be == 0 ? -1021 : be - 1022;
}

// trunc(x * 2^(58 - E)) for a block exponent E >= fx_exp(x)
__device__ __forceinline__ long long fx_scale(double x, int E) {
  const unsigned hi = (unsigned)__double2hiint(x), lo = (unsigned)__double2loint(x);
  const int be = (int)((hi >> 20) & 0x7ffu);
  const unsigned long long frac = ((unsigned long long)(hi & 0xfffffu) << 32) | lo;
  const unsigned long long m = be == 0 ? frac : (frac | (1ull << 52));
  const int sh = (be == 0 ? -1021 : be - 1022) + 5 - E;   // |x| = m * 2^(k - 53); U = m * 2^sh
  const unsigned long long u = sh >= 0 ? (m << sh) : (sh > -64 ? (m >> -sh) : 0ull);
  return (hi >> 31) ? -(long long)u : (long long)u;
}

// a fixed-point value split into 29-bit halves: U = h * 2^29 + l, |h| < 2^29, 0 <= l < 2^29
struct Fx2 {
  int h, l;
};
__device__ __forceinline__ Fx2 fx_split(long long U) {
  return Fx2{(int)(U >> 29), (int)(U & ((1ll << 29) - 1))};
}

// exact block-dot accumulator: sum Uh Vh, sum Uh Vl, sum Ul Vh, sum Ul Vl
struct FxAcc {
  long long hh, hl, lh, ll;
};
__device__ __forceinline__ void fx_mac(FxAcc& a, Fx2 u, Fx2 v) {
  a.hh += (long long)u.h * v.h;   // IMAD.WIDE
  a.hl += (long long)u.h * v.l;
  a.lh += (long long)u.l * v.h;
  a.ll += (long long)u.l * v.l;
}

// rare out-of-range tail of fx_to_double (subnormal or overflowing results), kept out of line
static __device__ __noinline__ double fx_to_double_tail(bool neg, unsigned long long top, bool sticky,
                                                 int be) {
  // top: the value's 64 leading bits (msb at bit 63) below which `sticky` bits are non-zero;
  // value = top * 2^(be - 1023 - 63)
  unsigned long long bits;
  if (be >= 2047) {
    bits = 0x7ffull << 52;   // overflow -> inf
  } else {
    const int sh = 12 - be;   // >= 12: keep 52 - (1 - be) fraction bits
    if (sh >= 64) {
      bits = (sh == 64 && (top > (1ull << 63) || (top == (1ull << 63) && sticky))) ? 1ull : 0ull;
    } else {
      const unsigned long long q = top >> sh, rem = top & ((1ull << sh) - 1),
                               half = 1ull << (sh - 1);
      bits = q + ((rem > half || (rem == half && (sticky || (q & 1ull)))) ? 1ull : 0ull);
    }
  }
  return __longlong_as_double((long long)(bits | ((unsigned long long)neg << 63)));
}

// RN((hi:lo) * 2^e2) for a signed 128-bit integer, with integer instructions only
__device__ __forceinline__ double fx_to_double(unsigned long long lo, long long hi, int e2) {
  const bool neg = hi < 0;
  unsigned long long mh = (unsigned long long)hi, ml = lo;
  if (neg) {   // two's-complement negation
    ml = ~ml + 1ull;
    mh = ~mh + (ml == 0 ? 1ull : 0ull);
  }
  if ((mh | ml) == 0) return 0.0;
  // normalise: top = the 64 leading bits, sticky = any bit below them
  const int lz = mh != 0 ? __clzll((long long)mh) : 64 + __clzll((long long)ml);
  unsigned long long top;
  bool sticky;
  if (lz >= 64) {
    top = ml << (lz - 64);
    sticky = false;
  } else if (lz == 0) {
    top = mh;
    sticky = ml != 0;
  } else {
    top = (mh << lz) | (ml >> (64 - lz));
    sticky = (ml << lz) != 0;
  }
  const int be = (127 - lz) + e2 + 1023;   // biased exponent of the leading bit
  if (be <= 0 || be >= 2047) return fx_to_double_tail(neg, top, sticky, be);
  unsigned long long mant = top >> 11;      // 53 bits
  const bool rbit = (top >> 10) & 1ull;
  const bool rest = sticky || (top & 0x3ffull) != 0;
  unsigned long long bits = ((unsigned long long)be << 52) + (mant & FX_FRAC);
  if (rbit && (rest || (mant & 1ull))) bits += 1ull;   // a carry into the exponent is correct
  return __longlong_as_double((long long)(bits | ((unsigned long long)neg << 63)));
}

// RN(dot): T = hh 2^58 + (hl + lh) 2^29 + ll, assembled exactly in 128 bits
__device__ __forceinline__ double fx_finish(const FxAcc& a, int Eu, int Ev) {
  const long long mid = a.hl + a.lh;   // |mid| < 2^64 can overflow: keep its carry separately
  const long long mid_hi = ((a.hl >> 63) + (a.lh >> 63)) +
                           (long long)((unsigned long long)mid < (unsigned long long)a.hl);
  // 128-bit: hh << 58
  unsigned long long lo = (unsigned long long)a.hh << 58;
  long long hi = a.hh >> 6;
  // + (mid_hi:mid) << 29
  const unsigned long long m_lo = (unsigned long long)mid << 29;
  const long long m_hi =
      (long long)(((unsigned long long)mid_hi << 29) | ((unsigned long long)mid >> 35));
  unsigned long long t = lo + m_lo;
  hi += m_hi + (long long)(t < lo);
  lo = t;
  // + ll (sign-extended)
  t = lo + (unsigned long long)a.ll;
  hi += (a.ll >> 63) + (long long)(t < lo);
  lo = t;
  return fx_to_double(lo, hi, Eu + Ev - 116);
}

}  // namespace gg
