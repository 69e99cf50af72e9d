// Bit-exact restatement of glibc 2.39 atan2 (x86_64 FMA ifunc variant).
//
// Why: the reference keys its angle sort with std::atan2
// (/root/reference/proj/include/hull2d/geom.hpp:42), i.e. glibc libm, which is
// NOT correctly rounded. Reproducing the reference's sort order bit for bit
// therefore needs glibc's exact arithmetic, not just "an accurate atan2".
//
// Third-party dependency (absent from /root/reference): glibc 2.39
// (Ubuntu GLIBC 2.39-0ubuntu8.5), sysdeps/ieee754/dbl-64/e_atan2.c with table
// uatan2.tbl. On x86_64 the library dispatches (ifunc) to a copy compiled with
// -mfma -mavx2 (`__atan2_fma`) on every CPU with FMA+AVX2; that copy's
// contraction pattern (which a*b+c became fused) is what is restated below,
// read from the shipped binary. Algorithm (finite inputs):
//   1. y = +-0, x = +-0 specials; |exp(y) - exp(x)| >= 57*2^20 shortcut to
//      +-pi/2, or ay/ax (x > 0) / +-pi (x < 0) on the other side.
//   2. Scale ax, ay by 2^+-500 when either leaves [2^-500, 2^500].
//   3. u = min/max with its exact remainder du (EMULV via fma).
//   4. Four octant cases (x>0 / x<0, ay<ax / ay>=ax); u < 1/16 uses an odd
//      degree-13 polynomial, otherwise the row i = round(256 u) - 16 of cij
//      (value, derivative, Taylor terms) around x_i, combined with the
//      pi/2 or pi double-double constants (hpi + hpi1, opi + opi1).
//   5. Result carries the sign of y.
// Non-finite inputs are outside the reference's contract and
// are not restated. The same source compiles for the host (C, built with
// -ffp-contract=off) and for sm_100a (every op an explicit _rn intrinsic, so
// nvcc cannot contract anything).
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define GA_FN static __device__ __forceinline__
#define GA_ADD(a, b) __dadd_rn((a), (b))
#define GA_SUB(a, b) __dsub_rn((a), (b))
#define GA_MUL(a, b) __dmul_rn((a), (b))
#define GA_DIV(a, b) __ddiv_rn((a), (b))
#define GA_FMA(a, b, c) __fma_rn((a), (b), (c))
#define GA_BITS(d) ((uint64_t)__double_as_longlong(d))
#define GA_DBL(u) __longlong_as_double((long long)(u))
#ifndef GSCAN_ATAN2_TABLE_QUAL
#define GSCAN_ATAN2_TABLE_QUAL static __device__ const
#endif
#else
#include <math.h>
#include <string.h>
#define GA_FN static inline
#define GA_ADD(a, b) ((a) + (b))
#define GA_SUB(a, b) ((a) - (b))
#define GA_MUL(a, b) ((a) * (b))
#define GA_DIV(a, b) ((a) / (b))
#define GA_FMA(a, b, c) fma((a), (b), (c))
static inline uint64_t ga_bits_(double d) { uint64_t u; memcpy(&u, &d, 8); return u; }
static inline double ga_dbl_(uint64_t u) { double d; memcpy(&d, &u, 8); return d; }
#define GA_BITS(d) ga_bits_(d)
#define GA_DBL(u) ga_dbl_(u)
#endif

#include "atan2_table.h"

// Constants of e_atan2.c / atnat2.h, as bit patterns.
#define GA_HPI 0x3ff921fb54442d18ull   // pi/2 (high part)
#define GA_MHPI 0xbff921fb54442d18ull  // -pi/2
#define GA_HPI1 0x3c91a62633145c07ull  // pi/2 - hpi (low part)
#define GA_OPI 0x400921fb54442d18ull   // pi
#define GA_MOPI 0xc00921fb54442d18ull  // -pi
#define GA_OPI1 0x3ca1a62633145c07ull  // pi - opi
#define GA_INV16 0x3fb0000000000000ull // 1/16
#define GA_D13 0x3fb375f08b31cbceull
#define GA_D11 0xbfb7458022b13c25ull
#define GA_D9 0x3fbc71c6e5129a3bull
#define GA_D7 0xbfc24924923f7603ull
#define GA_D5 0x3fc99999999997fdull
#define GA_D3 0xbfd5555555555555ull
#define GA_TWO52 0x4330000000000000ull
#define GA_TWO8 0x4070000000000000ull
#define GA_TWOM500 0x20b0000000000000ull
#define GA_TWO500 0x5f30000000000000ull

GA_FN double ga_copysign(double z, double y) {
  return GA_DBL((GA_BITS(z) & 0x7fffffffffffffffull) | (GA_BITS(y) & 0x8000000000000000ull));
}

GA_FN double ga_fabs(double z) { return GA_DBL(GA_BITS(z) & 0x7fffffffffffffffull); }

GA_FN double ga_cij(int row, int col) { return GA_DBL(gscan_atan2_cij_bits[row * 7 + col]); }

// Odd polynomial tail d3 + v(d5 + v(d7 + v(d9 + v(d11 + v d13)))) as the FMA
// build evaluates it (a Horner chain of fused multiply-adds).
GA_FN double ga_poly_d(double v) {
  double p = GA_DBL(GA_D13);
  p = GA_FMA(v, p, GA_DBL(GA_D11));
  p = GA_FMA(v, p, GA_DBL(GA_D9));
  p = GA_FMA(v, p, GA_DBL(GA_D7));
  p = GA_FMA(v, p, GA_DBL(GA_D5));
  p = GA_FMA(v, p, GA_DBL(GA_D3));
  return p;
}

// Row index i - 16 with i = (TWO52 + TWO8 * u) - TWO52 (the multiply-add is
// fused in the FMA build), truncated to int.
GA_FN int ga_row(double u) {
  double t = GA_FMA(u, GA_DBL(GA_TWO8), GA_DBL(GA_TWO52));
  t = GA_SUB(t, GA_DBL(GA_TWO52));
  return (int)t - 16;
}

// c2 + v(c3 + v(c4 + v(c5 + v c6))) Horner chain over one cij row.
GA_FN double ga_poly_row(int r, double v) {
  double p = ga_cij(r, 6);
  p = GA_FMA(v, p, ga_cij(r, 5));
  p = GA_FMA(v, p, ga_cij(r, 4));
  p = GA_FMA(v, p, ga_cij(r, 3));
  p = GA_FMA(v, p, ga_cij(r, 2));
  return p;
}

// atan2(y, x) for finite y, x, bit-identical to glibc 2.39 __atan2_fma.
GA_FN double glibc_atan2(double y, double x) {
  const uint64_t bx = GA_BITS(x), by = GA_BITS(y);
  const uint32_t ux = (uint32_t)(bx >> 32), uy = (uint32_t)(by >> 32);
  const uint32_t dx = (uint32_t)bx, dy = (uint32_t)by;

  // y = +-0
  if (uy == 0x00000000u && dy == 0u) return (ux & 0x80000000u) ? GA_DBL(GA_OPI) : 0.0;
  if (uy == 0x80000000u && dy == 0u) return (ux & 0x80000000u) ? GA_DBL(GA_MOPI) : -0.0;
  // x = +-0
  if (x == 0.0) return (uy & 0x80000000u) ? GA_DBL(GA_MHPI) : GA_DBL(GA_HPI);
  (void)dx;

  const double ax = ga_fabs(x);
  double ay = ga_fabs(y);
  const int de = (int)(uy & 0x7ff00000u) - (int)(ux & 0x7ff00000u);
  if (de >= 59768832) return (y > 0.0) ? GA_DBL(GA_HPI) : GA_DBL(GA_MHPI);
  if (de <= -59768832) {
    if (x > 0.0) return ga_copysign(GA_DIV(ay, ax), y);
    return (y > 0.0) ? GA_DBL(GA_OPI) : GA_DBL(GA_MOPI);
  }

  double sx = ax, sy = ay;
  if (sx < GA_DBL(GA_TWOM500) || sy < GA_DBL(GA_TWOM500)) {
    sx = GA_MUL(sx, GA_DBL(GA_TWO500));
    sy = GA_MUL(sy, GA_DBL(GA_TWO500));
  }
  if (sx > GA_DBL(GA_TWO500) || sy > GA_DBL(GA_TWO500)) {
    sx = GA_MUL(sx, GA_DBL(GA_TWOM500));
    sy = GA_MUL(sy, GA_DBL(GA_TWOM500));
  }

  double u, du;
  if (sy < sx) {
    u = GA_DIV(sy, sx);
    const double v = GA_MUL(u, sx);
    const double vv = GA_FMA(u, sx, -v);
    du = GA_DIV(GA_SUB(GA_SUB(sy, v), vv), sx);
  } else {
    u = GA_DIV(sx, sy);
    const double v = GA_MUL(u, sy);
    const double vv = GA_FMA(u, sy, -v);
    du = GA_DIV(GA_SUB(GA_SUB(sx, v), vv), sy);
  }

  const double inv16 = GA_DBL(GA_INV16);
  double z;
  if (x > 0.0) {
    if (sy < sx) {
      // (i) atan(ay/ax)
      if (u < inv16) {
        const double v = GA_MUL(u, u);
        const double zz = GA_FMA(GA_MUL(u, v), ga_poly_d(v), du);
        z = GA_ADD(u, zz);
      } else {
        const int r = ga_row(u);
        const double t3 = GA_SUB(u, ga_cij(r, 0));
        // EADD(t3, du, v, dv)
        const double v = GA_ADD(du, t3);
        const double dv = (ga_fabs(t3) > ga_fabs(du)) ? GA_ADD(GA_SUB(t3, v), du)
                                                      : GA_ADD(GA_SUB(du, v), t3);
        const double t2 = ga_cij(r, 2);
        double p = ga_cij(r, 6);
        p = GA_FMA(v, p, ga_cij(r, 5));
        p = GA_FMA(v, p, ga_cij(r, 4));
        p = GA_FMA(v, p, ga_cij(r, 3));
        p = GA_MUL(GA_MUL(v, v), p);
        p = GA_FMA(dv, t2, p);
        const double zz = GA_FMA(v, t2, p);
        z = GA_ADD(zz, ga_cij(r, 1));
      }
    } else {
      // (ii) pi/2 - atan(ax/ay)
      if (u < inv16) {
        const double v = GA_MUL(u, u);
        const double zz = GA_MUL(GA_MUL(u, v), ga_poly_d(v));
        const double hpi = GA_DBL(GA_HPI);
        const double t2 = GA_SUB(hpi, u);
        // ESUB(hpi, u, t2, cor); |hpi| > |u| always here
        const double cor = GA_SUB(GA_SUB(hpi, t2), u);
        double t3 = GA_ADD(cor, GA_DBL(GA_HPI1));
        t3 = GA_SUB(t3, du);
        t3 = GA_SUB(t3, zz);
        z = GA_ADD(t3, t2);
      } else {
        const int r = ga_row(u);
        const double v = GA_ADD(GA_SUB(u, ga_cij(r, 0)), du);
        const double zz = GA_FMA(-v, ga_poly_row(r, v), GA_DBL(GA_HPI1));
        const double t1 = GA_SUB(GA_DBL(GA_HPI), ga_cij(r, 1));
        z = GA_ADD(t1, zz);
      }
    }
  } else {
    if (sx < sy) {
      // (iii) pi/2 + atan(ax/ay)
      if (u < inv16) {
        const double v = GA_MUL(u, u);
        const double zz = GA_MUL(GA_MUL(u, v), ga_poly_d(v));
        const double hpi = GA_DBL(GA_HPI);
        const double t2 = GA_ADD(u, hpi);
        // EADD(hpi, u, t2, cor); |hpi| > |u| always here
        const double cor = GA_ADD(GA_SUB(hpi, t2), u);
        double t3 = GA_ADD(cor, GA_DBL(GA_HPI1));
        t3 = GA_ADD(t3, du);
        t3 = GA_ADD(t3, zz);
        z = GA_ADD(t3, t2);
      } else {
        const int r = ga_row(u);
        const double t1 = GA_ADD(GA_DBL(GA_HPI), ga_cij(r, 1));
        const double v = GA_ADD(GA_SUB(u, ga_cij(r, 0)), du);
        const double zz = GA_FMA(v, ga_poly_row(r, v), GA_DBL(GA_HPI1));
        z = GA_ADD(t1, zz);
      }
    } else {
      // (iv) pi - atan(ay/ax)
      if (u < inv16) {
        const double v = GA_MUL(u, u);
        const double zz = GA_MUL(GA_MUL(u, v), ga_poly_d(v));
        const double opi = GA_DBL(GA_OPI);
        const double t2 = GA_SUB(opi, u);
        const double cor = GA_SUB(GA_SUB(opi, t2), u);
        double t3 = GA_ADD(cor, GA_DBL(GA_OPI1));
        t3 = GA_SUB(t3, du);
        t3 = GA_SUB(t3, zz);
        z = GA_ADD(t3, t2);
      } else {
        const int r = ga_row(u);
        const double v = GA_ADD(GA_SUB(u, ga_cij(r, 0)), du);
        const double zz = GA_FMA(-v, ga_poly_row(r, v), GA_DBL(GA_OPI1));
        const double t1 = GA_SUB(GA_DBL(GA_OPI), ga_cij(r, 1));
        z = GA_ADD(t1, zz);
      }
    }
  }
  return ga_copysign(z, y);
}
