// glibc_sincos.cuh — device restatement of glibc 2.39's sincos as the
// reference executes it (x86-64 ifunc __sincos_fma: the IBM accurate
// mathematical library, sysdeps/ieee754/dbl-64/s_sincos.c + s_sin.c,
// compiled with -mfma so every `a*b + c` of the source is one FMA).  The
// reference's world_polygon / contour_radius (world.cpp:57-62,
// actions.cpp:15) call sincos through Vec2::rotated, so polygon poses are
// bit-identical only if the device reproduces this routine bit for bit,
// including its table (__sincostab, emitted from the system libm by
// tools/gen_sincostab.py — its low words are not recomputable).  The FMA
// placement below was read off the disassembly of the installed libm and is
// verified against the host sincos on random and edge-case arguments
// (tests/test_gpu_parity.py::test_device_sincos_matches_glibc).  Arguments
// here are |x| < 105414350 (object angles are wrapped to [-pi, pi)); larger
// ones would need __branred and are not supported.
#pragma once

#include <cstdint>

namespace ppg {

__device__ const uint64_t kSinCosTab[440] = {
#include "glibc_sincostab.inc"
};

namespace gsc {

PPG_DI double bits(uint64_t u) { return __longlong_as_double(static_cast<long long>(u)); }
PPG_DI double tab(int k) { return __longlong_as_double(static_cast<long long>(__ldg(kSinCosTab + k))); }

// usncs.h constants (values read from the binary)
#define PPG_GSC(name, hex) PPG_DI double name() { return bits(hex##ull); }
PPG_GSC(sn3, 0xbfc5555555555515)
PPG_GSC(sn5, 0x3f811110e829872f)
PPG_GSC(cs2, 0x3fe0000000000000)
PPG_GSC(cs4, 0xbfa5555555555535)
PPG_GSC(cs6, 0x3f56c16bedd9e239)
PPG_GSC(s1, 0xbfc5555555555555)
PPG_GSC(s2, 0x3f81111111110ece)
PPG_GSC(s3, 0xbf2a01a019db08b8)
PPG_GSC(s4, 0x3ec71de27b9a7ed9)
PPG_GSC(s5, 0xbe5addffc2fcdf59)
PPG_GSC(big, 0x42c8000000000000)
PPG_GSC(hp0, 0x3ff921fb54442d18)
PPG_GSC(hp1, 0x3c91a62633145c07)
PPG_GSC(toint, 0x4338000000000000)
PPG_GSC(hpinv, 0x3fe45f306dc9c883)
PPG_GSC(mp1, 0x3ff921fb58000000)
PPG_GSC(mp2, 0xbe4dde973c000000)
PPG_GSC(pp3, 0xbc8cb3b398000000)
PPG_GSC(pp4, 0xbacd747f23e32ed7)
PPG_GSC(taylor_lim, 0x3fc020c49ba5e354)  // 0.126
#undef PPG_GSC

// TAYLOR_SIN(x*x, x, dx): x + ((P(xx)*x - 0.5*dx)*xx + dx)
PPG_DI double taylor_sin(double x, double dx) {
  const double xx = x * x;
  double p = __fma_rn(xx, s5(), s4());
  p = __fma_rn(xx, p, s3());
  p = __fma_rn(xx, p, s2());
  p = __fma_rn(xx, p, s1());
  const double t = __fma_rn(xx, __fma_rn(p, x, -(0.5 * dx)), dx);
  return x + t;
}

// do_sin (s_sin.c)
PPG_DI double do_sin(double x, double dx) {
  const double xold = x;
  if (fabs(x) < taylor_lim()) return taylor_sin(x, dx);
  if (x <= 0) dx = -dx;
  const double u = big() + fabs(x);
  const int k = __double2loint(u) << 2;
  x = fabs(x) - (u - big());
  const double xx = x * x;
  const double s = x + __fma_rn(x * xx, __fma_rn(xx, sn5(), sn3()), dx);
  const double c = __fma_rn(x, dx, xx * __fma_rn(__fma_rn(xx, cs6(), cs4()), xx, cs2()));
  const double sn = tab(k), ssn = tab(k + 1), cs = tab(k + 2), ccs = tab(k + 3);
  const double cor = __fma_rn(s, cs, __fma_rn(-c, sn, __fma_rn(s, ccs, ssn)));
  return copysign(sn + cor, xold);
}

// do_cos (s_sin.c)
PPG_DI double do_cos(double x, double dx) {
  if (x < 0) dx = -dx;
  const double u = big() + fabs(x);
  const int k = __double2loint(u) << 2;
  x = fabs(x) - (u - big()) + dx;
  const double xx = x * x;
  const double s = __fma_rn(x * xx, __fma_rn(xx, sn5(), sn3()), x);
  const double c = xx * __fma_rn(__fma_rn(xx, cs6(), cs4()), xx, cs2());
  const double sn = tab(k), ssn = tab(k + 1), cs = tab(k + 2), ccs = tab(k + 3);
  const double cor = __fma_rn(-sn, s, __fma_rn(-cs, c, __fma_rn(-s, ssn, ccs)));
  return cs + cor;
}

// reduce_sincos (s_sin.c): x = n*pi/2 + (a + da)
PPG_DI int reduce(double x, double& a, double& da) {
  const double t = __fma_rn(x, hpinv(), toint());
  const double xn = t - toint();
  const int n = __double2loint(t) & 3;
  const double y = __fma_rn(-xn, mp2(), __fma_rn(-xn, mp1(), x));
  const double t2 = __fma_rn(-xn, pp3(), y);
  double db = __fma_rn(-xn, pp3(), y - t2);
  const double b = __fma_rn(-xn, pp4(), t2);
  db = db + __fma_rn(-xn, pp4(), t2 - b);
  a = b;
  da = db;
  return n;
}


}  // namespace gsc

// sincos (s_sincos.c) for |x| < 105414350.  Every branch of the library
// ends in do_sin and do_cos of one reduced argument (a, da); they are
// evaluated once here and the quadrant picks and signs them, so the body
// holds one copy of each (code size: this is inlined into every polygon
// kernel).
PPG_DI void glibc_sincos(double x, double* sinx, double* cosx) {
  const int k = __double2hiint(x) & 0x7fffffff;
  if (k < 0x3e400000) {  // |x| < 2^-27
    *sinx = x;
    *cosx = 1.0;
    return;
  }
  double a, da;
  int n;
  bool mid = false;
  if (k < 0x3feb6000) {  // |x| < 0.855469: sin = do_sin(x, 0), cos = do_cos(x, 0)
    a = x;
    da = 0.0;
    n = 0;
  } else if (k < 0x400368fd) {  // |x| < 2.426265: sin = copysign(do_cos(a, da), x), cos = do_sin(a, da)
    const double y = gsc::hp0() - fabs(x);
    a = y + gsc::hp1();
    da = (y - a) + gsc::hp1();
    n = 1;
    mid = true;
  } else {  // quadrant n: sin = +-(n odd ? do_cos : do_sin), cos = the other, sign of quadrant n + 1
    n = gsc::reduce(x, a, da);
  }
  const double s = gsc::do_sin(a, da), c = gsc::do_cos(a, da);
  const double rs = (n & 1) ? c : s, rc = (n & 1) ? s : c;
  if (mid) {
    *sinx = copysign(rs, x);
    *cosx = rc;
    return;
  }
  *sinx = (n & 2) ? -rs : rs;
  *cosx = ((n + 1) & 2) ? -rc : rc;
}

}  // namespace ppg
