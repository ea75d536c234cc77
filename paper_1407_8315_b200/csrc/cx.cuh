// cx.cuh -- complex128 arithmetic with the reference's exact rounding rules.
//
// The reference computes in two arithmetic dialects and the parity contract
// (supports bit-identical, values within 1e-9) is easiest to keep when every
// operation rounds the way the reference's does:
//
//  * "gcc" ops: the compiled kernels (_kernels/_core.pyx, built by gcc -O3
//    without -march, pkg/setup.py:14-30) use C99 double _Complex:
//      a*b  = (ar*br - ai*bi, ar*bi + ai*br), every product rounded (no FMA);
//      a/b  = libgcc __divdc3 (Smith's method with range scaling);
//      csqrt / cpow / cexp / cabs from glibc.
//  * "numpy" ops: the Python drivers (exact.py, general.py) use numpy ufuncs:
//      a*b  = (fma(ar, br, -(ai*bi)), fma(ar, bi, ai*br))   [SIMD loops]
//      a/b  = Smith's method with a reciprocal scale (umath loops).
//
// Every function here is __host__ __device__: the same source is compiled
// for sm_100a (the product) and for the host by tests/test_math.py, which
// checks it bit-for-bit against gcc/glibc.  On the device the transcendental
// calls (hypot, atan2, log, exp, sincos) are CUDA libm and may differ from
// glibc by an ulp; everything else is exactly rounded identically.
#pragma once

#include <math.h>
#include <stdint.h>
#include <float.h>

#if defined(__CUDACC__)
#define SFDT_HD __host__ __device__ __forceinline__
#else
#define SFDT_HD static inline
#endif
// The long scalar routines (complex division, csqrt, clog/cexp, hypot) as real
// calls instead of inline copies: a translation unit built with
// SFDT_NOINLINE_HEAVY keeps one copy of each, so a decode trial's straight-line
// code shrinks severalfold and stays in the instruction cache.  Same
// instructions, same results.
#if defined(__CUDACC__) && defined(SFDT_NOINLINE_HEAVY)
#define SFDT_HEAVY __host__ __device__ __noinline__
#else
#define SFDT_HEAVY SFDT_HD
#endif

#if defined(__CUDA_ARCH__)
#define DMUL(a, b) __dmul_rn((a), (b))
#define DADD(a, b) __dadd_rn((a), (b))
#define DSUB(a, b) __dsub_rn((a), (b))
#define DDIV(a, b) __ddiv_rn((a), (b))
#define DFMA(a, b, c) __fma_rn((a), (b), (c))
#else
#define DMUL(a, b) ((a) * (b))
#define DADD(a, b) ((a) + (b))
#define DSUB(a, b) ((a) - (b))
#define DDIV(a, b) ((a) / (b))
#define DFMA(a, b, c) fma((a), (b), (c))
#endif

namespace sfdt {

struct cx {
    double re, im;
};

SFDT_HD cx mk(double re, double im) { cx z; z.re = re; z.im = im; return z; }
SFDT_HD cx cadd(cx a, cx b) { return mk(DADD(a.re, b.re), DADD(a.im, b.im)); }
SFDT_HD cx csub(cx a, cx b) { return mk(DSUB(a.re, b.re), DSUB(a.im, b.im)); }
SFDT_HD cx cneg(cx a) { return mk(-a.re, -a.im); }
SFDT_HD cx cconj(cx a) { return mk(a.re, -a.im); }
SFDT_HD bool cis_zero(cx a) { return a.re == 0.0 && a.im == 0.0; }
// real scalar times complex (gcc lowers (s + 0i) * z to componentwise)
SFDT_HD cx cscale(double s, cx a) { return mk(DMUL(s, a.re), DMUL(s, a.im)); }
// complex divided by a real (gcc lowers z / (s + 0i) to componentwise)
SFDT_HD cx cdivr(cx a, double s) { return mk(DDIV(a.re, s), DDIV(a.im, s)); }

// gcc C99 complex multiply, no contraction
SFDT_HD cx gmul(cx a, cx b)
{
    return mk(DSUB(DMUL(a.re, b.re), DMUL(a.im, b.im)), DADD(DMUL(a.re, b.im), DMUL(a.im, b.re)));
}

// numpy complex multiply (SIMD loop with fused multiply-add)
SFDT_HD cx nmul(cx a, cx b)
{
    return mk(DFMA(a.re, b.re, -DMUL(a.im, b.im)), DFMA(a.re, b.im, DMUL(a.im, b.re)));
}

// libgcc __divdc3 (GCC >= 12): Smith's algorithm with range scaling.
SFDT_HEAVY cx gdiv(cx num, cx den)
{
    double a = num.re, b = num.im, c = den.re, d = den.im;
    const double RBIG = DBL_MAX / 2, RMIN = DBL_MIN, RMIN2 = DBL_EPSILON;
    const double RMINSCAL = 1.0 / DBL_EPSILON, RMAX2 = RBIG * RMIN2;
    double ratio, denom, x, y;
    if (fabs(c) < fabs(d)) {
        if (fabs(d) >= RBIG) { a = a / 2; b = b / 2; c = c / 2; d = d / 2; }
        if (fabs(d) < RMIN2) {
            a = DMUL(a, RMINSCAL); b = DMUL(b, RMINSCAL); c = DMUL(c, RMINSCAL); d = DMUL(d, RMINSCAL);
        } else if (((fabs(a) < RMIN) && (fabs(b) < RMAX2) && (fabs(d) < RMAX2))
                   || ((fabs(b) < RMIN) && (fabs(a) < RMAX2) && (fabs(d) < RMAX2))) {
            a = DMUL(a, RMINSCAL); b = DMUL(b, RMINSCAL); c = DMUL(c, RMINSCAL); d = DMUL(d, RMINSCAL);
        }
        ratio = DDIV(c, d);
        denom = DADD(DMUL(c, ratio), d);
        if (fabs(ratio) > RMIN) {
            x = DDIV(DADD(DMUL(a, ratio), b), denom);
            y = DDIV(DSUB(DMUL(b, ratio), a), denom);
        } else {
            x = DDIV(DADD(DMUL(c, DDIV(a, d)), b), denom);
            y = DDIV(DSUB(DMUL(c, DDIV(b, d)), a), denom);
        }
    } else {
        if (fabs(c) >= RBIG) { a = a / 2; b = b / 2; c = c / 2; d = d / 2; }
        if (fabs(c) < RMIN2) {
            a = DMUL(a, RMINSCAL); b = DMUL(b, RMINSCAL); c = DMUL(c, RMINSCAL); d = DMUL(d, RMINSCAL);
        } else if (((fabs(a) < RMIN) && (fabs(b) < RMAX2) && (fabs(c) < RMAX2))
                   || ((fabs(b) < RMIN) && (fabs(a) < RMAX2) && (fabs(c) < RMAX2))) {
            a = DMUL(a, RMINSCAL); b = DMUL(b, RMINSCAL); c = DMUL(c, RMINSCAL); d = DMUL(d, RMINSCAL);
        }
        ratio = DDIV(d, c);
        denom = DADD(DMUL(d, ratio), c);
        if (fabs(ratio) > RMIN) {
            x = DDIV(DADD(DMUL(b, ratio), a), denom);
            y = DDIV(DSUB(b, DMUL(a, ratio)), denom);
        } else {
            x = DDIV(DADD(a, DMUL(d, DDIV(b, c))), denom);
            y = DDIV(DSUB(b, DMUL(d, DDIV(a, c))), denom);
        }
    }
    // C99 Annex G recovery of infinities/zeros that computed as NaN+iNaN
    if (isnan(x) && isnan(y)) {
        if (c == 0.0 && d == 0.0 && (!isnan(a) || !isnan(b))) {
            x = copysign(INFINITY, c) * a;
            y = copysign(INFINITY, c) * b;
        } else if ((isinf(a) || isinf(b)) && isfinite(c) && isfinite(d)) {
            a = copysign(isinf(a) ? 1.0 : 0.0, a);
            b = copysign(isinf(b) ? 1.0 : 0.0, b);
            x = INFINITY * (a * c + b * d);
            y = INFINITY * (b * c - a * d);
        } else if ((isinf(c) || isinf(d)) && isfinite(a) && isfinite(b)) {
            c = copysign(isinf(c) ? 1.0 : 0.0, c);
            d = copysign(isinf(d) ? 1.0 : 0.0, d);
            x = 0.0 * (a * c + b * d);
            y = 0.0 * (b * c - a * d);
        }
    }
    return mk(x, y);
}

// numpy complex division (umath: Smith with reciprocal scale)
SFDT_HD cx ndiv(cx a, cx b)
{
    const double br = b.re, bi = b.im;
    const double abr = fabs(br), abi = fabs(bi);
    if (abr >= abi) {
        if (abr == 0.0 && abi == 0.0)
            return mk(a.re / abr, a.im / abr);
        const double rat = DDIV(bi, br);
        const double scl = DDIV(1.0, DADD(br, DMUL(bi, rat)));
        return mk(DMUL(DADD(a.re, DMUL(a.im, rat)), scl), DMUL(DSUB(a.im, DMUL(a.re, rat)), scl));
    }
    const double rat = DDIV(br, bi);
    const double scl = DDIV(1.0, DADD(bi, DMUL(br, rat)));
    return mk(DMUL(DADD(DMUL(a.re, rat), a.im), scl), DMUL(DSUB(DMUL(a.im, rat), a.re), scl));
}

SFDT_HEAVY double cabs_(cx a) { return hypot(a.re, a.im); }
// always-inline form for the rare boundary tests inside streaming kernels
SFDT_HD double cabs_i(cx a) { return hypot(a.re, a.im); }

// glibc csqrt (finite inputs): principal branch, Re >= 0, using the identity
// 2 Re(r) Im(r) = Im(z) to avoid cancellation.
SFDT_HEAVY cx gsqrt(cx z)
{
    double re = z.re, im = z.im;
    if (!isfinite(re) || !isfinite(im)) {
        if (isinf(im)) return mk(INFINITY, im);
        if (isinf(re)) {
            if (re < 0) return mk(isnan(im) ? NAN : 0.0, copysign(INFINITY, im));
            return mk(re, isnan(im) ? NAN : copysign(0.0, im));
        }
        return mk(NAN, NAN);
    }
    if (im == 0.0) {
        if (re < 0.0) return mk(0.0, copysign(sqrt(-re), im));
        return mk(fabs(sqrt(re)), copysign(0.0, im));
    }
    if (re == 0.0) {
        double r;
        if (fabs(im) >= 2.0 * DBL_MIN)
            r = sqrt(DMUL(0.5, fabs(im)));
        else
            r = DMUL(0.5, sqrt(DMUL(2.0, fabs(im))));
        return mk(r, copysign(r, im));
    }
    int scale = 0;
    if (fabs(re) > DBL_MAX / 4.0) {
        scale = 1;
        re = scalbn(re, -2);
        im = scalbn(im, -2);
    } else if (fabs(im) > DBL_MAX / 4.0) {
        scale = 1;
        if (fabs(re) >= 4.0 * DBL_MIN) re = scalbn(re, -2);
        else re = 0.0;
        im = scalbn(im, -2);
    } else if (fabs(re) < 2.0 * DBL_MIN && fabs(im) < 2.0 * DBL_MIN) {
        scale = -((DBL_MANT_DIG + 1) / 2);
        re = scalbn(re, -2 * scale);
        im = scalbn(im, -2 * scale);
    }
    double d = hypot(re, im);
    double r, s;
    if (re > 0) {
        r = sqrt(DMUL(0.5, DADD(d, re)));
        if (scale == 1 && fabs(im) < 1.0) {
            s = DDIV(im, r);
            r = scalbn(r, scale);
            scale = 0;
        } else {
            s = DMUL(0.5, DDIV(im, r));
        }
    } else {
        s = sqrt(DMUL(0.5, DSUB(d, re)));
        if (scale == 1 && fabs(im) < 1.0) {
            r = fabs(DDIV(im, s));
            s = scalbn(s, scale);
            scale = 0;
        } else {
            r = fabs(DMUL(0.5, DDIV(im, s)));
        }
    }
    if (scale) {
        r = scalbn(r, scale);
        s = scalbn(s, scale);
    }
    return mk(r, copysign(s, im));
}

// glibc cexp for finite arguments: exp(re) * (cos im, sin im)
SFDT_HEAVY cx gexp(cx z)
{
    double s, c;
#if defined(__CUDA_ARCH__)
    sincos(z.im, &s, &c);
#else
    s = sin(z.im);
    c = cos(z.im);
#endif
    if (z.re == 0.0)
        return mk(c, s);
    const double e = exp(z.re);
    return mk(DMUL(e, c), DMUL(e, s));
}

// glibc __x2y2m1: x^2 + y^2 - 1 with exact products and sorted
// error-free summation (used by clog near the unit circle).
SFDT_HD void sort_abs5(double *v, int lo)
{
    for (int i = lo + 1; i < 5; i++) {
        double key = v[i];
        int j = i - 1;
        while (j >= lo && fabs(v[j]) > fabs(key)) {
            v[j + 1] = v[j];
            j--;
        }
        v[j + 1] = key;
    }
}

SFDT_HD double x2y2m1(double x, double y)
{
    double v[5];
    v[1] = DMUL(x, x);
    v[0] = DFMA(x, x, -v[1]);
    v[3] = DMUL(y, y);
    v[2] = DFMA(y, y, -v[3]);
    v[4] = -1.0;
    sort_abs5(v, 0);
    for (int i = 0; i <= 3; i++) {
        const double a = v[i + 1], b = v[i];
        const double hi = DADD(a, b);
        v[i] = DADD(DSUB(a, hi), b);
        v[i + 1] = hi;
        sort_abs5(v, i + 1);
    }
    return DADD(DADD(DADD(DADD(v[4], v[3]), v[2]), v[1]), v[0]);
}

// glibc clog for finite, nonzero arguments
SFDT_HEAVY cx gclog(cx z)
{
    double absx = fabs(z.re), absy = fabs(z.im);
    int scale = 0;
    if (absx < absy) { double t = absx; absx = absy; absy = t; }
    if (absx > DBL_MAX / 2) {
        scale = -1;
        absx = scalbn(absx, scale);
        absy = (absy >= DBL_MIN * 2 ? scalbn(absy, scale) : 0.0);
    } else if (absx < DBL_MIN && absy < DBL_MIN) {
        scale = DBL_MANT_DIG;
        absx = scalbn(absx, scale);
        absy = scalbn(absy, scale);
    }
    double re;
    if (absx == 1.0 && scale == 0) {
        re = log1p(DMUL(absy, absy)) / 2;
    } else if (absx > 1.0 && absx < 2.0 && absy < 1.0 && scale == 0) {
        double d2m1 = DMUL(DSUB(absx, 1.0), DADD(absx, 1.0));
        if (absy >= DBL_EPSILON) d2m1 = DADD(d2m1, DMUL(absy, absy));
        re = log1p(d2m1) / 2;
    } else if (absx < 1.0 && absx >= 0.5 && absy < DBL_EPSILON / 2 && scale == 0) {
        re = log1p(DMUL(DSUB(absx, 1.0), DADD(absx, 1.0))) / 2;
    } else if (absx < 1.0 && absx >= 0.5 && scale == 0
               && DADD(DMUL(absx, absx), DMUL(absy, absy)) >= 0.5) {
        re = log1p(x2y2m1(absx, absy)) / 2;
    } else {
        re = DSUB(log(hypot(absx, absy)), DMUL((double)scale, 0.69314718055994530942));
    }
    return mk(re, atan2(z.im, z.re));
}

// cpow(a3, 1/3) as glibc computes it: cexp((1/3 + 0i) * clog(a3))
SFDT_HD cx gcbrt(cx z)
{
    if (z.re == 0.0 && z.im == 0.0)
        return mk(0.0, 0.0);
    const double third = 1.0 / 3.0;
    const cx l = gclog(z);
    return gexp(mk(DMUL(third, l.re), DMUL(third, l.im)));
}

// -------------------------------------------------- cofactor determinants
// _core.pyx:84-120 (first-row cofactor expansion, gcc arithmetic)
SFDT_HD cx det2(cx a00, cx a01, cx a10, cx a11) { return csub(gmul(a00, a11), gmul(a01, a10)); }

SFDT_HD cx det3(const cx *a)
{
    return cadd(csub(gmul(a[0], det2(a[4], a[5], a[7], a[8])), gmul(a[1], det2(a[3], a[5], a[6], a[8]))),
                gmul(a[2], det2(a[3], a[4], a[6], a[7])));
}

SFDT_HD cx det4(const cx *a)
{
    cx minor[9];
    cx acc = mk(0.0, 0.0);
    double sign = 1.0;
#pragma unroll
    for (int col = 0; col < 4; col++) {
        int i = 0;
#pragma unroll
        for (int r = 1; r < 4; r++)
#pragma unroll
            for (int c = 0; c < 4; c++)
                if (c != col) minor[i++] = a[4 * r + c];
        acc = cadd(acc, gmul(cscale(sign, a[col]), det3(minor)));
        sign = -sign;
    }
    return acc;
}

SFDT_HD cx detn(const cx *a, int n)
{
    if (n == 1) return a[0];
    if (n == 2) return det2(a[0], a[1], a[2], a[3]);
    if (n == 3) return det3(a);
    return det4(a);
}

// Hankel Cramer solve (_core.pyx:127-162): m has >= 2a entries.
SFDT_HD cx hankel_solve1(const cx *m, int a, cx *c)
{
    cx hank[16], work[16];
    for (int i = 0; i < a; i++)
        for (int j = 0; j < a; j++)
            hank[a * i + j] = m[i + j];
    cx det = detn(hank, a);
    for (int j = 0; j < a; j++) c[j] = mk(0.0, 0.0);
    if (cis_zero(det)) return det;
    for (int col = 0; col < a; col++) {
        for (int i = 0; i < a; i++)
            for (int j = 0; j < a; j++)
                work[a * i + j] = (j == col) ? cneg(m[a + i]) : hank[a * i + j];
        c[col] = gdiv(detn(work, a), det);
    }
    return det;
}

// ------------------------------------------------------ closed-form roots
// _core.pyx:169-266
SFDT_HD void quad_pair(cx b, cx c, cx *z0, cx *z1)
{
    cx disc = gsqrt(csub(gmul(b, b), cscale(4.0, c)));
    if (DSUB(DMUL(b.re, disc.re), DMUL(-b.im, disc.im)) < 0.0)   // creal(conj(b) * disc)
        disc = cneg(disc);
    cx q = cscale(-0.5, cadd(b, disc));
    *z0 = q;
    *z1 = cis_zero(q) ? cscale(-0.5, csub(b, disc)) : gdiv(c, q);
}

SFDT_HD void cube_pair(cx g, cx h, cx *aa, cx *bb)
{
    cx r = gsqrt(cadd(gmul(g, g), gmul(gmul(h, h), h)));
    cx lo = csub(g, r), hi = cadd(g, r);
    cx a3 = (cabs_(lo) >= cabs_(hi)) ? lo : hi;
    cx a = gcbrt(a3);
    *aa = a;
    *bb = cis_zero(a) ? mk(0.0, 0.0) : gdiv(cneg(h), a);
}

SFDT_HD void roots3(cx c0, cx c1, cx c2, cx *z)
{
    const cx W1 = mk(-0.5, 0.8660254037844386), W2 = mk(-0.5, -0.8660254037844386);
    cx g = cadd(csub(cdivr(c0, 2.0), cdivr(gmul(c1, c2), 6.0)), cdivr(gmul(gmul(c2, c2), c2), 27.0));
    cx h = csub(cdivr(c1, 3.0), cdivr(gmul(c2, c2), 9.0));
    cx a, b;
    cube_pair(g, h, &a, &b);
    cx shift = cdivr(cneg(c2), 3.0);
    z[0] = csub(csub(shift, a), b);
    z[1] = csub(csub(shift, gmul(W1, a)), gmul(W2, b));
    z[2] = csub(csub(shift, gmul(W2, a)), gmul(W1, b));
}

SFDT_HD void roots4(cx c0, cx c1, cx c2, cx c3, cx *z)
{
    cx g = cdivr(csub(csub(csub(cadd(gmul(cscale(72.0, c0), c2), gmul(gmul(cscale(9.0, c1), c2), c3)),
                                gmul(cscale(27.0, c1), c1)),
                           gmul(gmul(cscale(27.0, c0), c3), c3)),
                      gmul(gmul(cscale(2.0, c2), c2), c2)),
                 432.0);
    cx h = cdivr(csub(csub(gmul(cscale(3.0, c1), c3), cscale(12.0, c0)), gmul(c2, c2)), 36.0);
    cx cc, dd;
    cube_pair(g, h, &cc, &dd);
    cx y = csub(csub(cdivr(c2, 6.0), cc), dd);
    cx aa = gsqrt(cadd(csub(cdivr(gmul(c3, c3), 4.0), c2), cscale(2.0, y)));
    cx num = csub(gmul(c3, y), c1);
    const double ac3 = cabs_(c3), ay = cabs_(y);
    const double scale_a = DADD(DADD(DADD(1.0, DDIV(DMUL(ac3, ac3), 4.0)), cabs_(c2)), DMUL(2.0, ay));
    const double scale_b = DADD(DADD(1.0, DMUL(ay, ay)), cabs_(c0));
    cx bb;
    if (cabs_(aa) > DMUL(1e-6, sqrt(scale_a))) {
        bb = gdiv(num, cscale(2.0, aa));
    } else {
        bb = gsqrt(csub(gmul(y, y), c0));
        if (cabs_(bb) > DMUL(1e-6, sqrt(scale_b))) {
            aa = gdiv(num, cscale(2.0, bb));
        } else {
            aa = mk(0.0, 0.0);
            bb = mk(0.0, 0.0);
        }
    }
    cx c3h = cdivr(c3, 2.0);
    quad_pair(cadd(c3h, aa), cadd(y, bb), &z[0], &z[1]);
    quad_pair(csub(c3h, aa), csub(y, bb), &z[2], &z[3]);
}

SFDT_HD void poly_roots1(const cx *c, int a, cx *z)
{
    if (a == 1) z[0] = cneg(c[0]);
    else if (a == 2) quad_pair(c[1], c[0], &z[0], &z[1]);
    else if (a == 3) roots3(c[0], c[1], c[2], z);
    else roots4(c[0], c[1], c[2], c[3], z);
}

// ---------------------------------------------------- Vandermonde solve
// _core.pyx:273-312
SFDT_HD cx vandermonde_solve1(const cx *z, const cx *m, int a, cx *p)
{
    cx vand[16], work[16];
    for (int j = 0; j < a; j++) {
        cx acc = mk(1.0, 0.0);
        for (int i = 0; i < a; i++) {
            vand[a * i + j] = acc;
            acc = gmul(acc, z[j]);
        }
    }
    cx det = mk(1.0, 0.0);
    for (int i = 0; i < a; i++)
        for (int j = i + 1; j < a; j++)
            det = gmul(det, csub(z[j], z[i]));
    for (int j = 0; j < a; j++) p[j] = mk(0.0, 0.0);
    if (cis_zero(det)) return det;
    for (int col = 0; col < a; col++) {
        for (int i = 0; i < a; i++)
            for (int j = 0; j < a; j++)
                work[a * i + j] = (j == col) ? m[i] : vand[a * i + j];
        p[col] = gdiv(detn(work, a), det);
    }
    return det;
}

// Compile-time-degree forms (registers instead of local memory); same
// operation order as the runtime forms above.
template <int A>
SFDT_HD cx det_t(const cx *a) {
    if constexpr (A == 1) return a[0];
    else if constexpr (A == 2) return det2(a[0], a[1], a[2], a[3]);
    else if constexpr (A == 3) return det3(a);
    else return det4(a);
}

template <int A>
SFDT_HD cx hankel_solve_t(const cx *m, cx *c) {
    cx hank[A * A], work[A * A];
#pragma unroll
    for (int i = 0; i < A; i++)
#pragma unroll
        for (int j = 0; j < A; j++) hank[A * i + j] = m[i + j];
    const cx det = det_t<A>(hank);
#pragma unroll
    for (int j = 0; j < A; j++) c[j] = mk(0.0, 0.0);
    if (cis_zero(det)) return det;
#pragma unroll
    for (int col = 0; col < A; col++) {
#pragma unroll
        for (int i = 0; i < A; i++)
#pragma unroll
            for (int j = 0; j < A; j++) work[A * i + j] = (j == col) ? cneg(m[A + i]) : hank[A * i + j];
        c[col] = gdiv(det_t<A>(work), det);
    }
    return det;
}

template <int A>
SFDT_HD cx vandermonde_solve_t(const cx *z, const cx *m, cx *p) {
    cx vand[A * A], work[A * A];
#pragma unroll
    for (int j = 0; j < A; j++) {
        cx acc = mk(1.0, 0.0);
#pragma unroll
        for (int i = 0; i < A; i++) {
            vand[A * i + j] = acc;
            acc = gmul(acc, z[j]);
        }
    }
    cx det = mk(1.0, 0.0);
#pragma unroll
    for (int i = 0; i < A; i++)
#pragma unroll
        for (int j = i + 1; j < A; j++) det = gmul(det, csub(z[j], z[i]));
#pragma unroll
    for (int j = 0; j < A; j++) p[j] = mk(0.0, 0.0);
    if (cis_zero(det)) return det;
#pragma unroll
    for (int col = 0; col < A; col++) {
#pragma unroll
        for (int i = 0; i < A; i++)
#pragma unroll
            for (int j = 0; j < A; j++) work[A * i + j] = (j == col) ? m[i] : vand[A * i + j];
        p[col] = gdiv(det_t<A>(work), det);
    }
    return det;
}

template <int A>
SFDT_HD void poly_roots_t(const cx *c, cx *z) {
    if constexpr (A == 1) z[0] = cneg(c[0]);
    else if constexpr (A == 2) quad_pair(c[1], c[0], &z[0], &z[1]);
    else if constexpr (A == 3) roots3(c[0], c[1], c[2], z);
    else roots4(c[0], c[1], c[2], c[3], z);
}

// NaN-propagating max (numpy np.max / np.maximum semantics)
SFDT_HD double nanmax2(double a, double b)
{
    if (isnan(a) || isnan(b)) return NAN;
    return a > b ? a : b;
}

}  // namespace sfdt
