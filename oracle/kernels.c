/*
 * oracle/kernels.c -- TEST INFRASTRUCTURE ONLY (the parity checker).
 *
 * Plain-C restatement of the six numeric kernels behind the reference's
 * backend seam (`sfft_dt._kernels`, /root/reference/pkg/src/sfft_dt/_kernels/
 * __init__.py:19-24), following the compiled backend
 * (`_kernels/_core.pyx`).  The reference builds that file with gcc -O3 and
 * no -march (pkg/setup.py:14-30), i.e. C99 `double _Complex` arithmetic
 * without FMA contraction, complex division through libgcc's __divdc3 and
 * glibc's cexp/csqrt/cpow/cabs.  Compiling this file the same way gives
 * bit-identical results, which tests/test_oracle.py checks against the real
 * compiled reference (oracle/_ref) and the committed golden vectors.
 *
 * Nothing in the product (paper_1407_8315_b200/) links or calls this code.
 */
#include <complex.h>
#include <math.h>
#include <stdint.h>
#include <string.h>

typedef double _Complex cplx;

/* ------------------------------------------------------------------ FFT
 * _core.pyx:35-77: copy, bit-reverse, radix-2 DIT stages m = 2..n with a
 * per-block twiddle recurrence w *= wlen that is re-seeded by cexp every
 * 256 steps.  sign = -1 forward, +1 inverse; no scaling. */
int orc_fft_radix2(const cplx *in, cplx *a, int64_t n, int inverse)
{
    if (n <= 0 || (n & (n - 1)))
        return -1;
    if (a != in)
        memcpy(a, in, (size_t)n * sizeof(cplx));
    const double sign = inverse ? 1.0 : -1.0;
    for (int64_t i = 1, j = 0; i < n; i++) {
        int64_t bit = n >> 1;
        for (; j & bit; bit >>= 1)
            j ^= bit;
        j |= bit;
        if (i < j) {
            cplx u = a[i];
            a[i] = a[j];
            a[j] = u;
        }
    }
    const cplx two_i = 2.0 * I;
    for (int64_t m = 2; m <= n; m <<= 1) {
        const int64_t half = m >> 1;
        const cplx wlen = cexp(((cplx)sign * two_i * (cplx)M_PI) / (cplx)(double)m);
        for (int64_t start = 0; start < n; start += m) {
            cplx w = 1.0;
            for (int64_t k = 0; k < half; k++) {
                if ((k & 255) == 0 && k > 0)
                    w = cexp((((cplx)sign * two_i * (cplx)M_PI) * (cplx)(double)k) / (cplx)(double)m);
                cplx u = a[start + k];
                cplx t = a[start + k + half] * w;
                a[start + k] = u + t;
                a[start + k + half] = u - t;
                w = w * wlen;
            }
        }
    }
    return 0;
}

/* ------------------------------------------------- cofactor determinants
 * _core.pyx:84-120 (row-major, first-row expansion). */
static inline cplx det2(cplx a00, cplx a01, cplx a10, cplx a11)
{
    return a00 * a11 - a01 * a10;
}

static inline cplx det3(const cplx *a)
{
    return a[0] * det2(a[4], a[5], a[7], a[8]) - a[1] * det2(a[3], a[5], a[6], a[8])
         + a[2] * det2(a[3], a[4], a[6], a[7]);
}

static cplx det4(const cplx *a)
{
    cplx minor[9];
    cplx acc = 0.0;
    double sign = 1.0;
    for (int col = 0; col < 4; col++) {
        int i = 0;
        for (int r = 1; r < 4; r++)
            for (int cc = 0; cc < 4; cc++)
                if (cc != col)
                    minor[i++] = a[4 * r + cc];
        acc += ((cplx)sign * a[col]) * det3(minor);
        sign = -sign;
    }
    return acc;
}

static cplx detn(const cplx *a, int n)
{
    switch (n) {
    case 1: return a[0];
    case 2: return det2(a[0], a[1], a[2], a[3]);
    case 3: return det3(a);
    default: return det4(a);
    }
}

/* ---------------------------------------------------------- Hankel solve
 * _core.pyx:127-162: cd = det H (H_ij = m_{i+j}); c_col = det(H with column
 * col <- -m_{a..2a-1}) / cd; rows with cd == 0 stay zero.  m is (nb, ld). */
void orc_hankel_solve(const cplx *m, int64_t nb, int64_t ld, int a, cplx *c, cplx *cd)
{
    cplx hank[16], work[16];
    for (int64_t b = 0; b < nb; b++) {
        const cplx *mb = m + b * ld;
        for (int i = 0; i < a; i++)
            for (int j = 0; j < a; j++)
                hank[a * i + j] = mb[i + j];
        cplx det = detn(hank, a);
        cd[b] = det;
        for (int j = 0; j < a; j++)
            c[b * a + j] = 0.0;
        if (det == 0.0)
            continue;
        for (int col = 0; col < a; col++) {
            for (int i = 0; i < a; i++)
                for (int j = 0; j < a; j++)
                    work[a * i + j] = (j == col) ? -mb[a + i] : hank[a * i + j];
            c[b * a + col] = detn(work, a) / det;
        }
    }
}

/* ------------------------------------------------------ closed-form roots
 * _core.pyx:169-266. */
static const cplx W1 = -0.5 + 0.8660254037844386 * I;
static const cplx W2 = -0.5 - 0.8660254037844386 * I;

static void quad_pair(cplx b, cplx c, cplx *z0, cplx *z1)
{
    cplx disc = csqrt(b * b - 4.0 * c);
    if (creal(conj(b) * disc) < 0.0)
        disc = -disc;
    cplx q = -0.5 * (b + disc);
    *z0 = q;
    *z1 = (q == 0.0) ? -0.5 * (b - disc) : c / q;
}

static void cube_pair(cplx g, cplx h, cplx *aa, cplx *bb)
{
    cplx r = csqrt(g * g + h * h * h);
    cplx lo = g - r, hi = g + r;
    cplx a3 = (cabs(lo) >= cabs(hi)) ? lo : hi;
    cplx a = cpow(a3, 1.0 / 3.0);
    *aa = a;
    *bb = (a == 0.0) ? 0.0 : -h / a;
}

static void roots3(cplx c0, cplx c1, cplx c2, cplx *z)
{
    cplx g = c0 / 2.0 - c1 * c2 / 6.0 + c2 * c2 * c2 / 27.0;
    cplx h = c1 / 3.0 - c2 * c2 / 9.0;
    cplx a, b;
    cube_pair(g, h, &a, &b);
    cplx shift = -c2 / 3.0;
    z[0] = shift - a - b;
    z[1] = shift - W1 * a - W2 * b;
    z[2] = shift - W2 * a - W1 * b;
}

static void roots4(cplx c0, cplx c1, cplx c2, cplx c3, cplx *z)
{
    cplx g = (72.0 * c0 * c2 + 9.0 * c1 * c2 * c3 - 27.0 * c1 * c1
              - 27.0 * c0 * c3 * c3 - 2.0 * c2 * c2 * c2) / 432.0;
    cplx h = (3.0 * c1 * c3 - 12.0 * c0 - c2 * c2) / 36.0;
    cplx cc, dd;
    cube_pair(g, h, &cc, &dd);
    cplx y = c2 / 6.0 - cc - dd;
    cplx aa = csqrt(c3 * c3 / 4.0 - c2 + 2.0 * y);
    cplx num = c3 * y - c1;
    double scale_a = 1.0 + cabs(c3) * cabs(c3) / 4.0 + cabs(c2) + 2.0 * cabs(y);
    double scale_b = 1.0 + cabs(y) * cabs(y) + cabs(c0);
    cplx bb;
    if (cabs(aa) > 1e-6 * sqrt(scale_a)) {
        bb = num / (2.0 * aa);
    } else {
        bb = csqrt(y * y - c0);
        if (cabs(bb) > 1e-6 * sqrt(scale_b)) {
            aa = num / (2.0 * bb);
        } else {
            aa = 0.0;
            bb = 0.0;
        }
    }
    quad_pair(c3 / 2.0 + aa, y + bb, &z[0], &z[1]);
    quad_pair(c3 / 2.0 - aa, y - bb, &z[2], &z[3]);
}

/* c is (nb, a) with c_0..c_{a-1}; z is (nb, a). */
void orc_poly_roots(const cplx *c, int64_t nb, int a, cplx *z)
{
    for (int64_t b = 0; b < nb; b++) {
        const cplx *cb = c + b * a;
        cplx *zb = z + b * a;
        switch (a) {
        case 1: zb[0] = -cb[0]; break;
        case 2: quad_pair(cb[1], cb[0], &zb[0], &zb[1]); break;
        case 3: roots3(cb[0], cb[1], cb[2], zb); break;
        default: roots4(cb[0], cb[1], cb[2], cb[3], zb); break;
        }
    }
}

/* ----------------------------------------------------- Vandermonde solve
 * _core.pyx:273-312: V_ij = z_j^i by repeated products, pd = prod_{i<j}
 * (z_j - z_i), p_col = det(V with column col <- m_{0..a-1}) / pd. */
void orc_vandermonde_solve(const cplx *z, const cplx *m, int64_t nb, int a, int64_t ld,
                           cplx *p, cplx *pd)
{
    cplx vand[16], work[16];
    for (int64_t b = 0; b < nb; b++) {
        const cplx *zb = z + b * a;
        const cplx *mb = m + b * ld;
        for (int j = 0; j < a; j++) {
            cplx acc = 1.0;
            for (int i = 0; i < a; i++) {
                vand[a * i + j] = acc;
                acc = acc * zb[j];
            }
        }
        cplx det = 1.0;
        for (int i = 0; i < a; i++)
            for (int j = i + 1; j < a; j++)
                det = det * (zb[j] - zb[i]);
        pd[b] = det;
        for (int j = 0; j < a; j++)
            p[b * a + j] = 0.0;
        if (det == 0.0)
            continue;
        for (int col = 0; col < a; col++) {
            for (int i = 0; i < a; i++)
                for (int j = 0; j < a; j++)
                    work[a * i + j] = (j == col) ? mb[i] : vand[a * i + j];
            p[b * a + col] = detn(work, a) / det;
        }
    }
}

/* ------------------------------------------------------------ prune_eval
 * _core.pyx:319-346: |P(z_t)| at z_t = e^{2 pi i k/n} e^{2 pi i t/d},
 * Horner in descending order, recurrence re-seeded every 512 candidates. */
void orc_prune_eval(const cplx *c, const int64_t *k, int64_t nb, int a, int64_t n, int64_t d,
                    double *out)
{
    const cplx two_i = 2.0 * I;
    const cplx wd = cexp((two_i * (cplx)M_PI) / (cplx)(double)d);
    for (int64_t b = 0; b < nb; b++) {
        const cplx base = cexp(((two_i * (cplx)M_PI) * (cplx)(double)k[b]) / (cplx)(double)n);
        cplx zt = base;
        for (int64_t t = 0; t < d; t++) {
            cplx acc = 1.0;
            for (int j = a - 1; j >= 0; j--)
                acc = acc * zt + c[b * a + j];
            out[b * d + t] = cabs(acc);
            if ((t & 511) == 511)
                zt = base * cexp(((two_i * (cplx)M_PI) * (cplx)(double)(t + 1)) / (cplx)(double)d);
            else
                zt = zt * wd;
        }
    }
}

/* ------------------------------------------- Hankel singular values
 * _core.pyx:353-433: one-sided Jacobi on the columns of the a_max x a_max
 * Hankel matrix (<= 60 sweeps), column norms, insertion sort descending. */
static void jacobi_singvals(cplx *mat, int n, double *out)
{
    for (int sweep = 0; sweep < 60; sweep++) {
        int rotated = 0;
        for (int p = 0; p < n - 1; p++) {
            for (int q = p + 1; q < n; q++) {
                double app = 0.0, aqq = 0.0;
                cplx apq = 0.0;
                for (int i = 0; i < n; i++) {
                    cplx hp = mat[n * i + p], hq = mat[n * i + q];
                    app += creal(hp) * creal(hp) + cimag(hp) * cimag(hp);
                    aqq += creal(hq) * creal(hq) + cimag(hq) * cimag(hq);
                    apq += conj(hp) * hq;
                }
                double g = cabs(apq);
                if (g == 0.0 || g <= 1e-17 * sqrt(app * aqq))
                    continue;
                rotated = 1;
                double theta = (aqq - app) / (2.0 * g);
                double t = theta >= 0.0 ? 1.0 / (theta + sqrt(1.0 + theta * theta))
                                        : -1.0 / (-theta + sqrt(1.0 + theta * theta));
                double cs = 1.0 / sqrt(1.0 + t * t);
                double sn = t * cs;
                cplx ph = apq / (cplx)g;
                for (int i = 0; i < n; i++) {
                    cplx hp = mat[n * i + p], hq = mat[n * i + q];
                    mat[n * i + p] = (cplx)cs * hp - ((cplx)sn * conj(ph)) * hq;
                    mat[n * i + q] = ((cplx)sn * ph) * hp + (cplx)cs * hq;
                }
            }
        }
        if (!rotated)
            break;
    }
    for (int p = 0; p < n; p++) {
        double norm = 0.0;
        for (int i = 0; i < n; i++) {
            cplx hp = mat[n * i + p];
            norm += creal(hp) * creal(hp) + cimag(hp) * cimag(hp);
        }
        out[p] = sqrt(norm);
    }
    for (int p = 1; p < n; p++) {
        double key = out[p];
        int i = p - 1;
        while (i >= 0 && out[i] < key) {
            out[i + 1] = out[i];
            i--;
        }
        out[i + 1] = key;
    }
}

void orc_hankel_singular_values(const cplx *m, int64_t nb, int64_t ld, int a_max, double *out)
{
    cplx mat[16];
    for (int64_t b = 0; b < nb; b++) {
        for (int i = 0; i < a_max; i++)
            for (int j = 0; j < a_max; j++)
                mat[a_max * i + j] = m[b * ld + i + j];
        jacobi_singvals(mat, a_max, out + b * a_max);
    }
}
