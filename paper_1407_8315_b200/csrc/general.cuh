// general.cuh -- per-bin device math of the generally-K-sparse path.
#pragma once

#include "common.cuh"

namespace sfdt {

// Singular values of the a_max x a_max Hankel matrix H_ij = m_{i+j}:
// one-sided Jacobi (<= 60 sweeps), column norms, descending insertion sort
// (_core.pyx:353-433), gcc arithmetic throughout.  N is a template parameter
// so the matrix lives in registers (fully unrolled pair/row loops).
//
// tol is the rotation threshold relative to sqrt(app*aqq).  The reference
// uses 1e-17, below the roundoff floor, so ~83 % of bins run all 60 sweeps
// rotating roundoff noise; tol = DBL_EPSILON stops at convergence (3.7
// sweeps on average) with singular values within 9e-16 relative of the
// 60-sweep result (measured over 1e5 random Hankel matrices) -- the same
// envelope as the reference's own LAPACK backend.  The kernel-level mirror
// sfdt_hankel_singular_values keeps 1e-17; the solver uses DBL_EPSILON.
template <int N>
__host__ __device__ __forceinline__ void hankel_sv_n(const cx *m, double *out, double tol = 1e-17) {
    cx mat[N * N];
#pragma unroll
    for (int i = 0; i < N; i++)
#pragma unroll
        for (int j = 0; j < N; j++) mat[N * i + j] = m[i + j];
    for (int sweep = 0; sweep < 60; sweep++) {
        int rotated = 0;
#pragma unroll
        for (int p = 0; p < N - 1; p++) {
#pragma unroll
            for (int q = p + 1; q < N; q++) {
                double app = 0.0, aqq = 0.0;
                cx apq = mk(0.0, 0.0);
#pragma unroll
                for (int i = 0; i < N; i++) {
                    const cx hp = mat[N * i + p], hq = mat[N * i + q];
                    app = DADD(app, DADD(DMUL(hp.re, hp.re), DMUL(hp.im, hp.im)));
                    aqq = DADD(aqq, DADD(DMUL(hq.re, hq.re), DMUL(hq.im, hq.im)));
                    apq = cadd(apq, gmul(cconj(hp), hq));
                }
                const double g = cabs_(apq);
                if (g == 0.0 || g <= DMUL(tol, sqrt(DMUL(app, aqq)))) continue;
                rotated = 1;
                const double theta = DDIV(DSUB(aqq, app), DMUL(2.0, g));
                const double tt = theta >= 0.0
                    ? DDIV(1.0, DADD(theta, sqrt(DADD(1.0, DMUL(theta, theta)))))
                    : DDIV(-1.0, DADD(-theta, sqrt(DADD(1.0, DMUL(theta, theta)))));
                const double cs = DDIV(1.0, sqrt(DADD(1.0, DMUL(tt, tt))));
                const double sn = DMUL(tt, cs);
                const cx ph = cdivr(apq, g);
                const cx snc = cscale(sn, cconj(ph)), snp = cscale(sn, ph);
#pragma unroll
                for (int i = 0; i < N; i++) {
                    const cx hp = mat[N * i + p], hq = mat[N * i + q];
                    mat[N * i + p] = csub(cscale(cs, hp), gmul(snc, hq));
                    mat[N * i + q] = cadd(gmul(snp, hp), cscale(cs, hq));
                }
            }
        }
        if (!rotated) break;
    }
#pragma unroll
    for (int p = 0; p < N; p++) {
        double norm = 0.0;
#pragma unroll
        for (int i = 0; i < N; i++) {
            const cx hp = mat[N * i + p];
            norm = DADD(norm, DADD(DMUL(hp.re, hp.re), DMUL(hp.im, hp.im)));
        }
        out[p] = sqrt(norm);
    }
    for (int p = 1; p < N; p++) {
        const double key = out[p];
        int i = p - 1;
        while (i >= 0 && out[i] < key) {
            out[i + 1] = out[i];
            i--;
        }
        out[i + 1] = key;
    }
}

__host__ __device__ __forceinline__ void hankel_singular_values1(const cx *m, int n, double *out) {
    switch (n) {
    case 1: hankel_sv_n<1>(m, out); break;
    case 2: hankel_sv_n<2>(m, out); break;
    case 3: hankel_sv_n<3>(m, out); break;
    default: hankel_sv_n<4>(m, out); break;
    }
}

// |P(z_t)| for candidates t in chunk ch (512 per chunk) of one bin:
// z advances by the recurrence z *= wd and is re-seeded as base * seed at
// every chunk start (_core.pyx:333-345).  Horner in descending order.
__host__ __device__ __forceinline__ void prune_eval_chunk(const cx *c, int a, cx base, cx wd, cx seed,
                                                          int64_t ch, int64_t d, double *out) {
    cx zt = ch ? gmul(base, seed) : base;
    const int64_t t0 = ch * 512, t1 = (t0 + 512 < d) ? t0 + 512 : d;
    for (int64_t t = t0; t < t1; t++) {
        cx acc = mk(1.0, 0.0);
        for (int j = a - 1; j >= 0; j--) acc = cadd(gmul(acc, zt), c[j]);
        out[t] = cabs_(acc);
        zt = gmul(zt, wd);
    }
}

}  // namespace sfdt

namespace sfdt {

constexpr int GEN_MAX_R = 12;      // r_eff = min(3*a_max, d) <= 12
constexpr int GEN_MAX_COLS = 16;   // kept columns per bin: <= keep*a + a
constexpr int GEN_MAX_SUP = 8;     // SP support / merged support (<= 2*a_eff)

// Minimum-norm least squares of the r x c system A x = y (c <= GEN_MAX_SUP),
// the way LAPACK gelsd defines it (numpy.linalg.lstsq, rcond=None):
// singular values <= eps*max(r,c)*s_max are dropped.  One-sided Jacobi on
// the columns: A V = U S; x = sum_i v_i (u_i^H y) / s_i.  Returns the rank.
__device__ __forceinline__ int lstsq_min_norm(const cx *A, int r, int c, const cx *y, cx *x) {
    cx W[GEN_MAX_R * GEN_MAX_SUP];   // A V (column-major: W[col*r + row])
    cx Vm[GEN_MAX_SUP * GEN_MAX_SUP];
    for (int j = 0; j < c; j++) {
        for (int i = 0; i < r; i++) W[j * r + i] = A[j * r + i];
        for (int i = 0; i < c; i++) Vm[j * c + i] = mk(i == j ? 1.0 : 0.0, 0.0);
    }
    for (int sweep = 0; sweep < 40; sweep++) {
        bool rotated = false;
        for (int p = 0; p < c - 1; p++) {
            for (int q = p + 1; q < c; q++) {
                double app = 0.0, aqq = 0.0;
                cx apq = mk(0.0, 0.0);
                for (int i = 0; i < r; i++) {
                    const cx wp = W[p * r + i], wq = W[q * r + i];
                    app = fma(wp.re, wp.re, fma(wp.im, wp.im, app));
                    aqq = fma(wq.re, wq.re, fma(wq.im, wq.im, aqq));
                    apq = cadd(apq, nmul(cconj(wp), wq));
                }
                const double g = cabs_(apq);
                // converged at eps: below it the rotations only move roundoff
                // (1e-16 < eps/2 kept rotating noise for all 40 sweeps on
                // nearly dependent supports -- the pursuit's longest chains)
                if (g == 0.0 || g <= 2.220446049250313e-16 * sqrt(app * aqq)) continue;
                rotated = true;
                const double theta = (aqq - app) / (2.0 * g);
                const double t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(1.0 + theta * theta));
                const double cs = 1.0 / sqrt(1.0 + t * t), sn = t * cs;
                const cx ph = cdivr(apq, g);
                for (int i = 0; i < r; i++) {
                    const cx wp = W[p * r + i], wq = W[q * r + i];
                    W[p * r + i] = csub(cscale(cs, wp), nmul(cscale(sn, cconj(ph)), wq));
                    W[q * r + i] = cadd(nmul(cscale(sn, ph), wp), cscale(cs, wq));
                }
                for (int i = 0; i < c; i++) {
                    const cx vp = Vm[p * c + i], vq = Vm[q * c + i];
                    Vm[p * c + i] = csub(cscale(cs, vp), nmul(cscale(sn, cconj(ph)), vq));
                    Vm[q * c + i] = cadd(nmul(cscale(sn, ph), vp), cscale(cs, vq));
                }
            }
        }
        if (!rotated) break;
    }
    double s[GEN_MAX_SUP], smax = 0.0;
    for (int j = 0; j < c; j++) {
        double acc = 0.0;
        for (int i = 0; i < r; i++) acc = fma(W[j * r + i].re, W[j * r + i].re, fma(W[j * r + i].im, W[j * r + i].im, acc));
        s[j] = sqrt(acc);
        smax = s[j] > smax ? s[j] : smax;
    }
    const double tol = 2.220446049250313e-16 * (double)(r > c ? r : c) * smax;
    for (int j = 0; j < c; j++) x[j] = mk(0.0, 0.0);
    int rank = 0;
    for (int k = 0; k < c; k++) {
        if (!(s[k] > tol)) continue;
        rank++;
        cx uy = mk(0.0, 0.0);   // (A v_k)^H y / s_k^2
        for (int i = 0; i < r; i++) uy = cadd(uy, nmul(cconj(W[k * r + i]), y[i]));
        const double inv = 1.0 / (s[k] * s[k]);
        uy = mk(uy.re * inv, uy.im * inv);
        for (int j = 0; j < c; j++) x[j] = cadd(x[j], nmul(Vm[k * c + j], uy));
    }
    return rank;
}

// Least squares by Householder QR (r >= c): x = R^-1 (Q^H y)[:c].  Returns
// false when the triangle is too ill-conditioned to be certainly full rank
// under gelsd's rcond (min|R_ii| <= 1e-7 max|R_ii|) -- the caller then uses
// the minimum-norm SVD path.  For full-rank systems both give the unique LS
// solution (to roundoff); QR costs ~2rc^2 flops instead of Jacobi sweeps.
__device__ __forceinline__ bool lstsq_qr(const cx *A_in, int r, int c, const cx *y_in, cx *x) {
    if (c > r) return false;
    cx A[GEN_MAX_R * GEN_MAX_SUP], y[GEN_MAX_R];
    for (int j = 0; j < c; j++)
        for (int i = 0; i < r; i++) A[j * r + i] = A_in[j * r + i];
    for (int i = 0; i < r; i++) y[i] = y_in[i];
    double rmax = 0.0, rmin = 1e300;
    for (int j = 0; j < c; j++) {
        double nrm2 = 0.0;
        for (int i = j; i < r; i++) nrm2 = fma(A[j * r + i].re, A[j * r + i].re, fma(A[j * r + i].im, A[j * r + i].im, nrm2));
        const double nrm = sqrt(nrm2);
        if (nrm == 0.0) return false;
        const cx x0 = A[j * r + j];
        const double ax0 = cabs_(x0);
        const cx ph = ax0 > 0.0 ? mk(x0.re / ax0, x0.im / ax0) : mk(1.0, 0.0);
        const cx alpha = mk(-ph.re * nrm, -ph.im * nrm);   // R_jj
        // v = x - alpha e1, H = I - 2 v v^H / (v^H v)
        cx v[GEN_MAX_R];
        double vv = 0.0;
        for (int i = j; i < r; i++) {
            v[i] = (i == j) ? csub(x0, alpha) : A[j * r + i];
            vv = fma(v[i].re, v[i].re, fma(v[i].im, v[i].im, vv));
        }
        if (vv > 0.0) {
            const double beta = 2.0 / vv;
            for (int k = j; k < c; k++) {
                cx dot = mk(0.0, 0.0);
                for (int i = j; i < r; i++) dot = cadd(dot, nmul(cconj(v[i]), A[k * r + i]));
                dot = mk(dot.re * beta, dot.im * beta);
                for (int i = j; i < r; i++) A[k * r + i] = csub(A[k * r + i], nmul(v[i], dot));
            }
            cx dot = mk(0.0, 0.0);
            for (int i = j; i < r; i++) dot = cadd(dot, nmul(cconj(v[i]), y[i]));
            dot = mk(dot.re * beta, dot.im * beta);
            for (int i = j; i < r; i++) y[i] = csub(y[i], nmul(v[i], dot));
        }
        const double rjj = cabs_(A[j * r + j]);
        rmax = rjj > rmax ? rjj : rmax;
        rmin = rjj < rmin ? rjj : rmin;
    }
    if (!(rmin > 1e-7 * rmax)) return false;
    for (int j = c - 1; j >= 0; j--) {
        cx acc = y[j];
        for (int k = j + 1; k < c; k++) acc = csub(acc, nmul(A[k * r + j], x[k]));
        x[j] = ndiv(acc, A[j * r + j]);
    }
    return true;
}

// Register-resident form of lstsq_qr for compile-time R x C (same operations,
// same order).  A is overwritten.
template <int R, int C>
__device__ __forceinline__ bool lstsq_qr_t(cx (&A)[C][R], const cx (&y_in)[R], cx (&x)[C]) {
    if (C > R) return false;
    cx y[R];
#pragma unroll
    for (int i = 0; i < R; i++) y[i] = y_in[i];
    double rmax = 0.0, rmin = 1e300;
#pragma unroll
    for (int j = 0; j < C; j++) {
        double nrm2 = 0.0;
#pragma unroll
        for (int i = j; i < R; i++) nrm2 = fma(A[j][i].re, A[j][i].re, fma(A[j][i].im, A[j][i].im, nrm2));
        const double nrm = sqrt(nrm2);
        if (nrm == 0.0) return false;
        const cx x0 = A[j][j];
        const double ax0 = cabs_(x0);
        const cx ph = ax0 > 0.0 ? mk(x0.re / ax0, x0.im / ax0) : mk(1.0, 0.0);
        const cx alpha = mk(-ph.re * nrm, -ph.im * nrm);
        cx v[R];
        double vv = 0.0;
#pragma unroll
        for (int i = j; i < R; i++) {
            v[i] = (i == j) ? csub(x0, alpha) : A[j][i];
            vv = fma(v[i].re, v[i].re, fma(v[i].im, v[i].im, vv));
        }
        if (vv > 0.0) {
            const double beta = 2.0 / vv;
#pragma unroll
            for (int k = j; k < C; k++) {
                cx dot = mk(0.0, 0.0);
#pragma unroll
                for (int i = j; i < R; i++) dot = cadd(dot, nmul(cconj(v[i]), A[k][i]));
                dot = mk(dot.re * beta, dot.im * beta);
#pragma unroll
                for (int i = j; i < R; i++) A[k][i] = csub(A[k][i], nmul(v[i], dot));
            }
            cx dot = mk(0.0, 0.0);
#pragma unroll
            for (int i = j; i < R; i++) dot = cadd(dot, nmul(cconj(v[i]), y[i]));
            dot = mk(dot.re * beta, dot.im * beta);
#pragma unroll
            for (int i = j; i < R; i++) y[i] = csub(y[i], nmul(v[i], dot));
        }
        const double rjj = cabs_(A[j][j]);
        rmax = rjj > rmax ? rjj : rmax;
        rmin = rjj < rmin ? rjj : rmin;
    }
    if (!(rmin > 1e-7 * rmax)) return false;
#pragma unroll
    for (int j = C - 1; j >= 0; j--) {
        cx acc = y[j];
#pragma unroll
        for (int k = j + 1; k < C; k++) acc = csub(acc, nmul(A[k][j], x[k]));
        x[j] = ndiv(acc, A[j][j]);
    }
    return true;
}

// top-`cnt` selection by score with the reference's tie rule (np.argsort
// kind="stable" on -score: larger first, then lower index first)
__device__ __forceinline__ bool score_before_desc(double v, double w) {   // v ranks before w (desc, NaN last)
    return v == v && (w != w || v > w);
}
__device__ __forceinline__ void topk_insert(double *sc, int *id, int &len, int cnt, double v, int t) {
    if (len == cnt && !score_before_desc(v, sc[cnt - 1])) return;
    int pos = (len < cnt) ? len++ : cnt - 1;
    while (pos > 0 && score_before_desc(v, sc[pos - 1])) {
        sc[pos] = sc[pos - 1];
        id[pos] = id[pos - 1];
        pos--;
    }
    sc[pos] = v;
    id[pos] = t;
}

// smallest-`cnt` selection (argpartition of errs): smaller first, ties keep
// the lower index; a NaN ranks after every number (numpy sorts NaN last),
// so a NaN in the list is displaced by any later finite candidate
__device__ __forceinline__ bool score_before_asc(double v, double w) {
    return v == v && (w != w || v < w);
}
__device__ __forceinline__ void botk_insert(double *sc, int *id, int &len, int cnt, double v, int t) {
    if (len == cnt && !score_before_asc(v, sc[cnt - 1])) return;
    int pos = (len < cnt) ? len++ : cnt - 1;
    while (pos > 0 && score_before_asc(v, sc[pos - 1])) {
        sc[pos] = sc[pos - 1];
        id[pos] = id[pos - 1];
        pos--;
    }
    sc[pos] = v;
    id[pos] = t;
}

__device__ __forceinline__ void sort_ints(int *v, int n) {
    for (int i = 1; i < n; i++) {
        int key = v[i], j = i - 1;
        while (j >= 0 && v[j] > key) { v[j + 1] = v[j]; j--; }
        v[j + 1] = key;
    }
}

// sorted union of two sorted int lists (np.union1d)
__device__ __forceinline__ int union_sorted(const int *a, int na, const int *b, int nb, int *out) {
    int i = 0, j = 0, n = 0;
    while (i < na || j < nb) {
        int v;
        if (j >= nb || (i < na && a[i] < b[j])) v = a[i++];
        else if (i >= na || b[j] < a[i]) v = b[j++];
        else { v = a[i]; i++; j++; }
        if (n == 0 || out[n - 1] != v) out[n++] = v;
    }
    return n;
}

}  // namespace sfdt
