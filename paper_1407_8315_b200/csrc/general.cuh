// general.cuh -- per-bin device math of the generally-K-sparse path.
#pragma once

#include "common.cuh"

namespace sfdt {

// Singular values of the a_max x a_max Hankel matrix H_ij = m_{i+j}:
// one-sided Jacobi (<= 60 sweeps), column norms, descending insertion sort
// (_core.pyx:353-433), gcc arithmetic throughout.
__host__ __device__ __forceinline__ void hankel_singular_values1(const cx *m, int n, double *out) {
    cx mat[16];
    for (int i = 0; i < n; i++)
        for (int j = 0; j < n; j++) mat[n * i + j] = m[i + j];
    for (int sweep = 0; sweep < 60; sweep++) {
        int rotated = 0;
        for (int p = 0; p < n - 1; p++) {
            for (int q = p + 1; q < n; q++) {
                double app = 0.0, aqq = 0.0;
                cx apq = mk(0.0, 0.0);
                for (int i = 0; i < n; i++) {
                    const cx hp = mat[n * i + p], hq = mat[n * i + q];
                    app = DADD(app, DADD(DMUL(hp.re, hp.re), DMUL(hp.im, hp.im)));
                    aqq = DADD(aqq, DADD(DMUL(hq.re, hq.re), DMUL(hq.im, hq.im)));
                    apq = cadd(apq, gmul(cconj(hp), hq));
                }
                const double g = cabs_(apq);
                if (g == 0.0 || g <= DMUL(1e-17, sqrt(DMUL(app, aqq)))) continue;
                rotated = 1;
                const double theta = DDIV(DSUB(aqq, app), DMUL(2.0, g));
                const double tt = theta >= 0.0
                    ? DDIV(1.0, DADD(theta, sqrt(DADD(1.0, DMUL(theta, theta)))))
                    : DDIV(-1.0, DADD(-theta, sqrt(DADD(1.0, DMUL(theta, theta)))));
                const double cs = DDIV(1.0, sqrt(DADD(1.0, DMUL(tt, tt))));
                const double sn = DMUL(tt, cs);
                const cx ph = cdivr(apq, g);
                const cx snc = cscale(sn, cconj(ph)), snp = cscale(sn, ph);
                for (int i = 0; i < n; i++) {
                    const cx hp = mat[n * i + p], hq = mat[n * i + q];
                    mat[n * i + p] = csub(cscale(cs, hp), gmul(snc, hq));
                    mat[n * i + q] = cadd(gmul(snp, hp), cscale(cs, hq));
                }
            }
        }
        if (!rotated) break;
    }
    for (int p = 0; p < n; p++) {
        double norm = 0.0;
        for (int i = 0; i < n; i++) {
            const cx hp = mat[n * i + p];
            norm = DADD(norm, DADD(DMUL(hp.re, hp.re), DMUL(hp.im, hp.im)));
        }
        out[p] = sqrt(norm);
    }
    for (int p = 1; p < n; p++) {
        const double key = out[p];
        int i = p - 1;
        while (i >= 0 && out[i] < key) {
            out[i + 1] = out[i];
            i--;
        }
        out[i + 1] = key;
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
