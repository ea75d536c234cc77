// decode.cuh -- per-bin syndrome decoding under the a-collision model.
//
// One call evaluates exactly what one row of the reference's _batch_decode
// (exact.py:96-149) evaluates: locator solve (Hankel/Cramer), closed-form
// roots, Vandermonde/Cramer values, location snapping and the acceptance
// predicates (singularity, root residual, membership, distinctness,
// unit modulus, snap error, consistency over all S syndromes).  Rows are
// independent in the reference, so a thread owns a bin.
#pragma once

#include "common.cuh"

namespace sfdt {

struct Decoded {
    bool accept;
    bool retryable;    // ~ok: failed on singularity / conditioning
    int64_t loc[4];
    cx val[4];
    cx root[4];
};

// np.sum over a contiguous length-a complex vector (numpy's SIMD add reduce:
// pairs for a = 4, sequential otherwise; checked in tests/test_math.py)
__host__ __device__ __forceinline__ cx npsum(const cx *v, int a) {
    if (a == 4) return cadd(cadd(v[0], v[1]), cadd(v[2], v[3]));
    cx s = v[0];
    for (int i = 1; i < a; i++) s = cadd(s, v[i]);
    return s;
}

// scale ** a as numpy evaluates it (square for 2, pow otherwise)
__host__ __device__ __forceinline__ double powa(double s, int a) {
    if (a == 1) return s;
    if (a == 2) return DMUL(s, s);
    return pow(s, (double)a);
}

// exp(2i pi loc shift / n) with numpy's evaluation order
// (2j * np.pi * locs * shift / n, exact.py:240,271)
__host__ __device__ __forceinline__ cx phase(int64_t loc, int64_t shift, int64_t n) {
    const double th = DMUL(DMUL(TWO_PI, (double)loc), (double)shift) / (double)n;
    return gexp(mk(0.0, th));
}

__host__ __device__ __forceinline__ void decode_try(const cx *syn, int S, int a, int64_t n,
                                                    int64_t m, int64_t bin, Decoded &o) {
    double scale = 0.0;
    for (int l = 0; l < 2 * a; l++) scale = nanmax2(scale, cabs_(syn[l]));
    scale = nanmax2(scale, TINY);
    cx *roots = o.root;
    cx *vals = o.val;
    bool ok;
    if (a == 1) {
        ok = cabs_(syn[0]) > DMUL(SINGULARITY_RTOL, scale);
        roots[0] = ok ? ndiv(syn[1], syn[0]) : mk(0.0, 0.0);
        vals[0] = syn[0];
    } else {
        cx c[4];
        const cx cd = hankel_solve1(syn, a, c);
        ok = cabs_(cd) > DMUL(SINGULARITY_RTOL, powa(scale, a));
        poly_roots1(c, a, roots);
        double cmax = 0.0, resid = 0.0;
        for (int j = 0; j < a; j++) cmax = nanmax2(cmax, cabs_(c[j]));
        for (int r = 0; r < a; r++) {        // syndrome.py:101-106 (numpy Horner)
            cx acc = mk(1.0, 0.0);
            for (int j = a - 1; j >= 0; j--) acc = cadd(nmul(acc, roots[r]), c[j]);
            resid = (r == 0) ? cabs_(acc) : nanmax2(resid, cabs_(acc));
        }
        ok = ok && (resid <= DMUL(1e-8, nanmax2(1.0, cmax)));
        const cx pd = vandermonde_solve1(roots, syn, a, vals);
        double zmax = 0.0;
        for (int j = 0; j < a; j++) zmax = (j == 0) ? cabs_(roots[0]) : nanmax2(zmax, cabs_(roots[j]));
        ok = ok && (cabs_(pd) > DMUL(SINGULARITY_RTOL, powa(nanmax2(1.0, zmax), a)));
    }
    // snapping (exact.py:124-127)
    double snap = 0.0, circ = 0.0;
    for (int j = 0; j < a; j++) {
        const double pos = DMUL(atan2(roots[j].im, roots[j].re), (double)n) / TWO_PI;
        const double sn = rint(pos);
        const double e = fabs(DSUB(pos, sn));
        snap = (j == 0) ? e : nanmax2(snap, e);
        o.loc[j] = isfinite(sn) ? pmod((int64_t)sn, n) : INT64_MIN;
        const double ce = fabs(DSUB(cabs_(roots[j]), 1.0));
        circ = (j == 0) ? ce : nanmax2(circ, ce);
    }
    bool member = true, distinct = true;
    for (int j = 0; j < a; j++) {
        member = member && (o.loc[j] != INT64_MIN) && ((o.loc[j] & (m - 1)) == bin);
        for (int i = 0; i < j; i++) distinct = distinct && (o.loc[i] != o.loc[j]);
    }
    // consistency over all S syndromes (syndrome.py:136-144, exact.py:141-144)
    cx power[4], terms[4];
    for (int j = 0; j < a; j++) power[j] = mk(1.0, 0.0);
    double err = 0.0, smax = 0.0;
    for (int l = 0; l < S; l++) {
        for (int j = 0; j < a; j++) terms[j] = nmul(vals[j], power[j]);
        const cx rec = npsum(terms, a);
        const double e = cabs_(csub(rec, syn[l]));
        err = (l == 0) ? e : nanmax2(err, e);
        smax = (l == 0) ? cabs_(syn[0]) : nanmax2(smax, cabs_(syn[l]));
        for (int j = 0; j < a; j++) power[j] = nmul(power[j], roots[j]);
    }
    const bool consistent = err <= DMUL(CONSISTENCY_RTOL, nanmax2(smax, TINY));
    o.accept = ok && member && distinct && consistent && (circ <= UNIT_MODULUS_TOL) && (snap <= SNAP_TOL);
    o.retryable = !ok;
}

// decode_try with the collision count a compile-time constant: every array
// is register-resident (the runtime-a form keeps its Cramer work matrices in
// local memory).  Same arithmetic, same predicates.
template <int A, int S>
__host__ __device__ __forceinline__ void decode_try_t(const cx *syn, int64_t n, int64_t m, int64_t bin,
                                                      Decoded &o) {
    double scale = 0.0;
#pragma unroll
    for (int l = 0; l < 2 * A; l++) scale = nanmax2(scale, cabs_(syn[l]));
    scale = nanmax2(scale, TINY);
    cx *roots = o.root;
    cx *vals = o.val;
    bool ok;
    if constexpr (A == 1) {
        ok = cabs_(syn[0]) > DMUL(SINGULARITY_RTOL, scale);
        roots[0] = ok ? ndiv(syn[1], syn[0]) : mk(0.0, 0.0);
        vals[0] = syn[0];
    } else {
        cx c[A];
        const cx cd = hankel_solve_t<A>(syn, c);
        ok = cabs_(cd) > DMUL(SINGULARITY_RTOL, powa(scale, A));
        poly_roots_t<A>(c, roots);
        double cmax = 0.0, resid = 0.0;
#pragma unroll
        for (int j = 0; j < A; j++) cmax = nanmax2(cmax, cabs_(c[j]));
#pragma unroll
        for (int r = 0; r < A; r++) {
            cx acc = mk(1.0, 0.0);
#pragma unroll
            for (int j = A - 1; j >= 0; j--) acc = cadd(nmul(acc, roots[r]), c[j]);
            resid = (r == 0) ? cabs_(acc) : nanmax2(resid, cabs_(acc));
        }
        ok = ok && (resid <= DMUL(1e-8, nanmax2(1.0, cmax)));
        const cx pd = vandermonde_solve_t<A>(roots, syn, vals);
        double zmax = 0.0;
#pragma unroll
        for (int j = 0; j < A; j++) zmax = (j == 0) ? cabs_(roots[0]) : nanmax2(zmax, cabs_(roots[j]));
        ok = ok && (cabs_(pd) > DMUL(SINGULARITY_RTOL, powa(nanmax2(1.0, zmax), A)));
    }
    double snap = 0.0, circ = 0.0;
#pragma unroll
    for (int j = 0; j < A; j++) {
        const double pos = DMUL(atan2(roots[j].im, roots[j].re), (double)n) / TWO_PI;
        const double sn = rint(pos);
        const double e = fabs(DSUB(pos, sn));
        snap = (j == 0) ? e : nanmax2(snap, e);
        o.loc[j] = isfinite(sn) ? pmod((int64_t)sn, n) : INT64_MIN;
        const double ce = fabs(DSUB(cabs_(roots[j]), 1.0));
        circ = (j == 0) ? ce : nanmax2(circ, ce);
    }
    bool member = true, distinct = true;
#pragma unroll
    for (int j = 0; j < A; j++) {
        member = member && (o.loc[j] != INT64_MIN) && ((o.loc[j] & (m - 1)) == bin);
#pragma unroll
        for (int i = 0; i < j; i++) distinct = distinct && (o.loc[i] != o.loc[j]);
    }
    cx power[A], terms[A];
#pragma unroll
    for (int j = 0; j < A; j++) power[j] = mk(1.0, 0.0);
    double err = 0.0, smax = 0.0;
#pragma unroll
    for (int l = 0; l < S; l++) {
#pragma unroll
        for (int j = 0; j < A; j++) terms[j] = nmul(vals[j], power[j]);
        const cx rec = npsum(terms, A);
        const double e = cabs_(csub(rec, syn[l]));
        err = (l == 0) ? e : nanmax2(err, e);
        smax = (l == 0) ? cabs_(syn[0]) : nanmax2(smax, cabs_(syn[l]));
#pragma unroll
        for (int j = 0; j < A; j++) power[j] = nmul(power[j], roots[j]);
    }
    const bool consistent = err <= DMUL(CONSISTENCY_RTOL, nanmax2(smax, TINY));
    o.accept = ok && member && distinct && consistent && (circ <= UNIT_MODULUS_TOL) && (snap <= SNAP_TOL);
    o.retryable = !ok;
}

}  // namespace sfdt
