// decode_coop.cuh -- decode_try_t spread over a group of 8 lanes.
//
// One thread per bin (decode.cuh) leaves a multi-collision bin as one serial
// FP64 chain: 25k / 68k / 109k cycles for a = 2 / 3 / 4 (clock64, config 2),
// and the non-iterative solver tries a = 2, 3, 4 one after the other
// (exact.py:184-192), so a single a = 4 bin costs ~100 us whatever the batch
// size.  The pieces of one trial are independent of each other: the a + 1
// Cramer determinants of the Hankel solve (_core.pyx:127-162), the a root
// residuals (syndrome.py:101-106), the a Vandermonde columns
// (_core.pyx:273-312), the a snaps (exact.py:124-127) and the S syndrome
// reconstructions (exact.py:141-144).  Here lane g of an 8-lane group computes
// piece g of each stage and the group exchanges the results by shuffles; the
// closed-form roots (one chain by nature) are computed by every lane.  Every
// value is produced by the same operation sequence as in decode_try_t, so the
// results are bit-identical (tests/test_gpu_parity.py::
// test_cooperative_decode_bitwise); only the chain is ~3x shorter.  The trials
// for different a run in different warps of the CTA (k_decode_coop), which
// takes the minimum accepted a: the sequential early exit of the reference
// picks exactly that one, because a trial depends only on the bin's syndromes.
#pragma once

#include "decode.cuh"

// phase timestamps for tools/decode_phases.cu (empty in the product build)
#ifndef SFDT_COOP_CLK
#define SFDT_COOP_CLK(i)
#endif

namespace sfdt {

constexpr int COOP_G = 8;   // lanes per bin; >= S = 2 * a_max and >= a_max + 1

template <int N>
__device__ __forceinline__ cx cx_sel(const cx *v, int j) {
    cx r = v[0];
#pragma unroll
    for (int i = 1; i < N; i++)
        if (j == i) r = v[i];
    return r;
}

__device__ __forceinline__ cx grp_bcast(cx v, int src) {
    return mk(__shfl_sync(0xffffffffu, v.re, src, COOP_G), __shfl_sync(0xffffffffu, v.im, src, COOP_G));
}

__device__ __forceinline__ double grp_nanmax(double v) {
#pragma unroll
    for (int o = 1; o < COOP_G; o <<= 1) v = nanmax2(v, __shfl_xor_sync(0xffffffffu, v, o, COOP_G));
    return v;
}

struct DecodedCoop {
    bool accept;
    bool retryable;
    int64_t loc[4];
    cx val[4];
};

// All 32 lanes call this together; lanes g = lane & 7 of a group share one
// bin's syndromes (every lane holds all S of them).  On return every lane of
// the group holds the same DecodedCoop.
template <int A, int S>
__device__ __forceinline__ void decode_try_coop(const cx *syn, int64_t n, int64_t m, int64_t bin, int g,
                                                DecodedCoop &o) {
    static_assert(A >= 2 && A <= 4 && S <= COOP_G && 2 * A <= S, "group layout");
    // |syn[g]|: the scale (l < 2A) and the consistency bound (l < S)
    const cx mine = cx_sel<S>(syn, g < S ? g : 0);
    const double habs = cabs_(mine);
    double scale = grp_nanmax(g < 2 * A ? habs : 0.0);
    scale = nanmax2(scale, TINY);
    const double smax = grp_nanmax(habs);   // lanes >= S repeat syn[0]
    SFDT_COOP_CLK(1);

    // Hankel / Cramer: lane 0 the determinant, lane 1 + col column col
    cx c[A];
    cx cd;
    {
        const int col = g - 1;
        cx work[A * A];
#pragma unroll
        for (int i = 0; i < A; i++)
#pragma unroll
            for (int j = 0; j < A; j++) work[A * i + j] = (j == col) ? cneg(syn[A + i]) : syn[i + j];
        const cx dt = det_t<A>(work);
        cd = grp_bcast(dt, 0);
        const bool zero = cis_zero(cd);
        const cx cm = zero ? mk(0.0, 0.0) : gdiv(dt, cd);
#pragma unroll
        for (int j = 0; j < A; j++) c[j] = grp_bcast(cm, j + 1);
    }
    SFDT_COOP_CLK(2);
    bool ok = cabs_(cd) > DMUL(SINGULARITY_RTOL, powa(scale, A));
    cx roots[A];
    poly_roots_t<A>(c, roots);
    SFDT_COOP_CLK(3);

    // per-root work on lane j < A (lanes >= A repeat root 0)
    const int jr = g < A ? g : 0;
    const cx rj = cx_sel<A>(roots, jr);
    const double rabs = cabs_(rj);
    {
        cx acc = mk(1.0, 0.0);
#pragma unroll
        for (int j = A - 1; j >= 0; j--) acc = cadd(nmul(acc, rj), c[j]);
        const double resid = grp_nanmax(cabs_(acc));
        const double cmax = grp_nanmax(g < A ? cabs_(cx_sel<A>(c, jr)) : 0.0);
        ok = ok && (resid <= DMUL(1e-8, nanmax2(1.0, cmax)));
    }
    const double zmax = grp_nanmax(rabs);
    SFDT_COOP_CLK(4);

    // Vandermonde / Cramer: the determinant (a short product) on every lane,
    // column g on lane g < A
    {
        cx vand[A * A];
#pragma unroll
        for (int j = 0; j < A; j++) {
            cx acc = mk(1.0, 0.0);
#pragma unroll
            for (int i = 0; i < A; i++) {
                vand[A * i + j] = acc;
                acc = gmul(acc, roots[j]);
            }
        }
        cx pd = mk(1.0, 0.0);
#pragma unroll
        for (int i = 0; i < A; i++)
#pragma unroll
            for (int j = i + 1; j < A; j++) pd = gmul(pd, csub(roots[j], roots[i]));
        cx work[A * A];
#pragma unroll
        for (int i = 0; i < A; i++)
#pragma unroll
            for (int j = 0; j < A; j++) work[A * i + j] = (j == g) ? syn[i] : vand[A * i + j];
        const bool zero = cis_zero(pd);
        const cx pm = zero ? mk(0.0, 0.0) : gdiv(det_t<A>(work), pd);
#pragma unroll
        for (int j = 0; j < A; j++) o.val[j] = grp_bcast(pm, j);
        ok = ok && (cabs_(pd) > DMUL(SINGULARITY_RTOL, powa(nanmax2(1.0, zmax), A)));
    }

    SFDT_COOP_CLK(5);
    // snapping (exact.py:124-127) of root jr
    double snap, circ;
    {
        const double pos = DMUL(atan2(rj.im, rj.re), (double)n) / TWO_PI;
        const double sn = rint(pos);
        snap = grp_nanmax(fabs(DSUB(pos, sn)));
        const long long lm = isfinite(sn) ? pmod((int64_t)sn, n) : INT64_MIN;
#pragma unroll
        for (int j = 0; j < A; j++) o.loc[j] = __shfl_sync(0xffffffffu, lm, j, COOP_G);
        circ = grp_nanmax(fabs(DSUB(rabs, 1.0)));
    }
    bool member = true, distinct = true;
#pragma unroll
    for (int j = 0; j < A; j++) {
        member = member && (o.loc[j] != INT64_MIN) && ((o.loc[j] & (m - 1)) == bin);
#pragma unroll
        for (int i = 0; i < j; i++) distinct = distinct && (o.loc[i] != o.loc[j]);
    }

    SFDT_COOP_CLK(6);
    // consistency: lane l < S rebuilds syndrome l (powers by l successive
    // multiplications, as the reference's running product)
    double err;
    {
        const int l = g < S ? g : 0;
        cx power[A], terms[A];
#pragma unroll
        for (int j = 0; j < A; j++) power[j] = mk(1.0, 0.0);
#pragma unroll
        for (int it = 0; it < S - 1; it++) {
            if (it < l) {
#pragma unroll
                for (int j = 0; j < A; j++) power[j] = nmul(power[j], roots[j]);
            }
        }
#pragma unroll
        for (int j = 0; j < A; j++) terms[j] = nmul(o.val[j], power[j]);
        const cx rec = npsum(terms, A);
        err = grp_nanmax(cabs_(csub(rec, mine)));
    }
    const bool consistent = err <= DMUL(CONSISTENCY_RTOL, nanmax2(smax, TINY));
    o.accept = ok && member && distinct && consistent && (circ <= UNIT_MODULUS_TOL) && (snap <= SNAP_TOL);
    o.retryable = !ok;
    SFDT_COOP_CLK(7);
}

}  // namespace sfdt
