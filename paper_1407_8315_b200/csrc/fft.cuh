// fft.cuh -- batched FP64 radix-2 DIT FFT of downsampled views in shared memory.
//
// Arithmetic contract: identical to the reference's fft_radix2
// (_core.pyx:35-77) -- bit-reversal permutation, then stages m = 2..L whose
// butterflies compute t = a[i+h] * w (gcc complex multiply, no FMA),
// a[i] = u + t, a[i+h] = u - t, with w taken from a host-built table that
// replays the reference's twiddle recurrence (sfdt_fft_twiddles).  The
// output is scaled by 1/L exactly as `fft(view) / m` (spectral.py:166), so
// views are bit-identical to the reference's.
//
// The views are gathered straight from the signals (the downsample of
// spectral.py:151-160 fused into the load): view v of signal b is
//   x[b*sig_stride + ((j*jstride + off[v]) & wrap)],  j < L
// (jstride = d, off = shift, wrap = n - 1), loaded with the shifts of one
// d-block adjacent across lanes so every 32-byte sector is used whole.
// Output: out[(b*SV + v)*ldV + k].
#pragma once

#include "common.cuh"
#include <cstdlib>
#include <type_traits>

namespace sfdt {

constexpr int MAX_VIEWS = 24;


struct ViewSrc {
    const void *x;
    int is_c64;          // complex64 storage, upconverted at load
    int nshift;          // views per signal
    int64_t sig_stride;  // elements between signals
    int64_t jstride;     // elements between consecutive view samples (d)
    int64_t wrap;        // index mask (n - 1)
    int64_t off[MAX_VIEWS];
    // views v >= dyn_first take their shift from a device table instead:
    // off = dyn_off[b * dyn_stride + v - dyn_first] (per-signal random shifts)
    const int64_t *dyn_off;
    int dyn_first;
    int64_t dyn_stride;
    int jfast;           // 1: lanes walk j (contiguous rows), 0: lanes walk the views
    // per-signal number of views to compute: views v >= nview[b] are skipped
    // (their slots are never read); nullptr = all nshift views
    const int32_t *nview;
};

__device__ __forceinline__ cx ld_gather(const cx *p) { return ldcx(p); }

__device__ __forceinline__ cx view_load(const ViewSrc &src, int64_t b, int v, int64_t j) {
    const int64_t o = (v >= src.dyn_first) ? __ldg(src.dyn_off + b * src.dyn_stride + (v - src.dyn_first))
                                           : src.off[v];
    const int64_t e = b * src.sig_stride + ((j * src.jstride + o) & src.wrap);
    if (src.is_c64) {
        const float2 f = __ldg(reinterpret_cast<const float2 *>(src.x) + e);
        return mk((double)f.x, (double)f.y);
    }
    return ld_gather(reinterpret_cast<const cx *>(src.x) + e);
}

// 16-byte-granular swizzle of the shared-memory FFT buffers: the low 3 bits
// of the element index are XOR-ed with every higher 3-bit group.  Shared
// memory serves a warp's 16-byte accesses 8 lanes (one quarter) at a time,
// conflict-free iff the 8 lanes hit distinct (index & 7) groups; in every
// access pattern used here the 8 lanes of a quarter differ in 3 consecutive
// index bits (radix passes starting at stage multiples of 3, the bit-
// reversed scatter of the load, the natural-order store), and folding maps 3
// consecutive bit positions onto 3 distinct ones, so all are conflict-free.
__device__ __forceinline__ int swz(int p) {
    int f = p;
    f ^= f >> 3;
    f ^= f >> 6;
    f ^= f >> 12;
    return (p & ~7) | (f & 7);
}

// NST radix-2 stages (half-sizes h .. h*2^(NST-1)) on the G = 2^NST
// elements e0 + q*h of one group, in registers.  With lo = e0 mod h (the
// bits lh .. lh+NST-1 of e0 are zero) the butterfly twiddle index
// (e0 + q*h) mod (h*2^st) is lo + (q mod 2^st)*h: each of the 2^st distinct
// twiddles of stage st is loaded once and shared by its G/2^(st+1)
// butterflies.
template <int NST>
__device__ __forceinline__ void group_stages(cx (&x)[1 << NST], int lo, int h, const cx *__restrict__ tw) {
    constexpr int G = 1 << NST;
#pragma unroll
    for (int st = 0; st < NST; st++) {
        const int Hs = h << st;
        const cx *twh = tw + (Hs - 1) + lo;
#pragma unroll
        for (int qk = 0; qk < (1 << st); qk++) {
            // the reference's w starts at exactly 1 + 0i, and (a*1 - b*0,
            // a*0 + b*1) == (a, b) for finite a, b: the first twiddle of
            // every stage block needs no multiply
            const bool one = (Hs == 1);
            const cx w = one ? mk(1.0, 0.0) : ldcx(twh + qk * h);
#pragma unroll
            for (int q = qk; q < G; q += (2 << st)) {
                const cx u = x[q];
                const cx t = one ? x[q + (1 << st)] : gmul(x[q + (1 << st)], w);
                x[q] = cadd(u, t);
                x[q + (1 << st)] = csub(u, t);
            }
        }
    }
}

// group_stages with every twiddle of the group loaded up front (2^NST - 1
// independent loads in flight instead of one dependent round trip per
// stage); same butterflies, same twiddles -- for kernels with register room
template <int NST>
__device__ __forceinline__ void group_stages_pre(cx (&x)[1 << NST], int lo, int h, const cx *__restrict__ tw) {
    constexpr int G = 1 << NST;
    cx w[G - 1];
#pragma unroll
    for (int st = 0; st < NST; st++) {
        const int Hs = h << st;
#pragma unroll
        for (int qk = 0; qk < (1 << st); qk++)
            w[(1 << st) - 1 + qk] = (Hs == 1) ? mk(1.0, 0.0) : ldcx(tw + (Hs - 1) + lo + qk * h);
    }
#pragma unroll
    for (int st = 0; st < NST; st++) {
        const bool one = ((h << st) == 1);
#pragma unroll
        for (int qk = 0; qk < (1 << st); qk++) {
            const cx ww = w[(1 << st) - 1 + qk];
#pragma unroll
            for (int q = qk; q < G; q += (2 << st)) {
                const cx u = x[q];
                const cx t = one ? x[q + (1 << st)] : gmul(x[q + (1 << st)], ww);
                x[q] = cadd(u, t);
                x[q + (1 << st)] = csub(u, t);
            }
        }
    }
}

template <int NST, bool PRE = false>
__device__ __forceinline__ void fft_pass(cx *a, int nv, int logL, int lh, const cx *__restrict__ tw) {
    constexpr int G = 1 << NST;
    const int L = 1 << logL;
    const int h = 1 << lh;
    const int lg = logL - NST;   // log2(groups per view)
    const int ng = nv << lg;
    // swz(base + q*h) = (swz(base) | q*h) ^ dq[q] when lh >= 3 (bits lh..
    // lh+NST-1 of base are zero and the fold is XOR-linear); one table per
    // pass instead of a fold per element
    int dq[G];
#pragma unroll
    for (int q = 0; q < G; q++) dq[q] = swz(q << lh) & 7;
    for (int g = threadIdx.x; g < ng; g += blockDim.x) {
        const int v = g >> lg;
        const int gg = g & ((1 << lg) - 1);
        const int lo = gg & (h - 1), hi = gg >> lh;
        const int base = v * L + (hi << (lh + NST)) + lo;
        const int e0 = (hi << (lh + NST)) + lo;
        const int sb = swz(base);
        auto at = [&](int q) { return lh >= 3 ? ((sb | (q << lh)) ^ dq[q]) : swz(base + q * h); };   // index within the view
        cx x[G];
#pragma unroll
        for (int q = 0; q < G; q++) x[q] = a[at(q)];
        if constexpr (PRE) group_stages_pre<NST>(x, lo, h, tw);
        else group_stages<NST>(x, lo, h, tw);
#pragma unroll
        for (int q = 0; q < G; q++) a[at(q)] = x[q];
    }
}

// Last pass straight to global memory: the group's outputs are scaled and
// stored (with the activity epilogue) from registers instead of going back
// through shared memory for a separate epilogue sweep.
template <int NST, bool PRE = false, typename Epi>
__device__ __forceinline__ void fft_pass_out(const cx *a, int nv, int logL, int lh, const cx *__restrict__ tw,
                                             Epi &&epi) {
    constexpr int G = 1 << NST;
    const int L = 1 << logL;
    const int h = 1 << lh;
    const int lg = logL - NST;   // log2(groups per view)
    const int ng = nv << lg;
    // swz(base + q*h) = (swz(base) | q*h) ^ dq[q] when lh >= 3 (bits lh..
    // lh+NST-1 of base are zero and the fold is XOR-linear); one table per
    // pass instead of a fold per element
    int dq[G];
#pragma unroll
    for (int q = 0; q < G; q++) dq[q] = swz(q << lh) & 7;
    for (int g = threadIdx.x; g < ng; g += blockDim.x) {
        const int v = g >> lg;
        const int gg = g & ((1 << lg) - 1);
        const int lo = gg & (h - 1), hi = gg >> lh;
        const int base = v * L + (hi << (lh + NST)) + lo;
        const int e0 = (hi << (lh + NST)) + lo;
        const int sb = swz(base);
        auto at = [&](int q) { return lh >= 3 ? ((sb | (q << lh)) ^ dq[q]) : swz(base + q * h); };
        cx x[G];
#pragma unroll
        for (int q = 0; q < G; q++) x[q] = a[at(q)];
        if constexpr (PRE) group_stages_pre<NST>(x, lo, h, tw);
        else group_stages<NST>(x, lo, h, tw);
#pragma unroll
        for (int q = 0; q < G; q++) epi(v, e0 + q * h, x[q]);
    }
}

template <bool PRE = false>
__device__ __forceinline__ void fft_stages_smem(cx *a, int nv, int logL, int lh0, int lh1,
                                                const cx *__restrict__ tw) {
    // up to 3 stages (radix-8 groups) per shared-memory pass (radix-16
    // measured slower: 134 registers halve the resident CTAs)
    for (int lh = lh0; lh < lh1;) {
        const int rem = lh1 - lh;
        const int nst = rem >= 3 ? 3 : rem;
        if (nst == 3) fft_pass<3, PRE>(a, nv, logL, lh, tw);
        else if (nst == 2) fft_pass<2, PRE>(a, nv, logL, lh, tw);
        else fft_pass<1, PRE>(a, nv, logL, lh, tw);
        __syncthreads();
        lh += nst;
    }
}

// Views of length L = 2^logL >= 64 (nv per CTA, view-fastest lanes): the
// first radix-8 pass fused with the strided gather from the signal, the
// middle passes through shared memory, the last pass fused with the
// epilogue epi(view, k, value).  Input j of view v sits at
// s_ibase[v] + ((j*jstride + s_ioff[v]) & src.wrap).
template <typename Epi>
__device__ __forceinline__ void fft_fused_views(cx *a, const ViewSrc &src, int64_t jstride,
                                                const int64_t *s_ibase, const int64_t *s_ioff, int nv,
                                                int logvpc, int logL, const cx *__restrict__ tw, Epi &&epi) {
    const int L = 1 << logL, vpc = 1 << logvpc;
    // First pass fused with the gather: a thread loads the 8 inputs of
    // one radix-8 group (positions hi*8 + q hold inputs j = bitrev(hi*8
    // + q)) straight from the signal, runs stages 0-2 in registers and
    // writes shared memory once.  Lanes vary the view fastest, so one
    // d-block's adjacent shifts share sectors.
    const int gper = L >> 3;
    const int hbits = logL - 3;
    for (int g = threadIdx.x; g < (gper << logvpc); g += blockDim.x) {
        const int v = g & (vpc - 1), hi = g >> logvpc;
        if (v >= nv) continue;
        const int hb = (int)(__brev((unsigned)hi) >> (32 - hbits));
        cx x[8];
#pragma unroll
        for (int q = 0; q < 8; q++) {
            const int q3 = ((q & 1) << 2) | (q & 2) | ((q >> 2) & 1);   // bitrev_3(q)
            const int j = hb + (q3 << hbits);
            const int64_t e = s_ibase[v] + (((int64_t)j * jstride + s_ioff[v]) & src.wrap);
            if (src.is_c64) {
                const float2 f = __ldg(reinterpret_cast<const float2 *>(src.x) + e);
                x[q] = mk((double)f.x, (double)f.y);
            } else {
                x[q] = ld_gather(reinterpret_cast<const cx *>(src.x) + e);
            }
        }
        group_stages<3>(x, 0, 1, tw);
#pragma unroll
        for (int q = 0; q < 8; q++) a[swz(v * L + (hi << 3) + q)] = x[q];
    }
    __syncthreads();
    int lh = 3;
    while (logL - lh > 3) {
        fft_pass<3>(a, nv, logL, lh, tw);
        __syncthreads();
        lh += 3;
    }
    // last pass straight to global memory
    const int nst = logL - lh;
    if (nst == 3) fft_pass_out<3>(a, nv, logL, lh, tw, epi);
    else if (nst == 2) fft_pass_out<2>(a, nv, logL, lh, tw, epi);
    else fft_pass_out<1>(a, nv, logL, lh, tw, epi);
}

template <int MINB>
static __global__ void __launch_bounds__(256, MINB) k_fft_views(const ViewSrc src, int64_t B, int logL, int logvpc,
                                   const cx *__restrict__ tw, cx *__restrict__ out, int SV,
                                   int64_t ldV, int scale, const double *__restrict__ thr,
                                   uint8_t *__restrict__ act) {
    pdl_wait();
    extern __shared__ double4 smem_raw[];
    cx *a = reinterpret_cast<cx *>(smem_raw);
    __shared__ int64_t s_ibase[MAX_VIEWS], s_ioff[MAX_VIEWS], s_obase[MAX_VIEWS], s_sig[MAX_VIEWS];
    __shared__ double s_th[MAX_VIEWS], s_th2hi[MAX_VIEWS], s_th2lo[MAX_VIEWS];
    const int L = 1 << logL, vpc = 1 << logvpc;
    const int64_t nviews = B * src.nshift;
    const int64_t g0 = int64_t(blockIdx.x) << logvpc;
    const int nv = (int)((nviews - g0) < vpc ? (nviews - g0) : vpc);
    if (nv <= 0) return;
    // per-view addressing, once per CTA (no 64-bit divisions or dynamically
    // indexed parameter arrays in the element loops)
    if (src.nview) {   // CTA-uniform: skip when every view of the tile is unused
        __shared__ int s_live;
        if (threadIdx.x == 0) s_live = 0;
        __syncthreads();
        if (threadIdx.x < nv) {
            const int64_t g = g0 + threadIdx.x;
            const int64_t b = g / src.nshift;
            if ((int)(g - b * src.nshift) < __ldg(src.nview + b)) s_live = 1;
        }
        __syncthreads();
        if (!s_live) return;
    }
    if (threadIdx.x < nv) {
        const int64_t g = g0 + threadIdx.x;
        const int64_t b = g / src.nshift;
        const int s = (int)(g - b * src.nshift);
        s_ibase[threadIdx.x] = b * src.sig_stride;
        s_ioff[threadIdx.x] = (s >= src.dyn_first) ? src.dyn_off[b * src.dyn_stride + (s - src.dyn_first)]
                                                  : src.off[s];
        s_obase[threadIdx.x] = (b * SV + s) * ldV;
        s_sig[threadIdx.x] = b;
        if (act) {   // per-view activity bounds, once per CTA
            const double th = thr[b];
            s_th[threadIdx.x] = th;
            s_th2hi[threadIdx.x] = th * th * (1.0 + 1e-6);
            s_th2lo[threadIdx.x] = th * th * (1.0 - 1e-6);
        }
    }
    __syncthreads();
    const double sc = 1.0 / (double)L;   // exact power of two
    // output epilogue: scale, store, activity (exact.py:178): |v| >
    // zero_threshold*rms*d on any view; |v|^2 decides away from the
    // boundary, hypot inside a 1e-6 band
    auto epi = [&](int v, int k, cx y) {
        if (scale) y = mk(DMUL(y.re, sc), DMUL(y.im, sc));
        stcx(out + s_obase[v] + k, y);
        if (act) {
            const double q = y.re * y.re + y.im * y.im;
            if (q > s_th2hi[v] || (q >= s_th2lo[v] && cabs_i(y) > s_th[v]))
                act[s_sig[v] * (int64_t)L + k] = 1;
        }
    };
    if (logL >= 6 && !src.jfast) {
        fft_fused_views(a, src, src.jstride, s_ibase, s_ioff, nv, logvpc, logL, tw, epi);
        return;
    }
    // small views: gather (lanes vary the view fastest for one sample j),
    // bit-reversed scatter to smem, stages, epilogue sweep.  Loads are
    // issued in batches of 8 before their shared-memory stores.
    const int total = L << logvpc;
    for (int i0 = 0; i0 < total; i0 += 8 * 256) {
        cx vals[8];
        int dst[8];
#pragma unroll
        for (int u = 0; u < 8; u++) {
            const int i = i0 + u * 256 + threadIdx.x;
            dst[u] = -1;
            if (i < total) {
                const int v = src.jfast ? (i >> logL) : (i & (vpc - 1));
                const int j = src.jfast ? (i & (L - 1)) : (i >> logvpc);
                if (v < nv) {
                    const int64_t e = s_ibase[v] + (((int64_t)j * src.jstride + s_ioff[v]) & src.wrap);
                    if (src.is_c64) {
                        const float2 f = __ldg(reinterpret_cast<const float2 *>(src.x) + e);
                        vals[u] = mk((double)f.x, (double)f.y);
                    } else {
                        vals[u] = ld_gather(reinterpret_cast<const cx *>(src.x) + e);
                    }
                    const int r = logL ? (int)(__brev((unsigned)j) >> (32 - logL)) : 0;
                    dst[u] = swz(v * L + r);
                }
            }
        }
#pragma unroll
        for (int u = 0; u < 8; u++)
            if (dst[u] >= 0) a[dst[u]] = vals[u];
    }
    __syncthreads();
    fft_stages_smem(a, nv, logL, 0, logL, tw);
    for (int i = threadIdx.x; i < nv * L; i += blockDim.x) epi(i >> logL, i & (L - 1), a[swz(i)]);
}

// Pass A of the large-view FFT: CTA (view g, block c) owns bit-reversed
// positions [c*P, (c+1)*P), i.e. inputs j = rev_P(i)*Q + rev_Q(c); it runs the
// first logP stages (all butterflies stay inside the block) unscaled.
static __global__ void k_fft_large_a(const ViewSrc src, int logL, int logP,
                                     const cx *__restrict__ tw, cx *__restrict__ scratch) {
    extern __shared__ double4 smem_raw[];
    cx *a = reinterpret_cast<cx *>(smem_raw);
    const int logQ = logL - logP, P = 1 << logP, Q = 1 << logQ;
    // views fastest: the CTAs of block c of all a signal's views run side by
    // side, and the views' shifts are adjacent samples of x, so one DRAM
    // line (128 B) serves every view's 16-B sample from L2 instead of being
    // fetched once per view (block c alone reads one sample per line)
    const int s = (int)(blockIdx.x % (unsigned)src.nshift);
    const int64_t rest = blockIdx.x / (unsigned)src.nshift;
    const int c = (int)(rest & (Q - 1));
    const int64_t b = rest >> logQ;
    const int64_t g = b * src.nshift + s;
    if (src.nview && s >= __ldg(src.nview + b)) return;   // unused view
    const int rc = logQ ? (int)(__brev((unsigned)c) >> (32 - logQ)) : 0;
    // block c of view g is itself a P-point view: input i of the block is
    // view sample rev_P(i)*Q + rc, i.e. stride Q*d from offset shift + rc*d
    __shared__ int64_t s_ib[1], s_io[1];
    if (threadIdx.x == 0) {
        const int64_t o = (s >= src.dyn_first) ? src.dyn_off[b * src.dyn_stride + (s - src.dyn_first)]
                                               : src.off[s];
        s_ib[0] = b * src.sig_stride;
        s_io[0] = o + (int64_t)rc * src.jstride;
    }
    __syncthreads();
    cx *dst = scratch + (g << logL) + ((int64_t)c << logP);
    fft_fused_views(a, src, src.jstride << logQ, s_ib, s_io, 1, 0, logP, tw,
                    [&](int, int k, cx y) { dst[k] = y; });
}

// large views (L > FFT_SMEM_MAX): stage split through global memory.
// Pass A (above) runs the first logP stages on contiguous blocks of P
// points in shared memory; the remaining stages act independently on the
// residue classes i mod P and run as register passes of <= 4 stages.
// Pass B in registers: LQ stages starting at stage s0 (half-size 2^s0) per
// kernel, LQ <= 4.  Thread = one (view, high index, residue r < 2^s0),
// holding the 2^LQ elements i = r + q*2^s0 + hi*2^(s0+LQ); the butterflies,
// their order within a stage and the twiddle index k = r + qk*2^s0 are those
// of the radix-2 stage loop, so the result is bit-identical.  Intermediate
// passes work in place on the scratch; the last writes the views (scaled,
// with the activity epilogue).  Loads/stores are coalesced across threads
// (consecutive residues).
template <int LQ>
static __global__ void __launch_bounds__(256) k_fft_large_b_reg(cx *buf, int64_t nviews, int logL, int s0,
                                                                const cx *__restrict__ tw, cx *out,
                                                                int nshift, int SV, int64_t ldV, int scale,
                                                                const double *__restrict__ thr,
                                                                uint8_t *__restrict__ act,
                                                                const int32_t *__restrict__ nview) {
    constexpr int Q = 1 << LQ;
    const int64_t P = int64_t(1) << s0;
    const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t g = gt >> (logL - LQ);
    if (g >= nviews) return;
    if (nview && (int)(g - (g / nshift) * nshift) >= __ldg(nview + g / nshift)) return;   // unused view
    const int64_t rem = gt & ((int64_t(1) << (logL - LQ)) - 1);
    const int64_t r = rem & (P - 1);
    const int64_t hi = rem >> s0;
    const int64_t i0 = r + (hi << (s0 + LQ));
    cx *src = buf + (g << logL) + i0;
    cx x[Q];
#pragma unroll
    for (int q = 0; q < Q; q++) x[q] = ldcx(src + (int64_t)q * P);
#pragma unroll
    for (int st = 0; st < LQ; st++) {
        const int hq = 1 << st;
        const int64_t h = P << st;
        const cx *twh = tw + (h - 1) + r;
#pragma unroll
        for (int qk = 0; qk < hq; qk++) {   // each distinct twiddle loaded once
            const cx w = ldcx(twh + qk * P);
#pragma unroll
            for (int q = qk; q < Q; q += 2 * hq) {
                const cx u = x[q];
                const cx t = gmul(x[q + hq], w);
                x[q] = cadd(u, t);
                x[q + hq] = csub(u, t);
            }
        }
    }
    if (out == nullptr) {   // intermediate pass: in place
#pragma unroll
        for (int q = 0; q < Q; q++) src[(int64_t)q * P] = x[q];
        return;
    }
    const double sc = 1.0 / (double)(int64_t(1) << logL);
    const int64_t b = g / nshift;
    const int s = (int)(g - b * nshift);
    cx *o = out + (b * SV + s) * ldV + i0;
    const double th = act ? thr[b] : 0.0;
#pragma unroll
    for (int q = 0; q < Q; q++) {
        const cx y = scale ? mk(DMUL(x[q].re, sc), DMUL(x[q].im, sc)) : x[q];
        stcx(o + (int64_t)q * P, y);
        if (act) {   // activity epilogue, as in k_fft_views
            const double m2 = y.re * y.re + y.im * y.im;
            if (m2 > th * th * (1.0 + 1e-6) || (m2 >= th * th * (1.0 - 1e-6) && cabs_i(y) > th))
                act[(b << logL) + i0 + (int64_t)q * P] = 1;
        }
    }
}


// ---------------------------------------------------------------------------
// Large views, register-blocked pass A (P = 4096 points, 12 stages): thread t
// of 256 holds 16 elements in registers through three radix-16 rounds --
// stages 0-3 on positions 16t + k, stages 4-7 on (t & 15) + 256 (t >> 4) +
// 16k, stages 8-11 on t + 256k -- with two shared-memory exchanges between
// them (XOR-swizzled: conflict-free in all three access patterns).  All 16
// strided gathers of a thread are in flight at once, and every group loads
// its 15 twiddles up front.  Butterflies, pairs and twiddles are those of the radix-2
// stage loop, so the blocks are bit-identical to k_fft_large_a's.
__device__ __forceinline__ int swz16(int p) { return p ^ ((p >> 4) & 7); }

__device__ __forceinline__ cx ld_stream(const cx *p) {   // no L1 allocation
    double2 v;
    asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
    return mk(v.x, v.y);
}

// FINAL (L = 4096 exactly, the block is the whole view): the last round's
// outputs go straight to the views with the scale / activity epilogue of
// k_fft_views -- at L = 4096 this register-blocked form replaces the four
// radix-8 shared-memory passes of k_fft_views<3> (two exchanges instead of
// three, every twiddle of a round loaded up front): config 4 view FFT
// 1044 -> 951 us, bit-identical.
template <bool FINAL>
static __global__ void __launch_bounds__(256, 2) k_fft_large_a16(const ViewSrc src, int logL,
                                                                 const cx *__restrict__ tw,
                                                                 cx *__restrict__ scratch, int SV, int64_t ldV,
                                                                 int scale, const double *__restrict__ thr,
                                                                 uint8_t *__restrict__ act) {
    pdl_wait();
    extern __shared__ double4 smem_raw[];
    cx *a = reinterpret_cast<cx *>(smem_raw);
    constexpr int logP = 12;
    const int logQ = logL - logP, Q = 1 << logQ;
    const int s = (int)(blockIdx.x % (unsigned)src.nshift);
    const int64_t rest = blockIdx.x / (unsigned)src.nshift;
    const int c = (int)(rest & (Q - 1));
    const int64_t b = rest >> logQ;
    if (src.nview && s >= __ldg(src.nview + b)) return;   // unused view
    const int t = threadIdx.x;
    const int rc = logQ ? (int)(__brev((unsigned)c) >> (32 - logQ)) : 0;
    const int64_t o = (s >= src.dyn_first) ? __ldg(src.dyn_off + b * src.dyn_stride + (s - src.dyn_first))
                                           : src.off[s];
    // position p of the block holds block input rev12(p), view sample
    // rev12(p)*Q + rc, i.e. x[(sample*d + shift) mod n]
    const int64_t ib = b * src.sig_stride, io = o + (int64_t)rc * src.jstride, js = src.jstride << logQ;
    const int rt = (int)(__brev((unsigned)t) >> 24);   // rev8(t)
    cx x[16];
#pragma unroll
    for (int k = 0; k < 16; k++) {
        const int k4 = (int)(__brev((unsigned)k) >> 28);   // rev4(k)
        const int64_t jb = (int64_t)(k4 * 256 + rt);
        const int64_t e = ib + ((jb * js + io) & src.wrap);
        if (src.is_c64) {
            const float2 f = __ldg(reinterpret_cast<const float2 *>(src.x) + e);
            x[k] = mk((double)f.x, (double)f.y);
        } else {
            // L1-allocating loads: the eight views' CTAs of a block share
            // each line through L2 (no_allocate measured 1.2-1.3x the DRAM
            // reads and 5 % slower, profiles/r02_large_fft/)
            x[k] = ldcx(reinterpret_cast<const cx *>(src.x) + e);
        }
    }
    group_stages_pre<4>(x, 0, 1, tw);                       // stages 0-3
#pragma unroll
    for (int k = 0; k < 16; k++) a[swz16(16 * t + k)] = x[k];
    __syncthreads();
    const int base2 = (t & 15) + ((t >> 4) << 8);
#pragma unroll
    for (int k = 0; k < 16; k++) x[k] = a[swz16(base2 + 16 * k)];
    group_stages_pre<4>(x, t & 15, 16, tw);                 // stages 4-7
#pragma unroll
    for (int k = 0; k < 16; k++) a[swz16(base2 + 16 * k)] = x[k];
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 16; k++) x[k] = a[swz16(t + 256 * k)];
    group_stages_pre<4>(x, t, 256, tw);                     // stages 8-11
    if constexpr (FINAL) {
        cx *dst = scratch + (b * SV + s) * ldV;   // `scratch` is the view array here
        const double sc = 1.0 / 4096.0;
        double th = 0.0, th2hi = 0.0, th2lo = 0.0;
        if (act) {
            th = thr[b];
            th2hi = th * th * (1.0 + 1e-6);
            th2lo = th * th * (1.0 - 1e-6);
        }
#pragma unroll
        for (int k = 0; k < 16; k++) {
            cx y = x[k];
            if (scale) y = mk(DMUL(y.re, sc), DMUL(y.im, sc));
            stcx(dst + t + 256 * k, y);
            if (act) {
                const double q = y.re * y.re + y.im * y.im;
                if (q > th2hi || (q >= th2lo && cabs_i(y) > th)) act[b * 4096 + t + 256 * k] = 1;
            }
        }
    } else {
        cx *dst = scratch + ((b * src.nshift + s) << logL) + ((int64_t)c << logP);
#pragma unroll
        for (int k = 0; k < 16; k++) stcx(dst + t + 256 * k, x[k]);
    }
}

// ---------------------------------------------------------------------------
// 4096-point views of the general path through a WINDOW RING (tuning
// gen_window > 0).  k_fft_large_a16<true> gathers view v of signal b itself:
// a warp instruction reads one sample from each of 32 different d-blocks, so
// every 16-B sample opens its own DRAM row (36 G random line fetches/s, the
// measured fully-random ceiling).  A d-block's samples of ALL the signal's
// views fetched by one warp instruction share that row: tools/blockgather.cu
// measures 61 G lines/s for this pattern with the 64-B fetch hint
// (profiles/r02_blockgather.txt).  Here each CTA does both jobs in turn:
//   1. gather piece `s` (d-block tiles s, s + nv, ...) of signal b + LOOK:
//      half-warps over d-blocks, lanes over the views, rows W[slot][m][0..16)
//      of 256 B written whole;
//   2. the FFT of view s of signal b, its samples read from the ring (L2).
// CTAs take a ticket in start order, so the pieces of signal b were taken by
// CTAs that started before any consumer of b and wait on nothing newer:
// waiting on `arrive[b]` (pieces written) and on `done[b - ring]` (ring slot
// drained) cannot deadlock.  Same butterflies and twiddles as every other
// form: bit-identical views.
// Default for HOST-MAPPED signals (the zero-copy end-to-end path: the six
// consecutive shifts of a d-block are one PCIe read request instead of six
// from six CTAs; config 4 e2e 6.36k -> 14.4k signals/s).  For signals in HBM it
// is measured slower and off (profiles/r02_window/): config 4 DRAM reads
// 4.72 -> 2.77 GB per launch, but 0.95 -> 1.55 ms -- at 2 CTAs per SM (128
// registers, 64 KiB) the gather piece and the FFT serialise inside a CTA
// (gather alone 1.18 ms in this structure vs 0.61 ms standalone; the FFT
// from the ring alone 0.67 ms).
__device__ __forceinline__ cx ld_win64(const cx *p) {   // gather load: no L1 allocation, 64-B L2 fetch
    double2 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::64B.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
    return mk(v.x, v.y);
}
__device__ __forceinline__ cx ld_win64(const float2 *p) {
    float2 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::64B.v2.f32 {%0,%1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(p));
    return mk((double)v.x, (double)v.y);
}
__device__ __forceinline__ cx ld_win(const cx *p) {   // the same without the fetch-size hint (host-mapped x)
    double2 v;
    asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
    return mk(v.x, v.y);
}
__device__ __forceinline__ cx ld_win(const float2 *p) {
    float2 v;
    asm volatile("ld.global.nc.L1::no_allocate.v2.f32 {%0,%1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(p));
    return mk((double)v.x, (double)v.y);
}
__device__ __forceinline__ int ld_acquire(const int *p) {
    int v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

constexpr int WIN_NVP = 16;   // views per ring row (nv <= 16)

static __global__ void __launch_bounds__(256, 2) k_fft_win16(const ViewSrc src, int64_t B, int look, int ring,
                                                             cx *__restrict__ W, int *__restrict__ flags,
                                                             const cx *__restrict__ tw, cx *__restrict__ out,
                                                             int SV, int64_t ldV, int scale, int hint64) {
    pdl_wait();
    extern __shared__ double4 smem_raw[];
    cx *a = reinterpret_cast<cx *>(smem_raw);
    __shared__ unsigned s_ticket;
    const int t = threadIdx.x;
    const int nv = src.nshift;
    int *ticket = flags, *arrive = flags + 1, *done = flags + 1 + B;
    if (t == 0) s_ticket = (unsigned)atomicAdd(ticket, 1);
    __syncthreads();
    const int64_t u = (int64_t)s_ticket - (int64_t)look * nv;   // < 0: prologue (gather only)
    const int64_t tk = s_ticket;
    const int64_t b = u >= 0 ? u / nv : -1;
    const int s = (int)(u >= 0 ? u - b * nv : tk % nv);
    const int64_t bg = u >= 0 ? b + look : tk / nv;             // signal whose piece s this CTA gathers
    constexpr int L = 4096, NT = L / 16;
    if (bg < B) {
        if (bg >= ring) {   // the slot's previous signal must be drained
            if (t == 0)
                while (ld_acquire(done + (bg - ring)) < nv) __nanosleep(64);
            __syncthreads();
        }
        const int v = t & 15, h = t >> 4;
        if (v < nv) {
            const int64_t o = (v >= src.dyn_first) ? __ldg(src.dyn_off + bg * src.dyn_stride + (v - src.dyn_first))
                                                   : src.off[v];
            const int64_t ib = bg * src.sig_stride;
            cx *wr = W + ((int64_t)(bg % ring) * L) * WIN_NVP + v;
            for (int i0 = 0; s + nv * i0 < NT; i0 += 8) {
                cx val[8];
#pragma unroll
                for (int q = 0; q < 8; q++) {
                    const int tau = s + nv * (i0 + q);
                    if (tau < NT) {
                        const int64_t m = tau * 16 + h;
                        const int64_t e = ib + ((m * src.jstride + o) & src.wrap);
                        if (hint64)
                            val[q] = src.is_c64 ? ld_win64(reinterpret_cast<const float2 *>(src.x) + e)
                                                : ld_win64(reinterpret_cast<const cx *>(src.x) + e);
                        else
                            val[q] = src.is_c64 ? ld_win(reinterpret_cast<const float2 *>(src.x) + e)
                                                : ld_win(reinterpret_cast<const cx *>(src.x) + e);
                    }
                }
#pragma unroll
                for (int q = 0; q < 8; q++) {
                    const int tau = s + nv * (i0 + q);
                    if (tau < NT) stcx(wr + (int64_t)(tau * 16 + h) * WIN_NVP, val[q]);
                }
            }
        }
        __threadfence();
        __syncthreads();
        if (t == 0) {
            __threadfence();
            atomicAdd(arrive + bg, 1);
        }
    }
    if (b < 0) return;
    if (src.nview && s >= __ldg(src.nview + b)) {   // unused view: nothing to read from the slot
        if (t == 0) atomicAdd(done + b, 1);
        return;
    }
    if (t == 0)
        while (ld_acquire(arrive + b) < nv) __nanosleep(64);
    __syncthreads();
    const cx *ws = W + ((int64_t)(b % ring) * L) * WIN_NVP + s;
    const int rt = (int)(__brev((unsigned)t) >> 24);   // rev8(t)
    cx x[16];
#pragma unroll
    for (int k = 0; k < 16; k++) {
        const int k4 = (int)(__brev((unsigned)k) >> 28);   // rev4(k)
        const double2 w2 = __ldcg(reinterpret_cast<const double2 *>(ws + (int64_t)(k4 * 256 + rt) * WIN_NVP));
        x[k] = mk(w2.x, w2.y);
    }
    group_stages_pre<4>(x, 0, 1, tw);                       // stages 0-3
#pragma unroll
    for (int k = 0; k < 16; k++) a[swz16(16 * t + k)] = x[k];
    __syncthreads();
    if (t == 0) atomicAdd(done + b, 1);   // every thread's ring loads have landed
    const int base2 = (t & 15) + ((t >> 4) << 8);
#pragma unroll
    for (int k = 0; k < 16; k++) x[k] = a[swz16(base2 + 16 * k)];
    group_stages_pre<4>(x, t & 15, 16, tw);                 // stages 4-7
#pragma unroll
    for (int k = 0; k < 16; k++) a[swz16(base2 + 16 * k)] = x[k];
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 16; k++) x[k] = a[swz16(t + 256 * k)];
    group_stages_pre<4>(x, t, 256, tw);                     // stages 8-11
    cx *dst = out + (b * SV + s) * ldV;
    const double sc = 1.0 / 4096.0;
#pragma unroll
    for (int k = 0; k < 16; k++) {
        cx y = x[k];
        if (scale) y = mk(DMUL(y.re, sc), DMUL(y.im, sc));
        stcx(dst + t + 256 * k, y);
    }
}

// ring bytes / flag bytes of the window path for B signals (0: not applicable)
static inline bool win_applicable(int64_t B, int64_t L, int nshift, int look) {
    return look > 0 && L == 4096 && nshift <= WIN_NVP && B >= 4 * (int64_t)look;
}
static inline size_t win_ring_bytes(int look) { return size_t(2 * look) * 4096 * WIN_NVP * 16; }
static inline size_t win_flag_bytes(int64_t B) { return size_t(2 * B + 1) * 4; }

static inline int launch_fft_win16(const ViewSrc &src, int64_t B, const double *tw_, cx *out, int SV, int64_t ldV,
                                   cudaStream_t stream, int look, cx *ring, int *flags, int hint64, int scale = 1) {
    const cx *tw = reinterpret_cast<const cx *>(tw_);
    const size_t smem = size_t(4096) * 16;
    cudaMemsetAsync(flags, 0, win_flag_bytes(B), stream);
    cudaFuncSetAttribute(k_fft_win16, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_fft_win16, cudaFuncAttributePreferredSharedMemoryCarveout,
                         (int)((2 * (smem + 1024) * 100 + 228 * 1024 - 1) / (228 * 1024)));
    const int64_t grid = (B + look) * src.nshift;
    k_fft_win16<<<(unsigned)grid, 256, smem, stream>>>(src, B, look, 2 * look, ring, flags, tw, out, SV, ldV, scale, hint64);
    SFDT_CHECK_LAUNCH();
    return SFDT_OK;
}

// Large views, register-blocked pass B: the LQ (5..7) stages left after pass
// A act on the columns i = r + q*P (P = 2^(logL-LQ)) of each residue r.  A
// CTA of 32 * 2^(LQ-4) threads owns 32 consecutive residues of one view:
// thread (lane = residue, w) loads elements q = 16w + k of its column
// straight into registers (each row 32 residues = 512 contiguous bytes),
// runs column stages 0-3 as one radix-16 group, exchanges through shared
// memory once, runs the remaining LQ-4 stages as radix-2^(LQ-4) groups and
// writes the view (scale / activity epilogue) -- one read and one write of
// the scratch for all remaining stages.  Bit-identical to the register
// passes (same butterflies, pairs, twiddles tw[(H-1) + (i mod H)]).
template <int LQ>
static __global__ void __launch_bounds__(32 << (LQ - 4), 16 >> (LQ - 4)) k_fft_large_b16(
    const cx *__restrict__ buf, int64_t nviews, int logL, const cx *__restrict__ tw, cx *out, int nshift, int SV,
    int64_t ldV, int scale, const double *__restrict__ thr, uint8_t *__restrict__ act,
    const int32_t *__restrict__ nview) {
    constexpr int R2 = LQ - 4, G2 = 1 << R2, NT = 32 << R2;
    extern __shared__ double4 smem_raw[];
    cx *tile = reinterpret_cast<cx *>(smem_raw);   // [q][residue], 2^LQ x 32
    const int s0 = logL - LQ;
    const int64_t P = int64_t(1) << s0;
    const int64_t tiles = P >> 5;
    const int64_t g = blockIdx.x / tiles;
    const int64_t r0 = (blockIdx.x - g * tiles) << 5;
    const int64_t b = g / nshift;
    const int s = (int)(g - b * nshift);
    if (nview && s >= __ldg(nview + b)) return;   // unused view
    const int rl = threadIdx.x & 31, w = threadIdx.x >> 5;
    const cx *src = buf + (g << logL) + r0 + rl;
    cx x[16];
#pragma unroll
    for (int k = 0; k < 16; k++) x[k] = ld_stream(src + (int64_t)(16 * w + k) * P);
    // column stages 0-3: element q = 16w + k is i = r + q*P, so the group has
    // stride h = P and i mod P = r
    // (twiddles per stage, not all 15 up front: that spills at 128 registers)
    group_stages<4>(x, (int)(r0 + rl), (int)P, tw);
#pragma unroll
    for (int k = 0; k < 16; k++) tile[(16 * w + k) * 32 + rl] = x[k];
    __syncthreads();
    const double sc = 1.0 / (double)(int64_t(1) << logL);
    const double th = act ? thr[b] : 0.0;
    cx *o = out + (b * SV + s) * ldV + r0 + rl;
    // column stages 4 .. LQ-1: groups q = qb + 16k (qb < 16), 16 / G2 per thread
#pragma unroll
    for (int u = 0; u < 16 / G2; u++) {
        const int qb = u * (NT / 32) + w;   // this thread's u-th group base (0..15)
        cx y[G2];
#pragma unroll
        for (int k = 0; k < G2; k++) y[k] = tile[(qb + 16 * k) * 32 + rl];
        group_stages_pre<R2>(y, (int)(r0 + rl + (int64_t)qb * P), (int)(P << 4), tw);
#pragma unroll
        for (int k = 0; k < G2; k++) {
            const int64_t i = (int64_t)(qb + 16 * k) * P;
            const cx v = scale ? mk(DMUL(y[k].re, sc), DMUL(y[k].im, sc)) : y[k];
            stcx(o + i, v);
            if (act) {
                const double m2 = v.re * v.re + v.im * v.im;
                if (m2 > th * th * (1.0 + 1e-6) || (m2 >= th * th * (1.0 - 1e-6) && cabs_i(v) > th))
                    act[(b << logL) + r0 + rl + i] = 1;
            }
        }
    }
}

template <int LQ>
static inline void launch_large_b_reg(cx *buf, int64_t nviews, int logL, int s0, const cx *tw, cx *out,
                                      int nshift, int SV, int64_t ldV, int scale, const double *thr,
                                      uint8_t *act, cudaStream_t stream, const int32_t *nview) {
    const int64_t threads = nviews << (logL - LQ);
    k_fft_large_b_reg<LQ><<<(unsigned)((threads + 255) / 256), 256, 0, stream>>>(
        buf, nviews, logL, s0, tw, out, nshift, SV, ldV, scale, thr, act, nview);
}

// Large views (L > FFT_SMEM_MAX): pass A runs the first LARGE_LOGP stages on
// 4096-point blocks; the remaining stages act on the residue classes mod
// 4096.  5..7 remaining stages (L = 2^17 .. 2^19): register-blocked
// k_fft_large_a16 + one k_fft_large_b16.  Other large L: k_fft_large_a16 +
// register passes of <= 4 stages.  With `split` (the round-1 plan, kept for
// A/B runs and tests): k_fft_large_a + register passes of <= 4 stages.
constexpr int LARGE_LOGP = 12;
static inline int large_logp(int logL) { return LARGE_LOGP < logL ? LARGE_LOGP : logL - 1; }
static inline bool large_blocked(int logL, int split) {   // split: sfdt_tuning.fft_split (bit 0 here)
    const int lq = logL - LARGE_LOGP;
    return !(split & 1) && lq >= 5 && lq <= 7;
}
static inline int large_next(int logL, int s0) {
    const int rem = logL - s0;
    return rem <= 0 ? 0 : (rem >= 4 ? 4 : rem);
}

// kernel launches of one launch_fft_views call
static inline int fft_view_launches(int64_t L, int split = 0) {
    if (L <= FFT_SMEM_MAX) return 1;
    const int logL = ilog2_64(L);
    if (large_blocked(logL, split)) return 2;
    int s0 = large_logp(logL), n = 1;
    for (int k; (k = large_next(logL, s0)) > 0; s0 += k) n++;
    return n;
}

// FFT of every view of B signals; large_scratch (B*nshift*L complex) is
// needed only when L > FFT_SMEM_MAX.
static inline int launch_fft_views(const ViewSrc &src, int64_t B, int64_t L, const double *tw_,
                                   cx *out, int SV, int64_t ldV, cudaStream_t stream,
                                   cx *large_scratch = nullptr, int scale = 1,
                                   const double *thr = nullptr, uint8_t *act = nullptr, int split = 0) {
    const cx *tw = reinterpret_cast<const cx *>(tw_);
    const int logL = ilog2_64(L);
    const int64_t nviews = B * src.nshift;
    if (nviews == 0) return SFDT_OK;
    if (logL == 12 && !src.jfast && !(split & 2)) {
        // 4096-point views: the register-blocked radix-16 form
        const size_t smem = size_t(4096) * 16;
        cudaFuncSetAttribute(k_fft_large_a16<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(k_fft_large_a16<true>, cudaFuncAttributePreferredSharedMemoryCarveout,
                             (int)((2 * (smem + 1024) * 100 + 228 * 1024 - 1) / (228 * 1024)));
        launch_pdl(k_fft_large_a16<true>, dim3((unsigned)nviews), dim3(256), smem, stream, src, logL, tw, out, SV, ldV,
                   scale, thr, act);
        SFDT_CHECK_LAUNCH();
        return SFDT_OK;
    }
    if (L <= FFT_SMEM_MAX) {
        int logvpc = 0;
        // views per CTA: up to 2048 points, but small batches keep >= 2 CTAs
        // per SM instead of packing views (config 1: 8 CTAs of one view
        // rather than one CTA of eight)
        while ((L << (logvpc + 1)) <= 2048 && (1 << (logvpc + 1)) <= 2 * src.nshift &&
               (nviews >> (logvpc + 1)) >= 296)
            logvpc++;
        const size_t smem = (size_t(L) << logvpc) * 16;
        const unsigned grid = (unsigned)((nviews + (1 << logvpc) - 1) >> logvpc);
        // <= 32 KiB per CTA: cap registers at 64 for 4 CTAs/SM (measured
        // 717 -> 553 us at config 2); larger tiles keep 128 registers
        if (smem <= 32 * 1024) {
            launch_pdl(k_fft_views<4>, dim3(grid), dim3(256), smem, stream, src, B, logL, logvpc, tw, out, SV, ldV,
                       scale, thr, act);
        } else if (smem <= 64 * 1024) {
            // 64 KiB tiles: registers capped at 85 (3 CTAs/SM would fit).
            // Two CTAs per SM, the rest of the 256 KiB as L1: the view
            // stages read the (L-1)-entry twiddle table (64 KiB at L = 4096)
            // through L1, and with 3 CTAs' 192 KiB of smem it thrashed into
            // L2 (7.2 GB of L2 reads per config-4 batch; 4.78 -> 4.20 ms).
            cudaFuncSetAttribute(k_fft_views<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            cudaFuncSetAttribute(k_fft_views<3>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                 (int)((2 * (smem + 1024) * 100 + 228 * 1024 - 1) / (228 * 1024)));
            launch_pdl(k_fft_views<3>, dim3(grid), dim3(256), smem, stream, src, B, logL, logvpc, tw, out, SV, ldV,
                       scale, thr, act);
        } else {
            cudaFuncSetAttribute(k_fft_views<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            launch_pdl(k_fft_views<1>, dim3(grid), dim3(256), smem, stream, src, B, logL, logvpc, tw, out, SV, ldV,
                       scale, thr, act);
        }
        SFDT_CHECK_LAUNCH();
        return SFDT_OK;
    }
    if (!large_scratch) return SFDT_EINVAL;
    const int logP = large_logp(logL), P = 1 << logP;
    const int logQ = logL - logP;
    if (large_blocked(logL, split)) {
        // pass A: 4096-point blocks in registers (three radix-16 rounds)
        const size_t smem = size_t(P) * 16;
        cudaFuncSetAttribute(k_fft_large_a16<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(k_fft_large_a16<false>, cudaFuncAttributePreferredSharedMemoryCarveout,
                             (int)((2 * (smem + 1024) * 100 + 228 * 1024 - 1) / (228 * 1024)));
        k_fft_large_a16<false><<<(unsigned)(nviews << logQ), 256, smem, stream>>>(src, logL, tw, large_scratch, 0, 0,
                                                                                 0, nullptr, nullptr);
        SFDT_CHECK_LAUNCH();
        // pass B: every remaining stage in one register-blocked pass
        const int lq = logL - logP;
        const int64_t ctas = nviews * ((int64_t(1) << (logL - lq)) >> 5);
        auto pass_b = [&](auto lq_c) {
            constexpr int LQ = decltype(lq_c)::value;
            cudaFuncSetAttribute(k_fft_large_b16<LQ>, cudaFuncAttributeMaxDynamicSharedMemorySize, 512 << LQ);
            k_fft_large_b16<LQ><<<(unsigned)ctas, 32 << (LQ - 4), 512 << LQ, stream>>>(
                large_scratch, nviews, logL, tw, out, src.nshift, SV, ldV, scale, thr, act, src.nview);
        };
        if (lq == 5) pass_b(std::integral_constant<int, 5>{});
        else if (lq == 6) pass_b(std::integral_constant<int, 6>{});
        else pass_b(std::integral_constant<int, 7>{});
        SFDT_CHECK_LAUNCH();
        return SFDT_OK;
    }
    if (!(split & 1) && logP == LARGE_LOGP) {
        // other large L (2^13..2^16, >= 2^20): the register-blocked pass A,
        // then register passes of <= 4 stages
        const size_t smem = size_t(P) * 16;
        cudaFuncSetAttribute(k_fft_large_a16<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(k_fft_large_a16<false>, cudaFuncAttributePreferredSharedMemoryCarveout,
                             (int)((2 * (smem + 1024) * 100 + 228 * 1024 - 1) / (228 * 1024)));
        k_fft_large_a16<false><<<(unsigned)(nviews << logQ), 256, smem, stream>>>(src, logL, tw, large_scratch, 0, 0,
                                                                                 0, nullptr, nullptr);
        SFDT_CHECK_LAUNCH();
    } else {
        const size_t smem = size_t(P) * 16;
        cudaFuncSetAttribute(k_fft_large_a, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        // 2 CTAs/SM at 4096 points (4 at 2048), the rest L1 for the
        // (P-1)-entry twiddle table (as above)
        const int ctas = logP >= 12 ? 2 : 4;
        cudaFuncSetAttribute(k_fft_large_a, cudaFuncAttributePreferredSharedMemoryCarveout,
                             (int)((ctas * (smem + 1024) * 100 + 228 * 1024 - 1) / (228 * 1024)));
        k_fft_large_a<<<(unsigned)(nviews << logQ), 256, smem, stream>>>(src, logL, logP, tw, large_scratch);
        SFDT_CHECK_LAUNCH();
    }
    // remaining stages logP .. logL-1 (the last pass writes the views)
    for (int s0 = logP, lq; (lq = large_next(logL, s0)) > 0; s0 += lq) {
        cx *o = (s0 + lq == logL) ? out : nullptr;
        switch (lq) {
        case 1: launch_large_b_reg<1>(large_scratch, nviews, logL, s0, tw, o, src.nshift, SV, ldV, scale, thr, act, stream, src.nview); break;
        case 2: launch_large_b_reg<2>(large_scratch, nviews, logL, s0, tw, o, src.nshift, SV, ldV, scale, thr, act, stream, src.nview); break;
        case 3: launch_large_b_reg<3>(large_scratch, nviews, logL, s0, tw, o, src.nshift, SV, ldV, scale, thr, act, stream, src.nview); break;
        default: launch_large_b_reg<4>(large_scratch, nviews, logL, s0, tw, o, src.nshift, SV, ldV, scale, thr, act, stream, src.nview); break;
        }
        SFDT_CHECK_LAUNCH();
    }
    return SFDT_OK;
}

// Host-mapped signals, any L: the window gather as its own kernel.  Half-
// warps (quarter-... 256 >> lognvp groups) over d-blocks, lanes over the
// views, rows W[b][m][0..nvp) written whole to device memory; the ordinary
// view FFT then reads W (ViewSrc: sample j of view v at (b*L + j)*nvp + v).
// Over PCIe this is 1 + r_eff read requests per d-block instead of
// 2*a_max + r_eff issued from as many different CTAs.
static __global__ void __launch_bounds__(256) k_win_gather(const ViewSrc src, int64_t nsig, int64_t L, int lognvp,
                                                           cx *__restrict__ W, int hint64) {
    constexpr int U = 8;
    const int nvp = 1 << lognvp, per = 256 >> lognvp;   // d-blocks per CTA step
    const int t = threadIdx.x, v = t & (nvp - 1), h = t >> lognvp;
    if (v >= src.nshift) return;
    // persistent: CTA c walks the tiles c, c + grid, ... of the (signal, tile) list in order
    const int64_t tiles = (L + per * U - 1) / (per * U);
    for (int64_t item = blockIdx.x; item < tiles * nsig; item += gridDim.x) {
    const int64_t b = item / tiles, tile = item - b * tiles;
    const int64_t o = (v >= src.dyn_first) ? __ldg(src.dyn_off + b * src.dyn_stride + (v - src.dyn_first))
                                           : src.off[v];
    const int64_t ib = b * src.sig_stride;
    cx *wr = W + ((b * L) << lognvp) + v;
    const int64_t m0 = tile * per * U + h;
    cx val[U];
#pragma unroll
    for (int q = 0; q < U; q++) {
        const int64_t m = m0 + (int64_t)q * per;
        if (m < L) {
            const int64_t e = ib + ((m * src.jstride + o) & src.wrap);
            if (hint64)
                val[q] = src.is_c64 ? ld_win64(reinterpret_cast<const float2 *>(src.x) + e)
                                    : ld_win64(reinterpret_cast<const cx *>(src.x) + e);
            else
                val[q] = src.is_c64 ? ld_win(reinterpret_cast<const float2 *>(src.x) + e)
                                    : ld_win(reinterpret_cast<const cx *>(src.x) + e);
        }
    }
#pragma unroll
    for (int q = 0; q < U; q++) {
        const int64_t m = m0 + (int64_t)q * per;
        if (m < L) stcx(wr + (m << lognvp), val[q]);
    }
    }
}

static inline int win_lognvp(int nshift) { return nshift <= 16 ? 4 : 5; }
static inline size_t win_gather_bytes(int64_t B, int64_t L, int nshift) {
    return (size_t(B) * L << win_lognvp(nshift)) * 16;
}

// gather (above) + the ordinary view FFT from the window buffer
static inline int launch_fft_from_window(const ViewSrc &src, int64_t B, int64_t L, const double *tw_, cx *out,
                                         int SV, int64_t ldV, cudaStream_t stream, cx *W, cx *large_scratch,
                                         int hint64, int split) {
    const int lognvp = win_lognvp(src.nshift);
    const int per = 256 >> lognvp;
    // a persistent grid of half the SMs: over PCIe fewer gathers in flight keep
    // the read requests closer to address order -- measured 74 CTAs vs one per
    // tile: config 4 12.4k -> 13.8k, config 5 general K = 64 9.8k -> 12.2k,
    // K = 1024 2.10k -> 2.35k signals/s end to end; 37 CTAs starve the link at
    // L = 32768 (1.6k) (profiles/r02_window/e2e.txt)
    const int64_t items = ((L + per * 8 - 1) / (per * 8)) * B;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int64_t g = sms / 2 > 0 ? sms / 2 : 1;
    if (g > items) g = items;
    k_win_gather<<<(unsigned)g, 256, 0, stream>>>(src, B, L, lognvp, W, hint64);
    SFDT_CHECK_LAUNCH();
    ViewSrc ws;
    ws.x = W;
    ws.is_c64 = 0;
    ws.nshift = src.nshift;
    ws.sig_stride = L << lognvp;
    ws.jstride = int64_t(1) << lognvp;
    ws.wrap = (L << lognvp) - 1;
    for (int v = 0; v < MAX_VIEWS; v++) ws.off[v] = v;
    ws.dyn_off = nullptr;
    ws.dyn_first = MAX_VIEWS;
    ws.dyn_stride = 0;
    ws.jfast = 0;
    ws.nview = src.nview;
    return launch_fft_views(ws, B, L, tw_, out, SV, ldV, stream, large_scratch, 1, nullptr, nullptr, split);
}

static inline ViewSrc consecutive_views(const void *x, int is_c64, int64_t n, int64_t d, int shift0,
                                        int nshift) {
    ViewSrc s;
    s.x = x;
    s.is_c64 = is_c64;
    s.nshift = nshift;
    s.sig_stride = n;
    s.jstride = d;
    s.wrap = n - 1;
    for (int v = 0; v < MAX_VIEWS; v++) s.off[v] = (v < nshift) ? shift0 + v : 0;
    s.dyn_off = nullptr;
    s.dyn_first = MAX_VIEWS;
    s.dyn_stride = 0;
    s.jfast = 0;
    s.nview = nullptr;
    return s;
}

}  // namespace sfdt
