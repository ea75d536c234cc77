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
// Layout: input view v of signal b is the strided column
//   win[(b*Lw + j*rowstride)*S + shift0 + v],  j < L
// of the (B, Lw, S) window buffer written by k_stream; output goes to
//   out[(b*SV + v)*ldV + k].
#pragma once

#include "common.cuh"

namespace sfdt {

static __global__ void k_fft_views(const cx *__restrict__ win, int64_t B, int64_t Lw, int S,
                            int64_t rowstride, int shift0, int nshift, int logL, int vpc,
                            const cx *__restrict__ tw, cx *__restrict__ out, int SV, int64_t ldV,
                            int inverse_scale) {
    extern __shared__ double4 smem_raw[];
    cx *a = reinterpret_cast<cx *>(smem_raw);
    const int L = 1 << logL;
    const int64_t nviews = B * nshift;
    const int64_t g0 = int64_t(blockIdx.x) * vpc;
    const int nv = (int)((nviews - g0) < vpc ? (nviews - g0) : vpc);
    // load with bit reversal
    for (int i = threadIdx.x; i < nv * L; i += blockDim.x) {
        const int v = i >> logL, j = i & (L - 1);
        const int64_t g = g0 + v;
        const int64_t b = g / nshift;
        const int s = (int)(g - b * nshift);
        const int r = logL ? (int)(__brev((unsigned)j) >> (32 - logL)) : 0;
        a[v * L + r] = ldcx(win + (b * Lw + j * rowstride) * S + shift0 + s);
    }
    __syncthreads();
    const int nbf = nv * (L >> 1);
    for (int lh = 0; lh < logL; lh++) {
        const int h = 1 << lh;   // half of the stage length m = 2h
        const cx *twh = tw + (h - 1);
        for (int t = threadIdx.x; t < nbf; t += blockDim.x) {
            const int v = t >> (logL - 1);
            const int tt = t & ((L >> 1) - 1);
            const int k = tt & (h - 1);
            const int i0 = v * L + ((tt >> lh) << (lh + 1)) + k;
            const cx u = a[i0];
            const cx x = gmul(a[i0 + h], ldcx(twh + k));
            a[i0] = cadd(u, x);
            a[i0 + h] = csub(u, x);
        }
        __syncthreads();
    }
    const double sc = 1.0 / (double)L;   // exact power of two
    for (int i = threadIdx.x; i < nv * L; i += blockDim.x) {
        const int v = i >> logL, k = i & (L - 1);
        const int64_t g = g0 + v;
        const int64_t b = g / nshift;
        const int s = (int)(g - b * nshift);
        cx y = a[i];
        if (inverse_scale) y = mk(DMUL(y.re, sc), DMUL(y.im, sc));
        stcx(out + (b * SV + s) * ldV + k, y);
    }
}

// Pass A of the large-view FFT: CTA (view g, block c) owns bit-reversed
// positions [c*P, (c+1)*P), i.e. inputs j = rev_P(i)*Q + rev_Q(c); it runs the
// first logP stages (all butterflies stay inside the block) unscaled.
static __global__ void k_fft_large_a(const cx *__restrict__ win, int64_t B, int64_t Lw, int S,
                              int64_t rowstride, int shift0, int nshift, int logL, int logP,
                              const cx *__restrict__ tw, cx *__restrict__ scratch) {
    extern __shared__ double4 smem_raw[];
    cx *a = reinterpret_cast<cx *>(smem_raw);
    const int logQ = logL - logP, P = 1 << logP, Q = 1 << logQ;
    const int64_t g = blockIdx.x >> logQ;
    const int c = (int)(blockIdx.x & (Q - 1));
    const int64_t b = g / nshift;
    const int s = (int)(g - b * nshift);
    const int rc = logQ ? (int)(__brev((unsigned)c) >> (32 - logQ)) : 0;
    for (int i = threadIdx.x; i < P; i += blockDim.x) {
        const int64_t j = (int64_t)(__brev((unsigned)i) >> (32 - logP)) * Q + rc;
        a[i] = ldcx(win + (b * Lw + j * rowstride) * S + shift0 + s);
    }
    __syncthreads();
    for (int lh = 0; lh < logP; lh++) {
        const int h = 1 << lh;
        const cx *twh = tw + (h - 1);
        for (int t = threadIdx.x; t < (P >> 1); t += blockDim.x) {
            const int k = t & (h - 1);
            const int i0 = ((t >> lh) << (lh + 1)) + k;
            const cx u = a[i0];
            const cx x = gmul(a[i0 + h], ldcx(twh + k));
            a[i0] = cadd(u, x);
            a[i0 + h] = csub(u, x);
        }
        __syncthreads();
    }
    cx *dst = scratch + (g << logL) + ((int64_t)c << logP);
    for (int i = threadIdx.x; i < P; i += blockDim.x) dst[i] = a[i];
}

// large views (L > FFT_SMEM_MAX): stage split through global memory.
// Pass A runs the first logP stages on contiguous blocks of P points (in
// smem); pass B runs the remaining stages, which act independently on the
// residue classes i mod P, on tiles of R residues x Q = L/P rows.
static __global__ void k_fft_large_b(cx *__restrict__ buf, int64_t nviews, int logL, int logP, int logR,
                              const cx *__restrict__ tw, cx *__restrict__ out, int nshift, int SV,
                              int64_t ldV) {
    extern __shared__ double4 smem_raw[];
    cx *a = reinterpret_cast<cx *>(smem_raw);
    const int L = 1 << logL, P = 1 << logP, R = 1 << logR;
    const int logQ = logL - logP, Q = 1 << logQ;
    const int tiles_per_view = P >> logR;
    const int64_t g = blockIdx.x / tiles_per_view;
    const int r0 = (int)(blockIdx.x % tiles_per_view) * R;
    cx *src = buf + g * L;
    // tile element (q, rr) <-> global index r0 + rr + P*q ; smem [q*R + rr]
    for (int i = threadIdx.x; i < Q * R; i += blockDim.x) {
        const int q = i >> logR, rr = i & (R - 1);
        a[i] = src[r0 + rr + (int64_t)q * P];
    }
    __syncthreads();
    for (int lh = logP; lh < logL; lh++) {
        const int hq = 1 << (lh - logP);   // half in units of q
        const int h = 1 << lh;
        const cx *twh = tw + (h - 1);
        for (int t = threadIdx.x; t < (Q >> 1) * R; t += blockDim.x) {
            const int rr = t & (R - 1);
            const int tq = t >> logR;                      // butterfly index over q
            const int qk = tq & (hq - 1);
            const int q0 = ((tq >> (lh - logP)) << (lh - logP + 1)) + qk;
            const int k = r0 + rr + qk * P;                 // position within the stage block
            const int i0 = q0 * R + rr, i1 = (q0 + hq) * R + rr;
            const cx u = a[i0];
            const cx x = gmul(a[i1], ldcx(twh + k));
            a[i0] = cadd(u, x);
            a[i1] = csub(u, x);
        }
        __syncthreads();
    }
    const double sc = 1.0 / (double)L;
    const int64_t b = g / nshift;
    const int s = (int)(g - b * nshift);
    for (int i = threadIdx.x; i < Q * R; i += blockDim.x) {
        const int q = i >> logR, rr = i & (R - 1);
        const cx y = a[i];
        stcx(out + (b * SV + s) * ldV + r0 + rr + (int64_t)q * P, mk(DMUL(y.re, sc), DMUL(y.im, sc)));
    }
}

static inline int launch_fft_views(const cx *win, int64_t B, int64_t Lw, int S, int64_t rowstride,
                                   int shift0, int nshift, int64_t L, const double *tw_,
                                   cx *out, int SV, int64_t ldV, cudaStream_t stream,
                                   cx *large_scratch = nullptr) {
    const cx *tw = reinterpret_cast<const cx *>(tw_);
    const int logL = ilog2_64(L);
    const int64_t nviews = B * nshift;
    if (L <= FFT_SMEM_MAX) {
        int vpc = (int)(4096 / L);
        if (vpc < 1) vpc = 1;
        if (vpc > nshift * 4) vpc = nshift * 4;
        const size_t smem = size_t(vpc) * L * 16;
        if (smem > 48 * 1024)
            cudaFuncSetAttribute(k_fft_views, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        const unsigned grid = (unsigned)((nviews + vpc - 1) / vpc);
        k_fft_views<<<grid, 256, smem, stream>>>(win, B, Lw, S, rowstride, shift0, nshift, logL, vpc,
                                                 tw, out, SV, ldV, 1);
        SFDT_CHECK_LAUNCH();
        return SFDT_OK;
    }
    if (!large_scratch) return SFDT_EINVAL;
    // pass A: first logP stages, unscaled, into scratch (nviews, L)
    const int logP = 12, P = 1 << logP;
    {
        // reuse k_fft_views on P-point blocks: view g's block c = bit-reversed
        // positions [c*P, (c+1)*P) hold inputs j with rev(j) in that range,
        // i.e. j = c' + (L/P)*i with c' = rev_{logQ}(c)
        const int logQ = logL - logP;
        const size_t smem = size_t(P) * 16;
        cudaFuncSetAttribute(k_fft_large_a, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        const unsigned grid = (unsigned)(nviews << logQ);
        k_fft_large_a<<<grid, 256, smem, stream>>>(win, B, Lw, S, rowstride, shift0, nshift, logL,
                                                   logP, tw, large_scratch);
        SFDT_CHECK_LAUNCH();
    }
    {
        const int logQ = logL - logP;
        int logR = 13 - logQ;          // tile of 2^13 points
        if (logR > logP) logR = logP;
        if (logR < 0) return SFDT_EINVAL;
        const size_t smem = (size_t(1) << (logQ + logR)) * 16;
        cudaFuncSetAttribute(k_fft_large_b, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        const unsigned grid = (unsigned)(nviews * (P >> logR));
        k_fft_large_b<<<grid, 256, smem, stream>>>(large_scratch, nviews, logL, logP, logR, tw, out,
                                                   nshift, SV, ldV);
        SFDT_CHECK_LAUNCH();
    }
    return SFDT_OK;
}

}  // namespace sfdt
