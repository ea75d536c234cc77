// exact.cu -- sm_100a kernels of the exactly-K-sparse path.
//
//   k_sumsq        the one HBM pass over x: per-chunk sum |x|^2 (the rms of
//                  exact.py:176/215).  The only kernel that touches all of
//                  x; HBM roofline = 16 B per sample (8 B complex64).
//   k_rms          deterministic tree over the chunk partials -> rms, zero
//                  threshold zero_threshold*rms*d.
//   k_fft_views    gathers the 2*a_max shifted views x[d*j + s] straight from
//                  x (spectral.py:151-160) and runs the batched radix-2 DIT
//                  FFT in shared memory with the reference's exact butterfly
//                  arithmetic (fft.cuh).
//   k_decode_a1 / k_decode_multi  thread-per-bin non-iterative decode
//                  (exact.py:184-192): a = 1 for every bin, then a worklist
//                  of the bins that need a >= 2.
//   k_iter_pass    one pass l of the iterative solver (exact.py:223-285):
//                  fold, SubFreq, activation, descending-a decode with
//                  retry/deferral, per-bin subtraction of accepted terms.
//   compaction     per-signal scans -> compact (loc, value) lists in the
//                  reference's dict insertion order.
#include "common.cuh"
#include "decode.cuh"
#include "decode_coop.cuh"
#include "fft.cuh"
#ifdef SFDT_MULTI_PROFILE
#include <cstdio>
#endif

namespace sfdt {

// The non-iterative decode's per-solve scratch -- the activity flags of
// the signal's bins and the two worklist counters -- is zeroed by the rms
// kernel that precedes the FFT (instead of memset nodes, which would break
// the programmatic-dependent-launch chain of the latency path).
struct DecodeScratch {
    uint8_t *act;               // (B, L) activity flags, or nullptr
    int64_t L;
    unsigned long long *cnt0;   // worklist counters (zeroed by signal 0)
    unsigned long long *cnt1;
    unsigned long long *cnt2;
};

__device__ __forceinline__ void zero_scratch(const DecodeScratch &z, int64_t b, int lane, int nlanes) {
    if (z.act) {
        uint8_t *row = z.act + b * z.L;
        if ((z.L & 15) == 0)
            for (int64_t i = lane; i < (z.L >> 4); i += nlanes) reinterpret_cast<uint4 *>(row)[i] = make_uint4(0, 0, 0, 0);
        else
            for (int64_t i = lane; i < z.L; i += nlanes) row[i] = 0;
    }
    if (b == 0 && lane == 0) {
        if (z.cnt0) *z.cnt0 = 0;
        if (z.cnt1) *z.cnt1 = 0;
        if (z.cnt2) *z.cnt2 = 0;
    }
}

// ------------------------------------------------------------- stream pass
// grid (nchunk, B): each CTA streams CH contiguous samples of one signal and
// writes its |x|^2 partial (fixed-order reduction).  Pairs of samples are
// loaded per instruction -- 32 B (LDG.256, evict-first, no L1 allocate) for
// complex128, 16 B for complex64 storage -- the measured best shape on B200
// (tools/membw.cu: 7.55 TB/s pure read).  The shift windows are not touched
// here: the FFT kernel gathers them straight from x.
template <int C64, int THREADS, int UNROLL>
__global__ void __launch_bounds__(THREADS) k_sumsq(const void *__restrict__ x_, int64_t n, int64_t CH,
                                                  double *__restrict__ partial, DecodeScratch z) {
    pdl_wait();
    const int64_t b = blockIdx.y;
    const int64_t chunk = blockIdx.x;
    // latency path: the solve's first kernel zeroes the worklist counters
    if (chunk == 0) zero_scratch(z, b, threadIdx.x, THREADS);
    const int64_t CHp = CH >> 1;                        // sample pairs in this chunk
    const int64_t base = (b * n + chunk * CH) >> 1;     // pair index
    double acc = 0.0;
    for (int64_t off = 0; off < CHp; off += int64_t(THREADS) * UNROLL) {
        double v[UNROLL][4];
#pragma unroll
        for (int u = 0; u < UNROLL; u++) {
            const int64_t pidx = off + int64_t(u) * THREADS + threadIdx.x;
            if (pidx < CHp) {
                if (C64) {
                    const float4 f = __ldcs(reinterpret_cast<const float4 *>(x_) + base + pidx);
                    v[u][0] = f.x; v[u][1] = f.y; v[u][2] = f.z; v[u][3] = f.w;
                } else {
                    const double *pp = reinterpret_cast<const double *>(x_) + 4 * (base + pidx);
                    asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v4.f64 {%0,%1,%2,%3}, [%4];"
                                 : "=d"(v[u][0]), "=d"(v[u][1]), "=d"(v[u][2]), "=d"(v[u][3])
                                 : "l"(pp));
                }
            } else {
                v[u][0] = v[u][1] = v[u][2] = v[u][3] = 0.0;
            }
        }
#pragma unroll
        for (int u = 0; u < UNROLL; u++)
            acc = fma(v[u][0], v[u][0], fma(v[u][1], v[u][1], fma(v[u][2], v[u][2], fma(v[u][3], v[u][3], acc))));
    }
    // deterministic block reduction: warp xor-tree, then fixed-order smem tree
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    __shared__ double red[THREADS / 32];
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < THREADS / 32; w++) t += red[w];
        partial[b * gridDim.x + chunk] = t;
    }
}

// Persistent form: one CTA per SM grid-strides over (signal, chunk) items, so
// the kernel never holds pending CTAs and concurrent FFT/decode kernels of the
// previous signal chunk (aux stream) start at once in the SM resources this
// kernel leaves free (it reserves ~120 KB of shared memory to stay at one
// 1024-thread CTA per SM, which still streams at the full read rate).
template <int C64, int THREADS, int UNROLL>
__global__ void __launch_bounds__(THREADS) k_sumsq_persistent(const void *__restrict__ x_, int64_t n,
                                                             int64_t CH, int64_t nchunk, int64_t nitems,
                                                             double *__restrict__ partial) {
    extern __shared__ double s_reserved[];
    __shared__ double red[THREADS / 32];
    const int64_t CHp = CH >> 1;
    for (int64_t item = blockIdx.x; item < nitems; item += gridDim.x) {
        const int64_t b = item / nchunk, chunk = item - b * nchunk;
        const int64_t base = (b * n + chunk * CH) >> 1;
        double acc = 0.0;
        for (int64_t off = 0; off < CHp; off += int64_t(THREADS) * UNROLL) {
            double v[UNROLL][4];
#pragma unroll
            for (int u = 0; u < UNROLL; u++) {
                const int64_t pidx = off + int64_t(u) * THREADS + threadIdx.x;
                if (pidx < CHp) {
                    if (C64) {
                        const float4 f = __ldcs(reinterpret_cast<const float4 *>(x_) + base + pidx);
                        v[u][0] = f.x; v[u][1] = f.y; v[u][2] = f.z; v[u][3] = f.w;
                    } else {
                        const double *pp = reinterpret_cast<const double *>(x_) + 4 * (base + pidx);
                        asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v4.f64 {%0,%1,%2,%3}, [%4];"
                                     : "=d"(v[u][0]), "=d"(v[u][1]), "=d"(v[u][2]), "=d"(v[u][3])
                                     : "l"(pp));
                    }
                } else {
                    v[u][0] = v[u][1] = v[u][2] = v[u][3] = 0.0;
                }
            }
#pragma unroll
            for (int u = 0; u < UNROLL; u++)
                acc = fma(v[u][0], v[u][0], fma(v[u][1], v[u][1], fma(v[u][2], v[u][2], fma(v[u][3], v[u][3], acc))));
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
        __syncthreads();
        if (threadIdx.x == 0) {
            double t = 0.0;
            for (int w = 0; w < THREADS / 32; w++) t += red[w];
            partial[item] = t;
            if (t == -1.0) s_reserved[0] = t;   // keeps the reservation
        }
        __syncthreads();
    }
}

// rms and threshold per signal: fixed-order pairwise tree over the partials
__global__ void k_rms(const double *__restrict__ partial, int64_t nchunk, int64_t n, double zt,
                      int64_t d, double *__restrict__ rms, double *__restrict__ thr, DecodeScratch z) {
    pdl_wait();
    const int64_t b = blockIdx.x;
    zero_scratch(z, b, threadIdx.x, blockDim.x);
    __shared__ double buf[1024];
    double acc = 0.0;
    for (int64_t i = threadIdx.x; i < nchunk; i += blockDim.x) acc += partial[b * nchunk + i];
    buf[threadIdx.x] = acc;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) buf[threadIdx.x] += buf[threadIdx.x + s];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const double r = sqrt(buf[0] / (double)n);
        rms[b] = r;
        thr[b] = DMUL(DMUL(zt, r), (double)d);   // cfg.zero_threshold * rms(x) * d
    }
}

// the same tree for nchunk <= 64 with one warp per signal: the 1024-slot
// tree's levels above 32 only add exact zeros, so lane t starting from
// p[t] + p[t+32] and halving by shuffles reproduces it bit for bit
__global__ void k_rms_warp(const double *__restrict__ partial, int64_t B, int64_t nchunk, int64_t n, double zt,
                           int64_t d, double *__restrict__ rms, double *__restrict__ thr, DecodeScratch z) {
    pdl_wait();
    const int64_t b = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (b >= B) return;
    zero_scratch(z, b, lane, 32);
    const double *pb = partial + b * nchunk;
    double v = (lane < nchunk ? pb[lane] : 0.0) + (lane + 32 < nchunk ? pb[lane + 32] : 0.0);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (lane == 0) {
        const double r = sqrt(v / (double)n);
        rms[b] = r;
        thr[b] = DMUL(DMUL(zt, r), (double)d);
    }
}

static inline void launch_rms(const double *partial, int64_t B, int64_t nchunk, int64_t n, double zt,
                              int64_t d, double *rms, double *thr, cudaStream_t st,
                              DecodeScratch z = DecodeScratch{nullptr, 0, nullptr, nullptr, nullptr}) {
    if (nchunk <= 64)
        launch_pdl(k_rms_warp, dim3((unsigned)((B + 7) / 8)), dim3(256), 0, st, partial, B, nchunk, n, zt, d, rms,
                   thr, z);
    else
        launch_pdl(k_rms, dim3((unsigned)B), dim3(1024), 0, st, partial, nchunk, n, zt, d, rms, thr, z);
}

// thresholds from a known rms (rms_in): copy rms out, zt*rms*d
__global__ void k_thr_from_rms(const double *__restrict__ rms_in, int64_t B, double zt, int64_t d,
                               double *__restrict__ rms_out, double *__restrict__ thr, DecodeScratch z) {
    pdl_wait();
    const int64_t b = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (b < B) zero_scratch(z, b, 0, 1);
    if (b < B) {
        const double r = rms_in[b];
        rms_out[b] = r;
        thr[b] = DMUL(DMUL(zt, r), (double)d);
    }
}

__global__ void k_scale_thr(const double *__restrict__ rms, int64_t B, double zt, int64_t d,
                            double *__restrict__ out) {
    const int64_t b = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (b < B) out[b] = DMUL(DMUL(zt, rms[b]), (double)d);
}

// --------------------------------------------------- non-iterative decode
// status: 0 inactive, 1..a_max accepted at that a, 0xFF unresolved (0xFE =
// pending a >= 2 while the worklist is processed).
//
// Pass 1 (k_decode_a1): thread per bin, syndromes in registers (S is a
// template parameter), activity test + the a = 1 model; bins that fail it
// go to a compact worklist (warp-aggregated append).  Pass 2
// (k_decode_multi): grid-stride over the worklist, a = 2..a_max.  Every bin's
// result depends only on its own syndromes (exact.py:184-192), so the split
// and the worklist order change nothing.
template <int S>
__global__ void __launch_bounds__(128) k_decode_a1(const cx *__restrict__ V, int64_t B, int64_t L,
                                                   int a_max, int64_t n,
                                                   const double *__restrict__ thr,
                                                   uint8_t *__restrict__ status,
                                                   int64_t *__restrict__ bin_loc,
                                                   cx *__restrict__ bin_val,
                                                   int64_t *__restrict__ wl,
                                                   unsigned long long *__restrict__ wl_count) {
    pdl_wait();
    const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const bool valid = t < B * L;
    bool pending = false;
    if (valid) {
        const int64_t b = t / L, k = t - b * L;
        cx syn[S];
        const double th = thr[b];
        // |v| > th decided on |v|^2 away from the boundary; the exact hypot
        // comparison (numpy abs) only inside a 1e-6-relative band around it
        const double th2lo = th * th * (1.0 - 1e-6), th2hi = th * th * (1.0 + 1e-6);
        bool active = false;
#pragma unroll
        for (int s = 0; s < S; s++) {
            syn[s] = ldcx(V + (b * S + s) * L + k);
            const double q = syn[s].re * syn[s].re + syn[s].im * syn[s].im;
            active = active || (q > th2hi) || (q >= th2lo && cabs_i(syn[s]) > th);
        }
        uint8_t st = 0;
        if (active) {
            Decoded o;
            decode_try_t<1, S>(syn, n, L, k, o);
            if (o.accept) {
                st = 1;
                bin_loc[t * a_max] = o.loc[0];
                stcx(bin_val + t * a_max, o.val[0]);
            } else if (a_max > 1) {
                st = 0xFE;
                pending = true;
            } else {
                st = 0xFF;
            }
        }
        status[t] = st;
    }
    const unsigned mask = __ballot_sync(0xffffffffu, pending);
    if (mask) {
        const int lane = threadIdx.x & 31;
        unsigned long long base = 0;
        if (lane == __ffs(mask) - 1) base = atomicAdd(wl_count, (unsigned long long)__popc(mask));
        base = __shfl_sync(0xffffffffu, base, __ffs(mask) - 1);
        if (pending) wl[base + __popc(mask & ((1u << lane) - 1))] = t;
    }
}

// Latency path: k_decode_a1 with the rms tree of k_rms_warp in its prologue
// (every warp folds its signal's <= 64 partials the same way, so the threshold
// has the same bits), which removes the rms kernel and the activity
// compaction from a small solve's launch chain.  Needs L % 32 == 0 (a warp's
// bins belong to one signal).
template <int S>
__global__ void __launch_bounds__(128) k_decode_a1r(const cx *__restrict__ V, int64_t B, int64_t L, int a_max,
                                                    int64_t n, const double *__restrict__ partial, int64_t nchunk,
                                                    double zt, int64_t d, double *__restrict__ rms,
                                                    double *__restrict__ thr_out, uint8_t *__restrict__ status,
                                                    int64_t *__restrict__ bin_loc, cx *__restrict__ bin_val,
                                                    int64_t *__restrict__ wl,
                                                    unsigned long long *__restrict__ wl_count) {
    pdl_wait();
    const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    const int64_t t_first = t - lane;
    if (t_first >= B * L) return;   // whole warp out of range
    const int64_t b = t_first / L, k = t - b * L;
    double th;
    {
        const double *pb = partial + b * nchunk;
        double v = (lane < nchunk ? pb[lane] : 0.0) + (lane + 32 < nchunk ? pb[lane + 32] : 0.0);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
        const double r = sqrt(v / (double)n);
        th = DMUL(DMUL(zt, r), (double)d);
        if (lane == 0 && t_first == b * L) {
            rms[b] = r;
            thr_out[b] = th;
        }
        th = __shfl_sync(0xffffffffu, th, 0);
    }
    bool pending = false;
    {
        cx syn[S];
        const double th2lo = th * th * (1.0 - 1e-6), th2hi = th * th * (1.0 + 1e-6);
        bool active = false;
#pragma unroll
        for (int s = 0; s < S; s++) {
            syn[s] = ldcx(V + (b * S + s) * L + k);
            const double q = syn[s].re * syn[s].re + syn[s].im * syn[s].im;
            active = active || (q > th2hi) || (q >= th2lo && cabs_i(syn[s]) > th);
        }
        uint8_t st = 0;
        if (active) {
            Decoded o;
            decode_try_t<1, S>(syn, n, L, k, o);
            if (o.accept) {
                st = 1;
                bin_loc[t * a_max] = o.loc[0];
                stcx(bin_val + t * a_max, o.val[0]);
            } else if (a_max > 1) {
                st = 0xFE;
                pending = true;
            } else {
                st = 0xFF;
            }
        }
        status[t] = st;
    }
    const unsigned mask = __ballot_sync(0xffffffffu, pending);
    if (mask) {
        unsigned long long base = 0;
        if (lane == __ffs(mask) - 1) base = atomicAdd(wl_count, (unsigned long long)__popc(mask));
        base = __shfl_sync(0xffffffffu, base, __ffs(mask) - 1);
        if (pending) wl[base + __popc(mask & ((1u << lane) - 1))] = t;
    }
}

// Dense a = 1 decode.  The FFT epilogue marks active bins (act); a compaction
// pass lists them, and the decode runs one active bin per thread (no idle
// lanes for the ~78 % inactive bins of config 2).
__global__ void __launch_bounds__(1024) k_act_compact(const uint8_t *__restrict__ act, int64_t nbins,
                                                      uint8_t *__restrict__ status,
                                                      int64_t *__restrict__ awl,
                                                      unsigned long long *__restrict__ awlc) {
    pdl_wait();
    // one global atomic per 4096-bin block (a single counter hammered once
    // per warp measured 95 us at config 2)
    __shared__ int wsum[32];
    __shared__ unsigned long long s_base;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t t0 = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) * 4;
    bool on[4];
    int mine = 0;
#pragma unroll
    for (int u = 0; u < 4; u++) {
        const int64_t t = t0 + u;
        on[u] = t < nbins && act[t];
        if (t < nbins && !on[u]) status[t] = 0;
        mine += on[u];
    }
    int inc = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) wsum[warp] = inc;
    __syncthreads();
    if (threadIdx.x == 0) {
        int tot = 0;
        for (int w = 0; w < 32; w++) {
            const int c = wsum[w];
            wsum[w] = tot;
            tot += c;
        }
        s_base = tot ? atomicAdd(awlc, (unsigned long long)tot) : 0;
    }
    __syncthreads();
    unsigned long long pos = s_base + wsum[warp] + (inc - mine);
#pragma unroll
    for (int u = 0; u < 4; u++)
        if (on[u]) awl[pos++] = t0 + u;
}

#ifndef SFDT_A1D_MINB
#define SFDT_A1D_MINB 1   // resident CTAs per SM: 3 neutral, 8 (64 registers) 15 % slower (tools/exp_decode_occ.sh)
#endif
template <int S>
__global__ void __launch_bounds__(128, SFDT_A1D_MINB) k_decode_a1_dense(const cx *__restrict__ V, int64_t L, int a_max,
                                                         int64_t n, uint8_t *__restrict__ status,
                                                         int64_t *__restrict__ bin_loc,
                                                         cx *__restrict__ bin_val,
                                                         const int64_t *__restrict__ awl,
                                                         const unsigned long long *__restrict__ awlc,
                                                         int64_t *__restrict__ wl,
                                                         unsigned long long *__restrict__ wl_count) {
    pdl_wait();
    const int64_t cnt = (int64_t)*awlc;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < cnt;
         i += int64_t(gridDim.x) * blockDim.x) {
        const int64_t t = awl[i];
        const int64_t b = t / L, k = t - b * L;
        cx syn[S];
#pragma unroll
        for (int s = 0; s < S; s++) syn[s] = ldcx(V + (b * S + s) * L + k);
        Decoded o;
        decode_try_t<1, S>(syn, n, L, k, o);
        if (o.accept) {
            status[t] = 1;
            bin_loc[t * a_max] = o.loc[0];
            stcx(bin_val + t * a_max, o.val[0]);
        } else {
            status[t] = a_max > 1 ? 0xFE : 0xFF;
        }
        // warp-aggregated append of the bins that need a >= 2
        const bool pend = !o.accept && a_max > 1;
        const unsigned act_mask = __activemask();
        const unsigned m = __ballot_sync(act_mask, pend);
        if (m) {
            const int lane = threadIdx.x & 31;
            const int leader = __ffs(m) - 1;
            unsigned long long base = 0;
            if (lane == leader) base = atomicAdd(wl_count, (unsigned long long)__popc(m));
            base = __shfl_sync(act_mask, base, leader);
            if (pend) wl[base + __popc(m & ((1u << lane) - 1))] = t;
        }
    }
}

#ifndef SFDT_MULTI_TEMPLATED
#define SFDT_MULTI_TEMPLATED 1
#endif
#ifndef SFDT_MULTI_MINB
#define SFDT_MULTI_MINB 3   // resident CTAs per SM: 6 -> 3 measured 12-15 % faster (instruction-fetch bound: fewer warps, no spills), profiles/r02_decode_minb.txt
#endif
template <int S>
__global__ void __launch_bounds__(128, SFDT_MULTI_MINB) k_decode_multi(const cx *__restrict__ V, int64_t L, int a_max,
                                                      int a_hi, int64_t n, uint8_t *__restrict__ status,
                                                      int64_t *__restrict__ bin_loc,
                                                      cx *__restrict__ bin_val,
                                                      const int64_t *__restrict__ wl,
                                                      const unsigned long long *__restrict__ wl_count,
                                                      int64_t *__restrict__ wl2,
                                                      unsigned long long *__restrict__ wl2_count, int a_lo = 2,
                                                      long long gate_min = -1) {
    pdl_wait();
    // tries a = a_lo..a_hi; with a_hi < a_max the bins still unsolved go to
    // wl2 (the a >= 3 launches take a_hi + 1..a_max).  gate_min: run only
    // when the list holds more than gate_min bins (k_decode_coop takes it
    // otherwise)
    const int64_t cnt = (int64_t)*wl_count;
    if (cnt <= gate_min) return;
#ifdef SFDT_MULTI_PROFILE
    const long long k0_ = clock64();
    if (blockIdx.x == 0 && threadIdx.x == 0)
        printf("MULTI start a_lo=%d a_hi=%d cnt=%lld grid=%d\n", a_lo, a_hi, (long long)cnt, (int)gridDim.x);
#endif
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < cnt;
         i += int64_t(gridDim.x) * blockDim.x) {
#ifdef SFDT_MULTI_PROFILE
        const long long c0_ = clock64();
#endif
        const int64_t t = wl[i];
        const int64_t b = t / L, k = t - b * L;
        cx syn[S];
#pragma unroll
        for (int s = 0; s < S; s++) syn[s] = ldcx(V + (b * S + s) * L + k);
        uint8_t st = a_hi < a_max ? 0xFE : 0xFF;
        Decoded o;
        for (int a = a_lo; a <= a_hi; a++) {
#if SFDT_MULTI_TEMPLATED
            if (a == 2) decode_try_t<2, S>(syn, n, L, k, o);
            else if (a == 3) decode_try_t<3, S>(syn, n, L, k, o);
            else decode_try_t<4, S>(syn, n, L, k, o);
#else
            decode_try(syn, S, a, n, L, k, o);
#endif
            if (o.accept) {
                st = (uint8_t)a;
                for (int j = 0; j < a; j++) {
                    bin_loc[t * a_max + j] = o.loc[j];
                    stcx(bin_val + t * a_max + j, o.val[j]);
                }
                break;
            }
        }
        status[t] = st;
#ifdef SFDT_MULTI_PROFILE
        if ((i & 8191) == 0)
            printf("MULTI item i=%lld st=%d start_off=%lld cyc=%lld sm=%d\n", (long long)i, (int)st, c0_ - k0_, clock64() - c0_, (int)blockIdx.x);
#endif
        if (a_hi < a_max) {
            const bool pend = st == 0xFE;
            const unsigned act_mask = __activemask();
            const unsigned m = __ballot_sync(act_mask, pend);
            if (m) {
                const int lane = threadIdx.x & 31;
                const int leader = __ffs(m) - 1;
                unsigned long long base = 0;
                if (lane == leader) base = atomicAdd(wl2_count, (unsigned long long)__popc(m));
                base = __shfl_sync(act_mask, base, leader);
                if (pend) wl2[base + __popc(m & ((1u << lane) - 1))] = t;
            }
        }
    }
}

// Cooperative multi-collision decode (decode_coop.cuh).  A CTA of `nw` warps
// takes four worklist bins at a time (eight lanes per bin, so a warp executes
// one trial's code without divergence): warp w runs the a = a_lo + w trial of
// all four bins at once, and the smallest accepted a wins -- the one the
// reference's ascending loop (exact.py:184-192) stops at, because a trial
// depends only on the bin's syndromes.  Trials beyond a_lo + nw - 1 (rare:
// 3 % of config-1 signals hold a 4-collision bin) run afterwards on warp 0,
// only when one of the four bins is still unsolved.
constexpr int COOP_BINS = 32 / COOP_G;

template <int S>
__device__ __forceinline__ void coop_trial(int A, const cx *syn, int64_t n, int64_t L, int64_t k, int g,
                                           DecodedCoop &o) {
    o.accept = false;
    if (A == 2) {
        if constexpr (S >= 4) decode_try_coop<2, S>(syn, n, L, k, g, o);
    } else if (A == 3) {
        if constexpr (S >= 6) decode_try_coop<3, S>(syn, n, L, k, g, o);
    } else {
        if constexpr (S >= 8) decode_try_coop<4, S>(syn, n, L, k, g, o);
    }
}

template <int S>
__global__ void __launch_bounds__(96) k_decode_coop(const cx *__restrict__ V, int64_t L, int a_max, int a_lo,
                                                    int64_t n, uint8_t *__restrict__ status,
                                                    int64_t *__restrict__ bin_loc, cx *__restrict__ bin_val,
                                                    const int64_t *__restrict__ wl,
                                                    const unsigned long long *__restrict__ wl_count,
                                                    long long gate_max = 0x7fffffffffffffffLL) {
    pdl_wait();
    if ((long long)*wl_count > gate_max) return;   // CTA-uniform: k_decode_multi took the list
    __shared__ int s_acc[3][COOP_BINS];
    __shared__ long long s_loc[3][COOP_BINS][4];
    __shared__ double2 s_val[3][COOP_BINS][4];
    __shared__ int s_more;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane & (COOP_G - 1), grp = lane / COOP_G;
    const int nw = blockDim.x >> 5;
    const int64_t cnt = (int64_t)*wl_count;
    for (int64_t base = int64_t(blockIdx.x) * COOP_BINS; base < cnt; base += int64_t(gridDim.x) * COOP_BINS) {
        const int64_t i = base + grp;
        const bool valid = i < cnt;
        const int64_t t = valid ? wl[i] : 0;
        const int64_t b = t / L, k = t - b * L;
        cx syn[S];
#pragma unroll
        for (int s = 0; s < S; s++) syn[s] = valid ? ldcx(V + (b * S + s) * L + k) : mk(0.0, 0.0);
        int A = a_lo + warp, next = a_lo + nw;
        bool run = true;
        int a_win = 0, slot = 0;   // warp 0's verdict on its four bins
        for (;;) {
            if (run) {
                DecodedCoop o;
                coop_trial<S>(A, syn, n, L, k, g, o);
                if (g == 0 && a_win == 0) {
                    s_acc[warp][grp] = o.accept ? 1 : 0;
                    if (o.accept) {
                        for (int j = 0; j < A; j++) {
                            s_loc[warp][grp][j] = o.loc[j];
                            s_val[warp][grp][j] = make_double2(o.val[j].re, o.val[j].im);
                        }
                    }
                }
            }
            __syncthreads();
            if (warp == 0) {
                if (a_win == 0) {
                    for (int w = nw - 1; w >= 0; w--)
                        if (s_acc[w][grp]) {
                            a_win = w == 0 ? A : a_lo + w;
                            slot = w;
                        }
                }
                const bool open = __any_sync(0xffffffffu, valid && a_win == 0 && next <= a_max);
                if (lane == 0) s_more = open ? next : 0;
            }
            __syncthreads();
            const int mo = s_more;   // CTA-uniform
            if (!mo) break;
            // later trials (rare) on warp 0 alone; the other warps' flags for
            // a still-open bin stay 0
            A = mo;
            next = mo + 1;
            run = warp == 0;
        }
        if (warp == 0 && valid) {
            if (g == 0) status[t] = a_win ? (uint8_t)a_win : 0xFF;
            if (g < a_win) {
                bin_loc[t * a_max + g] = s_loc[slot][grp][g];
                *reinterpret_cast<double2 *>(bin_val + t * a_max + g) = s_val[slot][grp][g];
            }
        }
        __syncthreads();
    }
}

// decode_coop (sfdt_tuning): 0 one thread per bin for every a; 1 cooperative
// trials, a = 2 and 3 side by side (a = 4 afterwards where needed); 2 thread
// per bin for a = 2, cooperative for a = 3 then 4; 3 cooperative, every a
// side by side; -1 picks 1 while the batch has few bins (a latency-bound
// solve), else 2.
static inline int decode_coop_mode(int req, int64_t nbins, int a_max) {
    if (a_max < 2) return 0;
    int mode = req;
    if (mode < 0) mode = nbins <= (int64_t)1 << 17 ? 1 : 2;
    if (mode == 2 && a_max < 3) mode = 0;
    return mode;
}

// a >= 2 trials on the worklist of bins the a = 1 model failed on
template <int S>
static int launch_decode_multi(const cx *V, int64_t nbins, int64_t L, int a_max, int64_t n, uint8_t *status,
                               int64_t *bin_loc, cx *bin_val, int64_t *wl, unsigned long long *wl_count,
                               int64_t *wl2, unsigned long long *wl2_count, int coop, cudaStream_t stream) {
    if (a_max > 1) {
        const int mode = decode_coop_mode(coop, nbins, a_max);
        if (mode != 1 && mode != 3) {
            const int a_hi = mode == 2 ? 2 : a_max;
            launch_pdl(k_decode_multi<S>, dim3(wl_grid(nbins, 128, one_wave(k_decode_multi<S>, 128))), dim3(128), 0,
                       stream, V, L, a_max, a_hi, n, status, bin_loc, bin_val, (const int64_t *)wl,
                       (const unsigned long long *)wl_count, wl2, wl2_count, 2, -1LL);
            SFDT_CHECK_LAUNCH();
        }
        if (mode != 0) {
            const int a_lo = mode == 2 ? 3 : 2;
            int nw = mode == 2 ? 1 : (mode == 3 ? 3 : 2);
            if (nw > a_max - a_lo + 1) nw = a_max - a_lo + 1;
            const int threads = 32 * nw;
            const int wave = one_wave(k_decode_coop<S>, threads);
            // mode 2: eight lanes per bin pay while the a >= 3 bins fit one
            // cooperative wave (~9.5k bins; config 2's ~9k sit at the
            // crossover, either kernel takes ~70 us there); a high alias load
            // (config 3 at mu = 1: 21k such bins, several waves) is faster one
            // thread per bin (2.72 -> 2.59 ms per batch).  The count is known
            // only on the device: both kernels are enqueued and the list's
            // length picks the one that runs.
            const long long gate = mode == 2 ? (long long)wave * COOP_BINS : 0x7fffffffffffffffLL;
            if (mode == 2) {
                launch_pdl(k_decode_multi<S>, dim3(wl_grid(nbins, 128, one_wave(k_decode_multi<S>, 128))), dim3(128),
                           0, stream, V, L, a_max, a_max, n, status, bin_loc, bin_val, (const int64_t *)wl2,
                           (const unsigned long long *)wl2_count, (int64_t *)nullptr,
                           (unsigned long long *)nullptr, 3, gate);
                SFDT_CHECK_LAUNCH();
            }
            launch_pdl(k_decode_coop<S>, dim3(wl_grid(nbins, COOP_BINS, wave)),
                       dim3(threads), 0, stream, V, L, a_max, a_lo, n, status, bin_loc, bin_val,
                       (const int64_t *)(mode == 2 ? wl2 : wl),
                       (const unsigned long long *)(mode == 2 ? wl2_count : wl_count), gate);
            SFDT_CHECK_LAUNCH();
        }
    }
    return SFDT_OK;
}

// the latency path's decode: rms + activity + a = 1 in one kernel, then a >= 2
template <int S>
static int launch_decode_small(const cx *V, int64_t B, int64_t L, int a_max, int64_t n, const double *partial,
                               int64_t nchunk, double zt, int64_t d, double *rms, double *thr, uint8_t *status,
                               int64_t *bin_loc, cx *bin_val, int64_t *wl, unsigned long long *wl_count,
                               int64_t *wl2, unsigned long long *wl2_count, int coop, cudaStream_t stream) {
    const int64_t nbins = B * L;
    launch_pdl(k_decode_a1r<S>, dim3((unsigned)((nbins + 127) / 128)), dim3(128), 0, stream, V, B, L, a_max, n,
               partial, nchunk, zt, d, rms, thr, status, bin_loc, bin_val, wl, wl_count);
    SFDT_CHECK_LAUNCH();
    return launch_decode_multi<S>(V, nbins, L, a_max, n, status, bin_loc, bin_val, wl, wl_count, wl2, wl2_count, coop,
                                  stream);
}

template <int S>
static int launch_decode_noniter(const cx *V, int64_t B, int64_t L, int a_max, int64_t n,
                                 const double *thr, uint8_t *status, int64_t *bin_loc, cx *bin_val,
                                 int64_t *wl, unsigned long long *wl_count, cudaStream_t stream,
                                 const uint8_t *act, int64_t *awl, unsigned long long *awlc,
                                 int64_t *wl2, unsigned long long *wl2_count, int coop) {
    const int64_t nbins = B * L;
    // with `act` (the dense path) the counters were zeroed by the rms kernel
    if (!act) {
        cudaMemsetAsync(wl_count, 0, sizeof(unsigned long long), stream);
        cudaMemsetAsync(wl2_count, 0, sizeof(unsigned long long), stream);
    }
    if (act) {
        launch_pdl(k_act_compact, dim3((unsigned)((nbins + 4095) / 4096)), dim3(1024), 0, stream, act, nbins, status,
                   awl, awlc);
        SFDT_CHECK_LAUNCH();
        launch_pdl(k_decode_a1_dense<S>, dim3(wl_grid(nbins, 128, one_wave(k_decode_a1_dense<S>, 128))), dim3(128), 0,
                   stream, V, L, a_max, n, status, bin_loc, bin_val, (const int64_t *)awl,
                   (const unsigned long long *)awlc, wl, wl_count);
    } else {
        launch_pdl(k_decode_a1<S>, dim3((unsigned)((nbins + 127) / 128)), dim3(128), 0, stream, V, B, L, a_max, n, thr,
                   status, bin_loc, bin_val, wl, wl_count);
    }
    SFDT_CHECK_LAUNCH();
    return launch_decode_multi<S>(V, nbins, L, a_max, n, status, bin_loc, bin_val, wl, wl_count, wl2, wl2_count, coop,
                                  stream);
}

// ----------------------------------------------------- iterative pass l
// V holds S views per signal with leading dimension L0 (bins < m used).
// Before the pass, views 2l and 2l+1 hold fresh scaled FFTs at the current
// d.  Slots: per pass p and bin (< m_p), up to a_max entries.
struct IterState {
    cx *V;                 // (B, S, L0)
    uint8_t *deferred;     // (B, L0)  current deferred flags (bins < m)
    int64_t *slot_loc;     // (B, 4 passes, L0, a_max)
    cx *slot_val;          // same
    uint8_t *slot_a;       // (B, 4, L0): a_try that accepted (0 = none)
    uint8_t *slot_dupmask; // (B, 4, L0): roots that overwrote an earlier slot
    unsigned long long *cnt;  // (B, 4, 4): attempted, solved, deferred_events, n_active
};

struct PassInfo {
    int64_t m[4], d[4];
};

__device__ __forceinline__ int64_t slot_index(int64_t b, int p, int64_t k, int64_t L0) {
    return (b * 4 + p) * L0 + k;
}

// Pass l, phase 1 (thread per bin): fold, SubFreq, activity; active bins
// are appended (block-aggregated) to a dense list for phase 2.
__global__ void __launch_bounds__(256) k_iter_prep(IterState st, int64_t B, int64_t L0, int S, int a_max,
                                                   int l, int64_t n, int64_t m, int fold,
                                                   const double *__restrict__ thr_base,
                                                   int64_t *__restrict__ awl,
                                                   unsigned long long *__restrict__ awlc) {
    const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const bool valid = t < B * m;
    const int64_t b = valid ? t / m : 0, k = valid ? t - b * m : 0;
    bool active = false;
    if (valid) {
        cx *Vb = st.V + b * S * L0;
        // fold previous views to the doubled d (exact.py:225-229)
        if (fold) {
            for (int j = 0; j < 2 * l; j++) {
                const cx lo = Vb[j * L0 + k], hi = Vb[j * L0 + k + m];
                Vb[j * L0 + k] = cadd(lo, hi);
            }
            const uint8_t dl = st.deferred[b * L0 + k], dh = st.deferred[b * L0 + k + m];
            st.deferred[b * L0 + k] = dl | dh;
        }
        // SubFreq of every solved entry mapped to this bin, in dict insertion
        // order: pass asc, a_try desc, origin bin asc, root order
        // (exact.py:234-240, np.subtract.at)
        cx v0 = Vb[(2 * l) * L0 + k], v1 = Vb[(2 * l + 1) * L0 + k];
        for (int p = 0; p < l; p++) {
            const int nb = 1 << (l - p);
            // origin bins k + i*m at pass p, ordered by (a desc, bin asc)
            int order[8];
            int cntb = 0;
            for (int i = 0; i < nb; i++) {
                const uint8_t ai = st.slot_a[slot_index(b, p, k + i * m, L0)];
                if (!ai) continue;
                int pos = cntb++;
                while (pos > 0) {
                    const int prev = order[pos - 1];
                    const uint8_t ap = st.slot_a[slot_index(b, p, k + prev * m, L0)];
                    if (ap >= ai) break;   // stable: keep bin order for equal a
                    order[pos] = prev;
                    pos--;
                }
                order[pos] = i;
            }
            for (int q = 0; q < cntb; q++) {
                const int64_t si = slot_index(b, p, k + order[q] * m, L0);
                const int a = st.slot_a[si];
                const uint8_t dup = st.slot_dupmask[si];
                for (int j = 0; j < a; j++) {
                    if (dup & (1u << j)) continue;   // overwrite, not a new key
                    const int64_t loc = st.slot_loc[si * a_max + j];
                    const cx val = st.slot_val[si * a_max + j];
                    v0 = csub(v0, nmul(val, phase(loc, 2 * l, n)));
                    v1 = csub(v1, nmul(val, phase(loc, 2 * l + 1, n)));
                }
            }
        }
        Vb[(2 * l) * L0 + k] = v0;
        Vb[(2 * l + 1) * L0 + k] = v1;
        active = (cabs_(v0) > thr_base[b + B * (l + 1)]) || (cabs_(v1) > thr_base[b + B * (l + 1)]) ||
                 st.deferred[b * L0 + k];
        const int64_t sp = slot_index(b, l, k, L0);
        st.slot_a[sp] = 0;
        st.slot_dupmask[sp] = 0;
    }
    // attempted count per signal (warp-aggregated) + block-aggregated append
    const unsigned full = 0xffffffffu;
    const int64_t bw = __shfl_sync(full, b, 0);
    const bool same = __all_sync(full, !valid || b == bw);
    const unsigned am = __ballot_sync(full, active);
    if (same) {
        if ((threadIdx.x & 31) == 0 && am) atomicAdd(st.cnt + (bw * 4 + l) * 4, (unsigned long long)__popc(am));
    } else if (active) {
        atomicAdd(st.cnt + (b * 4 + l) * 4, 1ull);
    }
    __shared__ int wsum[8];
    __shared__ unsigned long long s_base;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) wsum[warp] = __popc(am);
    __syncthreads();
    if (threadIdx.x == 0) {
        int tot = 0;
        for (int w = 0; w < 8; w++) {
            const int c = wsum[w];
            wsum[w] = tot;
            tot += c;
        }
        s_base = tot ? atomicAdd(awlc, (unsigned long long)tot) : 0;
    }
    __syncthreads();
    if (active) awl[s_base + wsum[warp] + __popc(am & ((1u << lane) - 1))] = t;
}

// Pass l, phase 2 (thread per active bin): descending-a decode with the
// singular-only retry, deferral, duplicate overwrite, and removal of the
// accepted terms from every live view (exact.py:253-280).  LP = l is a
// template parameter so the 2l+2 syndromes and every Cramer matrix are
// register-resident.
#ifndef SFDT_ITER_MINB
#define SFDT_ITER_MINB 4   // 2 / 3: the four passes 324 -> 307 / 315 us at config 2 (within 0.2 % of the step)
#endif
template <int LP>
__global__ void __launch_bounds__(128, SFDT_ITER_MINB) k_iter_decode(IterState st, int64_t L0, int S, int a_max,
                                                        int64_t n, int64_t m,
                                                        const int64_t *__restrict__ awl,
                                                        const unsigned long long *__restrict__ awlc) {
    constexpr int SL = 2 * LP + 2;
    const int64_t cnt = (int64_t)*awlc;
    for (int64_t it = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; it < cnt;
         it += int64_t(gridDim.x) * blockDim.x) {
        const int64_t t = awl[it];
        const int64_t b = t / m, k = t - b * m;
        cx *Vb = st.V + b * S * L0;
        cx syn[SL];
#pragma unroll
        for (int j = 0; j < SL; j++) syn[j] = Vb[j * L0 + k];
        const int64_t sp = slot_index(b, LP, k, L0);
        bool solved = false, deferred_evt = false;
        Decoded o;
        for (int a_try = LP + 1; a_try >= 1; a_try--) {
            if (a_try == 1) decode_try_t<1, SL>(syn, n, m, k, o);
            else if (a_try == 2) { if constexpr (LP >= 1) decode_try_t<2, SL>(syn, n, m, k, o); }
            else if (a_try == 3) { if constexpr (LP >= 2) decode_try_t<3, SL>(syn, n, m, k, o); }
            else { if constexpr (LP >= 3) decode_try_t<4, SL>(syn, n, m, k, o); }
            if (o.accept) {
                solved = true;
                st.deferred[b * L0 + k] = 0;
                // duplicate locations overwrite the earlier slot's value
                uint8_t dupmask = 0;
                for (int j = 0; j < a_try; j++) {
                    bool found = false;
                    for (int p = 0; p < LP && !found; p++) {
                        const int nb = 1 << (LP - p);
                        for (int i = 0; i < nb && !found; i++) {
                            const int64_t si = slot_index(b, p, k + i * m, L0);
                            const int ap = st.slot_a[si];
                            const uint8_t dp = st.slot_dupmask[si];
                            for (int r = 0; r < ap; r++) {
                                if (!(dp & (1u << r)) && st.slot_loc[si * a_max + r] == o.loc[j]) {
                                    st.slot_val[si * a_max + r] = o.val[j];
                                    found = true;
                                    break;
                                }
                            }
                        }
                    }
                    if (found) dupmask |= (1u << j);
                    st.slot_loc[sp * a_max + j] = o.loc[j];
                    st.slot_val[sp * a_max + j] = o.val[j];
                }
                st.slot_a[sp] = (uint8_t)a_try;
                st.slot_dupmask[sp] = dupmask;
                // remove the decoded contribution from every live view
                // (exact.py:269-271)
#pragma unroll
                for (int j = 0; j < SL; j++) {
                    cx terms[4];
                    for (int r = 0; r < a_try; r++) terms[r] = nmul(o.val[r], phase(o.loc[r], j, n));
                    Vb[j * L0 + k] = csub(Vb[j * L0 + k], npsum(terms, a_try));
                }
                break;
            }
            if (!(a_try > 1 && o.retryable)) {
                st.deferred[b * L0 + k] = 1;
                deferred_evt = true;
                break;
            }
        }
        const unsigned act = __activemask();
        const int64_t bw = __shfl_sync(act, b, __ffs(act) - 1);
        const bool same = __all_sync(act, b == bw);
        const unsigned ns = __ballot_sync(act, solved), nd = __ballot_sync(act, deferred_evt);
        if (same) {
            if ((threadIdx.x & 31) == __ffs(act) - 1) {
                unsigned long long *c = st.cnt + (bw * 4 + LP) * 4;
                if (ns) atomicAdd(c + 1, (unsigned long long)__popc(ns));
                if (nd) atomicAdd(c + 2, (unsigned long long)__popc(nd));
            }
        } else {
            unsigned long long *c = st.cnt + (b * 4 + LP) * 4;
            if (solved) atomicAdd(c + 1, 1ull);
            if (deferred_evt) atomicAdd(c + 2, 1ull);
        }
    }
}

// residual max |v| over all views at the final m + remaining deferred bins
__global__ void k_iter_final(const cx *__restrict__ V, const uint8_t *__restrict__ deferred,
                             int64_t L0, int S, int64_t m, double *__restrict__ resid,
                             int64_t *__restrict__ ndef) {
    const int64_t b = blockIdx.x;
    double r = 0.0;
    long long nd = 0;
    for (int64_t i = threadIdx.x; i < int64_t(S) * m; i += blockDim.x) {
        const int64_t j = i / m, k = i - j * m;
        r = nanmax2(r, cabs_(V[(b * S + j) * L0 + k]));
    }
    for (int64_t k = threadIdx.x; k < m; k += blockDim.x) nd += deferred[b * L0 + k];
    __shared__ double rb[256];
    __shared__ long long db[256];
    rb[threadIdx.x] = r;
    db[threadIdx.x] = nd;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) {
            rb[threadIdx.x] = nanmax2(rb[threadIdx.x], rb[threadIdx.x + s]);
            db[threadIdx.x] += db[threadIdx.x + s];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        resid[b] = rb[0];
        ndef[b] = db[0];
    }
}

// ------------------------------------------------------------ compaction
// Non-iterative: per-signal block scan over bins ordered by (a, bin) ->
// entry offsets; unresolved bins ascending.  A signal's bins are split into
// segments of NONITER_SEG bins (one CTA each), so small batches of long
// views still fill the GPU: count per segment, fold the segments per
// signal, and emit each segment at its signal's class bases plus the counts
// of the segments before it.
constexpr int64_t NONITER_SEG = 8192;
constexpr int SEGF = 8;   // per-segment fields: unresolved, entries a=1..4, active, tries

// counts of one signal's bins [k0, k1): on return red[q][0], q = 0..6, hold
// unresolved bins, entries of a = 1..4, active bins, trials (all threads call)
template <int THREADS>
__device__ __forceinline__ void noniter_count_bins(const uint8_t *__restrict__ row, int64_t k0, int64_t k1,
                                                   int a_max, long long (*red)[THREADS]) {
    long long cnt[5] = {0, 0, 0, 0, 0};   // entries per a (1..4) and unresolved in [0]
    long long active = 0, tries = 0;
    for (int64_t k = k0 + threadIdx.x; k < k1; k += THREADS) {
        const uint8_t s = row[k];
        if (s == 0) continue;
        active++;
        if (s == 0xFF) {
            cnt[0]++;
            tries += a_max;
        } else {
            cnt[s] += s;
            tries += s;
        }
    }
    red[0][threadIdx.x] = cnt[0];
    red[1][threadIdx.x] = cnt[1];
    red[2][threadIdx.x] = cnt[2];
    red[3][threadIdx.x] = cnt[3];
    red[4][threadIdx.x] = cnt[4];
    red[5][threadIdx.x] = active;
    red[6][threadIdx.x] = tries;
    __syncthreads();
    for (int s = THREADS / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s)
            for (int q = 0; q < 7; q++) red[q][threadIdx.x] += red[q][threadIdx.x + s];
        __syncthreads();
    }
}

template <int THREADS>
__global__ void __launch_bounds__(THREADS) k_noniter_count(const uint8_t *__restrict__ status, int64_t L,
                                                           int a_max, int64_t nseg,
                                                           long long *__restrict__ segcnt) {
    pdl_wait();
    const int64_t b = blockIdx.x / nseg, g = blockIdx.x - b * nseg;
    const int64_t k0 = g * NONITER_SEG, k1 = (k0 + NONITER_SEG < L) ? k0 + NONITER_SEG : L;
    __shared__ long long red[7][THREADS];
    noniter_count_bins<THREADS>(status + b * L, k0, k1, a_max, red);
    if (threadIdx.x < 7) segcnt[blockIdx.x * SEGF + threadIdx.x] = red[threadIdx.x][0];
}

// the stats record of a non-iterative solve from a signal's counts r[0..6]
__device__ __forceinline__ void noniter_fill_stats(int64_t *st, const long long *r, int S, int64_t L, int64_t d) {
    const long long nent = r[1] + r[2] + r[3] + r[4];
    st[SFDT_ST_NITER] = 1;
    st[SFDT_ST_FULL_SUCCESS] = r[0] == 0;
    st[SFDT_ST_NENTRIES] = nent;
    st[SFDT_ST_NUNRESOLVED] = r[0];
    st[SFDT_ST_NDUP] = 0;
    st[SFDT_ST_SYNDROMES] = r[6] * S;
    st[SFDT_ST_FFT_SAMPLES] = int64_t(S) * L;
    int64_t *it = st + SFDT_ST_ITER0;
    it[0] = d;
    it[1] = r[5];            // attempted
    it[2] = r[5] - r[0];     // solved
    it[3] = r[0];            // deferred
    it[4] = r[6] * S;        // syndromes
    it[5] = int64_t(S) * L;  // fft samples
    // per-a entry counts for the emit pass
    st[24] = r[1];
    st[25] = r[2];
    st[26] = r[3];
    st[27] = r[4];
    // unused slots are zero: the record is a pure function of the signal
    st[7] = 0;
    for (int q = SFDT_ST_ITER0 + 6; q < 24; q++) st[q] = 0;
    for (int q = 28; q < SFDT_ST_PER_SIGNAL; q++) st[q] = 0;
}

// per signal: fold the segment counts into the stats record
__global__ void k_noniter_fin(const long long *__restrict__ segcnt, int64_t B, int64_t nseg, int64_t L,
                              int S, int64_t d, int64_t *__restrict__ stats) {
    pdl_wait();
    const int64_t b = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (b >= B) return;
    long long r[7] = {0, 0, 0, 0, 0, 0, 0};
    for (int64_t g = 0; g < nseg; g++)
        for (int q = 0; q < 7; q++) r[q] += segcnt[(b * nseg + g) * SEGF + q];
    noniter_fill_stats(stats + b * SFDT_ST_PER_SIGNAL, r, S, L, d);
}

// exclusive scans of up to three per-signal stats fields -> offsets (one
// CTA, B up to any size; out[B] = total).  Warp-shuffle block scan.
struct ScanFields {
    int field[3];
    int64_t *out[3];
    int nf;
};

__global__ void __launch_bounds__(1024) k_scan_offsets(const int64_t *__restrict__ stats, int64_t B,
                                                       ScanFields f) {
    pdl_wait();
    // thread t owns signals [t*per, (t+1)*per): its sums (independent loads,
    // one memory latency), one block scan of the thread sums, then its
    // offsets -- instead of a barrier-bound pass per 1024 signals
    __shared__ long long wtot[3][32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t per = (B + blockDim.x - 1) / blockDim.x;
    const int64_t i0 = threadIdx.x * per, i1 = (i0 + per < B) ? i0 + per : B;
    long long sum[3] = {0, 0, 0}, inc[3];
    for (int64_t i = i0; i < i1; i++)
#pragma unroll
        for (int q = 0; q < 3; q++)
            if (q < f.nf) sum[q] += stats[i * SFDT_ST_PER_SIGNAL + f.field[q]];
#pragma unroll
    for (int q = 0; q < 3; q++) {
        inc[q] = sum[q];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const long long y = __shfl_up_sync(0xffffffffu, inc[q], o);
            if (lane >= o) inc[q] += y;
        }
        if (lane == 31) wtot[q][warp] = inc[q];
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 3; q++) {
        if (q >= f.nf) continue;
        long long run = inc[q] - sum[q], total = 0;
        for (int w2 = 0; w2 < (int)(blockDim.x >> 5); w2++) {
            const long long c = wtot[q][w2];
            run += (w2 < warp) ? c : 0;
            total += c;
        }
        for (int64_t i = i0; i < i1; i++) {
            f.out[q][i] = run;
            run += stats[i * SFDT_ST_PER_SIGNAL + f.field[q]];
        }
        if (threadIdx.x == 0) f.out[q][B] = total;
    }
}

// emit entries in (a, bin) order and unresolved bins ascending.  One CTA per
// signal; each thread owns 4 consecutive bins of a tile; the per-class bin
// counts (a = 1..4 and unresolved: 5 x 12-bit fields of one uint64) get a
// single block-wide exclusive scan per tile.
__device__ __forceinline__ unsigned long long block_excl_scan_u64(unsigned long long v,
                                                                  unsigned long long *wtot,
                                                                  unsigned long long &total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    unsigned long long inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) wtot[warp] = inc;
    __syncthreads();
    unsigned long long before = 0, tot = 0;
    for (int w2 = 0; w2 < nw; w2++) {
        const unsigned long long c = wtot[w2];
        before += (w2 < warp) ? c : 0;
        tot += c;
    }
    __syncthreads();
    total = tot;
    return before + inc - v;
}

// emit the bins [k0, k1) of signal b: entries in (a, bin) order at the class
// bases base[0..3], unresolved bins ascending at base[4] (all threads call)
template <int THREADS>
__device__ __forceinline__ void noniter_emit_bins(const uint8_t *__restrict__ status,
                                                  const int64_t *__restrict__ bin_loc,
                                                  const cx *__restrict__ bin_val, int64_t L, int a_max, int64_t b,
                                                  int64_t k0, int64_t k1, const long long *base,
                                                  int64_t *__restrict__ locs, cx *__restrict__ vals,
                                                  int32_t *__restrict__ ubins, unsigned long long *wtot) {
    long long carry[5] = {0, 0, 0, 0, 0};
    for (int64_t t0 = k0; t0 < k1; t0 += THREADS * 4) {
        int ci[4];
        unsigned long long packed = 0;
#pragma unroll
        for (int u = 0; u < 4; u++) {
            const int64_t k = t0 + 4 * threadIdx.x + u;
            const uint8_t sv = (k < k1) ? status[b * L + k] : 0;
            ci[u] = (sv == 0xFF) ? 4 : (sv >= 1 && sv <= 4 ? sv - 1 : -1);
            if (ci[u] >= 0) packed += 1ull << (12 * ci[u]);
        }
        unsigned long long total;
        const unsigned long long pre = block_excl_scan_u64(packed, wtot, total);
#pragma unroll
        for (int u = 0; u < 4; u++) {
            const int c = ci[u];
            if (c < 0) continue;
            int local = 0;
            for (int u2 = 0; u2 < u; u2++) local += (ci[u2] == c);
            const long long rank = carry[c] + (long long)((pre >> (12 * c)) & 0xFFF) + local;
            const int64_t k = t0 + 4 * threadIdx.x + u;
            if (c == 4) {
                ubins[base[4] + rank] = (int32_t)k;
            } else {
                const int a = c + 1;
                const long long pos = base[c] + rank * a;
                const int64_t t = b * L + k;
                for (int j = 0; j < a; j++) {
                    locs[pos + j] = bin_loc[t * a_max + j];
                    stcx(vals + pos + j, bin_val[t * a_max + j]);
                }
            }
        }
#pragma unroll
        for (int c = 0; c < 5; c++) carry[c] += (long long)((total >> (12 * c)) & 0xFFF);
    }
}

template <int THREADS>
__global__ void __launch_bounds__(THREADS) k_noniter_emit(
    const uint8_t *__restrict__ status, const int64_t *__restrict__ bin_loc,
    const cx *__restrict__ bin_val, int64_t L, int a_max, const int64_t *__restrict__ stats,
    const int64_t *__restrict__ eoff, const int64_t *__restrict__ uoff, int64_t *__restrict__ locs,
    cx *__restrict__ vals, int32_t *__restrict__ ubins, int64_t nseg, const long long *__restrict__ segcnt) {
    pdl_wait();
    __shared__ unsigned long long wtot[THREADS / 32];
    const int64_t b = blockIdx.x / nseg, g = blockIdx.x - b * nseg;
    const int64_t *st = stats + b * SFDT_ST_PER_SIGNAL;
    long long base[5];
    base[0] = eoff[b];
    for (int c = 1; c < 4; c++) base[c] = base[c - 1] + st[24 + c - 1];
    base[4] = uoff[b];
    // segments before this one: entries per class (classes store entries,
    // so a bin of class c advances its base by c + 1) and unresolved bins
    for (int64_t g2 = 0; g2 < g; g2++) {
        const long long *sc = segcnt + (b * nseg + g2) * SEGF;
        base[4] += sc[0];
        for (int c = 0; c < 4; c++) base[c] += sc[1 + c];
    }
    const int64_t k0 = g * NONITER_SEG, k1 = (k0 + NONITER_SEG < L) ? k0 + NONITER_SEG : L;
    noniter_emit_bins<THREADS>(status, bin_loc, bin_val, L, a_max, b, k0, k1, base, locs, vals, ubins, wtot);
}

// Latency path (few signals, L <= NONITER_SEG): count, stats, offsets and
// emission of every signal in ONE CTA -- the four-kernel compaction above costs
// four launch latencies, which is most of a config-1 solve.  Same counts, same
// order, same record.
template <int THREADS>
__global__ void __launch_bounds__(THREADS) k_noniter_small(
    const uint8_t *__restrict__ status, const int64_t *__restrict__ bin_loc, const cx *__restrict__ bin_val,
    int64_t B, int64_t L, int a_max, int S, int64_t d, int64_t *__restrict__ stats, int64_t *__restrict__ eoff,
    int64_t *__restrict__ uoff, int64_t *__restrict__ doff, int64_t *__restrict__ locs, cx *__restrict__ vals,
    int32_t *__restrict__ ubins) {
    pdl_wait();
    __shared__ long long red[7][THREADS];
    __shared__ unsigned long long wtot[THREADS / 32];
    long long e_run = 0, u_run = 0;
    for (int64_t b = 0; b < B; b++) {
        noniter_count_bins<THREADS>(status + b * L, 0, L, a_max, red);
        long long r[7];
        for (int q = 0; q < 7; q++) r[q] = red[q][0];
        __syncthreads();   // red is rewritten by the next signal's count
        if (threadIdx.x == 0) {
            noniter_fill_stats(stats + b * SFDT_ST_PER_SIGNAL, r, S, L, d);
            eoff[b] = e_run;
            uoff[b] = u_run;
            if (doff) doff[b] = 0;
        }
        long long base[5];
        base[0] = e_run;
        for (int c = 1; c < 4; c++) base[c] = base[c - 1] + r[c];
        base[4] = u_run;
        noniter_emit_bins<THREADS>(status, bin_loc, bin_val, L, a_max, b, 0, L, base, locs, vals, ubins, wtot);
        e_run += r[1] + r[2] + r[3] + r[4];
        u_run += r[0];
    }
    if (threadIdx.x == 0) {
        eoff[B] = e_run;
        uoff[B] = u_run;
        if (doff) doff[B] = 0;
    }
}

// Iterative: per-signal emission in insertion order (pass, a desc, bin asc,
// root order) skipping duplicate overwrites; unresolved = deferred bins at the
// final m; duplicates listed in write order.  One CTA per signal.
template <int THREADS>
__global__ void __launch_bounds__(THREADS) k_iter_count(const IterState st, int64_t L0, int S, int a_max,
                                                        int npass, const PassInfo pi,
                                                        const double *__restrict__ resid,
                                                        const double *__restrict__ thr_last,
                                                        const int64_t *__restrict__ ndef,
                                                        int64_t *__restrict__ stats) {
    const int64_t b = blockIdx.x;
    __shared__ long long red[2][THREADS];
    long long nent = 0, ndup = 0;
    for (int p = 0; p < npass; p++) {
        const int64_t m = pi.m[p];
        for (int64_t k = threadIdx.x; k < m; k += THREADS) {
            const int64_t si = slot_index(b, p, k, L0);
            const int a = st.slot_a[si];
            const int dm = __popc(st.slot_dupmask[si]);
            nent += a - dm;
            ndup += dm;
        }
    }
    red[0][threadIdx.x] = nent;
    red[1][threadIdx.x] = ndup;
    __syncthreads();
    for (int s = THREADS / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) {
            red[0][threadIdx.x] += red[0][threadIdx.x + s];
            red[1][threadIdx.x] += red[1][threadIdx.x + s];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        int64_t *o = stats + b * SFDT_ST_PER_SIGNAL;
        long long syn = 0, fft = 0;
        for (int p = 0; p < npass; p++) {
            const unsigned long long *c = st.cnt + (b * 4 + p) * 4;
            int64_t *it = o + SFDT_ST_ITER0 + 6 * p;
            it[0] = pi.d[p];
            it[1] = (int64_t)c[0];
            it[2] = (int64_t)c[1];
            it[3] = (int64_t)c[2];
            it[4] = (int64_t)c[0] * (2 * p + 2);
            it[5] = 2 * pi.m[p];
            syn += it[4];
            fft += it[5];
        }
        for (int q = SFDT_ST_ITER0 + 6 * npass; q < SFDT_ST_PER_SIGNAL; q++) o[q] = 0;
        o[7] = 0;
        o[SFDT_ST_NITER] = npass;
        o[SFDT_ST_NENTRIES] = red[0][0];
        o[SFDT_ST_NDUP] = red[1][0];
        o[SFDT_ST_NUNRESOLVED] = ndef[b];
        o[SFDT_ST_SYNDROMES] = syn;
        o[SFDT_ST_FFT_SAMPLES] = fft;
        o[SFDT_ST_FULL_SUCCESS] = (ndef[b] == 0) && (resid[b] <= thr_last[b]);
    }
}

// Four per-class counters held in scalar registers: a runtime class index
// selects with predicated adds instead of indexing a local array (which
// ptxas places in stack memory).
struct C4 {
    long long v0 = 0, v1 = 0, v2 = 0, v3 = 0;
    __device__ __forceinline__ long long get(int c) const {
        return c == 0 ? v0 : c == 1 ? v1 : c == 2 ? v2 : v3;
    }
    __device__ __forceinline__ void add(int c, long long x) {
        v0 += (c == 0) ? x : 0;
        v1 += (c == 1) ? x : 0;
        v2 += (c == 2) ? x : 0;
        v3 += (c == 3) ? x : 0;
    }
    __device__ __forceinline__ void set(int c, long long x) {
        v0 = (c == 0) ? x : v0;
        v1 = (c == 1) ? x : v1;
        v2 = (c == 2) ? x : v2;
        v3 = (c == 3) ? x : v3;
    }
};

// Per-lane chunk of up to 32 consecutive bytes (bins t0 + lane*cb ..) held
// in eight 32-bit registers; cb is a power of two <= 32.
struct Chunk32 {
    uint32_t w[8];
    __device__ __forceinline__ int at(int i) const { return (w[i >> 2] >> (8 * (i & 3))) & 0xFF; }
};

__device__ __forceinline__ void load_chunk(const uint8_t *__restrict__ src, int cb, bool valid, Chunk32 &c) {
#pragma unroll
    for (int q = 0; q < 8; q++) c.w[q] = 0;
    if (!valid) return;
    if (cb >= 16) {
        const uint4 *v = reinterpret_cast<const uint4 *>(src);
        const uint4 u0 = __ldg(v);
        c.w[0] = u0.x; c.w[1] = u0.y; c.w[2] = u0.z; c.w[3] = u0.w;
        if (cb == 32) {
            const uint4 u1 = __ldg(v + 1);
            c.w[4] = u1.x; c.w[5] = u1.y; c.w[6] = u1.z; c.w[7] = u1.w;
        }
    } else if (cb >= 4) {
        const uint32_t *v = reinterpret_cast<const uint32_t *>(src);
        c.w[0] = __ldg(v);
        if (cb == 8) c.w[1] = __ldg(v + 1);
    } else {
        uint32_t x = 0;
        for (int i = 0; i < cb; i++) x |= (uint32_t)__ldg(src + i) << (8 * i);
        c.w[0] = x;
    }
}

__device__ __forceinline__ unsigned long long warp_incl_scan_u64(unsigned long long v, int lane) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += y;
    }
    return v;
}

// Iterative emission: per pass p the entries of bins accepted with a_try =
// p+1, p, ..., 1 in bin order (non-duplicate entries to the spectrum, the
// duplicate overwrites to the warning list), then the unresolved bins.
// One WARP per signal (no block barriers; 8 signals per CTA keep the SM's
// memory pipeline full): a lane owns a contiguous chunk of up to 32 bins of
// a 1024-bin tile, read as 16-byte vectors; one packed warp scan (4 classes
// x 16-bit fields) per tile places every entry.  Passes whose m exceeds one
// tile take a counting sweep first for the class bases.
template <int THREADS>
__global__ void __launch_bounds__(THREADS) k_iter_emit(
    const IterState st, int64_t B, int64_t L0, int a_max, int npass, const PassInfo pi, int64_t m_final,
    const int64_t *__restrict__ eoff, const int64_t *__restrict__ uoff,
    const int64_t *__restrict__ doff, int64_t *__restrict__ locs, cx *__restrict__ vals,
    int32_t *__restrict__ ubins, int64_t *__restrict__ dups) {
    constexpr int TILE = 1024;
    const int lane = threadIdx.x & 31;
    const int64_t b = (int64_t)blockIdx.x * (THREADS / 32) + (threadIdx.x >> 5);
    if (b >= B) return;
    long long carry_e = eoff[b], carry_d = doff ? doff[b] : 0;
    for (int p = 0; p < npass; p++) {
        const int64_t m = p == 0 ? pi.m[0] : p == 1 ? pi.m[1] : p == 2 ? pi.m[2] : pi.m[3];
        const int64_t tile = m < TILE ? m : TILE;
        const int cb = tile >= 32 ? (int)(tile >> 5) : 1;
        const uint8_t *sa = st.slot_a + slot_index(b, p, 0, L0);
        const uint8_t *sd = st.slot_dupmask + slot_index(b, p, 0, L0);
        auto counts = [&](const Chunk32 &ca, const Chunk32 &cd, unsigned long long &pe,
                          unsigned long long &pd) {
            pe = 0;
            pd = 0;
#pragma unroll
            for (int i = 0; i < 32; i++) {
                if (i < cb) {
                    const int a = ca.at(i);
                    if (a) {
                        const int dn = __popc(cd.at(i));
                        pe += (unsigned long long)(a - dn) << (16 * (a - 1));
                        pd += (unsigned long long)dn << (16 * (a - 1));
                    }
                }
            }
        };
        Chunk32 ca, cd;
        unsigned long long pe, pd;
        C4 tot_e, tot_d;
        if (m > TILE) {           // counting sweep for the class bases
            for (int64_t t0 = 0; t0 < m; t0 += TILE) {
                const int64_t k0 = t0 + (int64_t)lane * cb;
                load_chunk(sa + k0, cb, true, ca);
                load_chunk(sd + k0, cb, true, cd);
                counts(ca, cd, pe, pd);
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    pe += __shfl_xor_sync(0xffffffffu, pe, o);
                    pd += __shfl_xor_sync(0xffffffffu, pd, o);
                }
#pragma unroll
                for (int c = 0; c < 4; c++) {
                    tot_e.add(c, (long long)((pe >> (16 * c)) & 0xFFFF));
                    tot_d.add(c, (long long)((pd >> (16 * c)) & 0xFFFF));
                }
            }
        }
        C4 base_e, base_d, acc_e, acc_d;
        for (int64_t t0 = 0; t0 < m; t0 += TILE) {
            const int64_t k0 = t0 + (int64_t)lane * cb;
            const bool valid = k0 < m;
            load_chunk(sa + k0, cb, valid, ca);
            load_chunk(sd + k0, cb, valid, cd);
            counts(ca, cd, pe, pd);
            const unsigned long long ie = warp_incl_scan_u64(pe, lane);
            const unsigned long long id = warp_incl_scan_u64(pd, lane);
            const unsigned long long te = __shfl_sync(0xffffffffu, ie, 31);
            const unsigned long long td = __shfl_sync(0xffffffffu, id, 31);
            if (t0 == 0) {
                if (m <= TILE) {
#pragma unroll
                    for (int c = 0; c < 4; c++) {
                        tot_e.set(c, (long long)((te >> (16 * c)) & 0xFFFF));
                        tot_d.set(c, (long long)((td >> (16 * c)) & 0xFFFF));
                    }
                }
                long long ce = carry_e, cdd = carry_d;
#pragma unroll
                for (int c = 3; c >= 0; c--) {
                    base_e.set(c, ce);
                    base_d.set(c, cdd);
                    if (c <= p) {
                        ce += tot_e.get(c);
                        cdd += tot_d.get(c);
                    }
                }
                carry_e = ce;
                carry_d = cdd;
            }
            unsigned long long oe = ie - pe, od = id - pd;   // exclusive, packed
            if (pe | pd) {
#pragma unroll
                for (int i = 0; i < 32; i++) {
                    if (i < cb) {
                        const int a = ca.at(i);
                        if (a) {
                            const int c = a - 1, dm = cd.at(i);
                            long long pe_ = base_e.get(c) + acc_e.get(c) + (long long)((oe >> (16 * c)) & 0xFFFF);
                            long long pd_ = base_d.get(c) + acc_d.get(c) + (long long)((od >> (16 * c)) & 0xFFFF);
                            const int64_t si = slot_index(b, p, k0 + i, L0);
                            const int dn = __popc(dm);
                            for (int j = 0; j < a; j++) {
                                const int64_t loc = st.slot_loc[si * a_max + j];
                                if (dm & (1 << j)) {
                                    if (dups) dups[pd_] = loc;
                                    pd_++;
                                } else {
                                    locs[pe_] = loc;
                                    stcx(vals + pe_, st.slot_val[si * a_max + j]);
                                    pe_++;
                                }
                            }
                            oe += (unsigned long long)(a - dn) << (16 * c);
                            od += (unsigned long long)dn << (16 * c);
                        }
                    }
                }
            }
#pragma unroll
            for (int c = 0; c < 4; c++) {
                acc_e.add(c, (long long)((te >> (16 * c)) & 0xFFFF));
                acc_d.add(c, (long long)((td >> (16 * c)) & 0xFFFF));
            }
        }
    }
    // unresolved = deferred bins at the final m, ascending
    {
        const int64_t tile = m_final < TILE ? m_final : TILE;
        const int cb = tile >= 32 ? (int)(tile >> 5) : 1;
        long long carry_u = uoff[b];
        Chunk32 cf;
        for (int64_t t0 = 0; t0 < m_final; t0 += TILE) {
            const int64_t k0 = t0 + (int64_t)lane * cb;
            load_chunk(st.deferred + b * L0 + k0, cb, k0 < m_final, cf);
            unsigned long long cnt = 0;
#pragma unroll
            for (int q = 0; q < 8; q++) cnt += __popc(cf.w[q]);   // flags are 0/1 bytes
            const unsigned long long inc = warp_incl_scan_u64(cnt, lane);
            long long pos = carry_u + (long long)(inc - cnt);
            if (cnt) {
#pragma unroll
                for (int i = 0; i < 32; i++)
                    if (i < cb && cf.at(i)) ubins[pos++] = (int32_t)(k0 + i);
            }
            carry_u += (long long)__shfl_sync(0xffffffffu, inc, 31);
        }
    }
}

// ------------------------------------------------------------- host side
static inline size_t align_up(size_t v) { return (v + 255) & ~size_t(255); }

struct ExactPlan {
    int64_t B, n, d, L, S, CH, nchunk, npass;
    int logd;
    size_t off_V, off_partial, off_thr, off_status, off_bloc, off_bval, off_def,
        off_sloc, off_sval, off_sa, off_sdup, off_cnt, off_resid, off_ndef, off_scratch, off_fft, off_wl, off_wl2,
        off_act, off_awl, off_seg,
        total;
};

static int make_plan(const sfdt_exact_args *a, ExactPlan &p) {
    if (!a || a->batch < 1 || a->n < 2 || (a->n & (a->n - 1))) return SFDT_EINVAL;
    if (a->a_max < 1 || a->a_max > 4 || a->d < 1 || a->d > a->n || (a->d & (a->d - 1)))
        return SFDT_EINVAL;
    if (a->x_dtype != SFDT_C128 && a->x_dtype != SFDT_C64) return SFDT_EINVAL;
    p.B = a->batch;
    p.n = a->n;
    p.d = a->d;
    p.logd = ilog2_64(a->d);
    p.L = a->n / a->d;
    p.S = 2 * a->a_max;
    p.CH = a->n < 16384 ? a->n : 16384;
    p.nchunk = a->n / p.CH;
    p.npass = a->iterative ? a->a_max : 1;
    size_t o = 0;
    auto take = [&](size_t bytes) { size_t r = o; o = align_up(o + bytes); return r; };
    p.off_V = take(size_t(p.B) * p.L * p.S * 16);
    p.off_partial = take(size_t(p.B) * p.nchunk * 8);
    p.off_thr = take(size_t(p.B) * 5 * 8);
    if (!a->iterative) {
        p.off_status = take(size_t(p.B) * p.L);
        p.off_bloc = take(size_t(p.B) * p.L * a->a_max * 8);
        p.off_bval = take(size_t(p.B) * p.L * a->a_max * 16);
        p.off_wl = take(size_t(p.B) * p.L * 8);
        p.off_wl2 = take(size_t(p.B) * p.L * 8);
        p.off_act = take(size_t(p.B) * p.L);
        p.off_awl = take(size_t(p.B) * p.L * 8);
        p.off_seg = take(size_t(p.B) * ((p.L + NONITER_SEG - 1) / NONITER_SEG) * SEGF * 8);
    } else {
        p.off_def = take(size_t(p.B) * p.L);
        p.off_sloc = take(size_t(p.B) * 4 * p.L * a->a_max * 8);
        p.off_sval = take(size_t(p.B) * 4 * p.L * a->a_max * 16);
        p.off_sa = take(size_t(p.B) * 4 * p.L);
        p.off_sdup = take(size_t(p.B) * 4 * p.L);
        p.off_cnt = take(size_t(p.B) * 16 * 8);
        p.off_resid = take(size_t(p.B) * 8);
        p.off_ndef = take(size_t(p.B) * 8);
        p.off_awl = take(size_t(p.B) * p.L * 8);
    }
    p.off_scratch = take(192 * 8);
    p.off_fft = (p.L > FFT_SMEM_MAX) ? take(size_t(p.B) * p.L * p.S * 16) : 0;
    p.total = o;
    return SFDT_OK;
}

}  // namespace sfdt

using namespace sfdt;

extern "C" int sfdt_exact_caps(const sfdt_exact_args *a, int64_t *entry_cap, int64_t *unres_cap,
                               int64_t *dup_cap) {
    ExactPlan p;
    int rc = make_plan(a, p);
    if (rc) return rc;
    // every bin yields at most a_max entries per pass; unresolved <= L
    if (entry_cap) *entry_cap = p.B * p.L * a->a_max * (a->iterative ? 2 : 1);
    if (unres_cap) *unres_cap = p.B * p.L;
    if (dup_cap) *dup_cap = a->iterative ? p.B * p.L * a->a_max * 2 : 0;
    return SFDT_OK;
}

extern "C" size_t sfdt_exact_workspace_bytes(const sfdt_exact_args *a) {
    ExactPlan p;
    if (make_plan(a, p)) return 0;
    return p.total;
}

extern "C" int sfdt_exact_solve(sfdt_exact_args *a, void *ws, size_t ws_bytes,
                                sfdt_stream_t stream_) {
    ExactPlan p;
    int rc = make_plan(a, p);
    if (rc) return rc;
    if (ws_bytes < p.total || !ws) return SFDT_EWORKSPACE;
    int64_t ecap, ucap, dcap;
    sfdt_exact_caps(a, &ecap, &ucap, &dcap);
    if (a->entry_cap < ecap || a->unres_cap < ucap || (a->iterative && a->dup_locs && a->dup_cap < dcap))
        return SFDT_ECAPACITY;
    cudaStream_t stream = (cudaStream_t)stream_;
    const sfdt_tuning tn = tuning_or_default(a->tuning);
    char *w = (char *)ws;
    cx *V = (cx *)(w + p.off_V);
    double *partial = (double *)(w + p.off_partial);
    double *thr = (double *)(w + p.off_thr);
    cx *fft_scratch = p.off_fft ? (cx *)(w + p.off_fft) : nullptr;

    int launches = 0;
    const int is_c64 = a->x_dtype == SFDT_C64;
    // With an aux stream the stream kernel runs one 1024-thread CTA per SM
    // (a dynamic shared-memory reservation caps residency): measured on B200
    // to hold the full 7.55 TB/s read rate (tools/membw.cu) while leaving half
    // of every SM's threads and shared memory to the FFT/decode of the
    // previous chunk.
    const bool reserve = a->aux_stream != nullptr;
    const DecodeScratch no_scratch{nullptr, 0, nullptr, nullptr, nullptr};
    auto launch_stream = [&](int64_t c0, int64_t bc, DecodeScratch zc) -> int {
        dim3 grid((unsigned)p.nchunk, (unsigned)bc);
        const char *xc = (const char *)a->x + c0 * p.n * (is_c64 ? 8 : 16);
        if (reserve) {
            constexpr int TH = 1024, UN = 4, SMEM = 120000;
            int dev = 0, sms = 148;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            const int64_t nitems = p.nchunk * bc;
            const unsigned g = (unsigned)(nitems < sms ? nitems : sms);
            if (is_c64) {
                cudaFuncSetAttribute(k_sumsq_persistent<1, TH, UN>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
                k_sumsq_persistent<1, TH, UN><<<g, TH, SMEM, stream>>>(xc, p.n, p.CH, p.nchunk, nitems,
                                                                       partial + c0 * p.nchunk);
            } else {
                cudaFuncSetAttribute(k_sumsq_persistent<0, TH, UN>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
                k_sumsq_persistent<0, TH, UN><<<g, TH, SMEM, stream>>>(xc, p.n, p.CH, p.nchunk, nitems,
                                                                       partial + c0 * p.nchunk);
            }
        } else {
            constexpr int TH = 512, UN = 4;
            if (is_c64)
                launch_pdl(k_sumsq<1, TH, UN>, grid, dim3(TH), 0, stream, (const void *)xc, p.n, p.CH,
                           partial + c0 * p.nchunk, zc);
            else
                launch_pdl(k_sumsq<0, TH, UN>, grid, dim3(TH), 0, stream, (const void *)xc, p.n, p.CH,
                           partial + c0 * p.nchunk, zc);
        }
        SFDT_CHECK_LAUNCH();
        launches += 1;
        return SFDT_OK;
    };

    if (!a->iterative) {
        // Pipeline over signal chunks: the HBM-bound stream kernel of chunk
        // c+1 (main stream) runs concurrently with the latency-bound FFT +
        // decode of chunk c (aux stream).
        cudaStream_t aux = a->aux_stream ? (cudaStream_t)a->aux_stream : stream;
        int64_t bc = p.B;
        if (a->aux_stream) {
            bc = a->chunk_signals > 0 ? a->chunk_signals : (p.B + 15) / 16;
            const int64_t min_bc = (p.B + 63) / 64;   // <= 64 chunk counters
            if (bc < min_bc) bc = min_bc;
        }
        const int64_t nc = (p.B + bc - 1) / bc;
        uint8_t *status = (uint8_t *)(w + p.off_status);
        int64_t *bloc = (int64_t *)(w + p.off_bloc);
        cx *bval = (cx *)(w + p.off_bval);
        int64_t *wl = (int64_t *)(w + p.off_wl);
        int64_t *wl2 = (int64_t *)(w + p.off_wl2);
        unsigned long long *wlc = (unsigned long long *)(w + p.off_scratch);
        cudaEvent_t ev_done = nullptr;
        if (a->ev_stream_begin) cudaEventRecord((cudaEvent_t)a->ev_stream_begin, stream);
        if (aux != stream) {   // aux work may start only after everything queued before this call
            cudaEvent_t ev;
            if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess) return SFDT_ECUDA;
            cudaEventRecord(ev, stream);
            cudaStreamWaitEvent(aux, ev, 0);
            cudaEventDestroy(ev);
        }
        // Latency path (a few short signals, config 1): five or six kernels
        // instead of ten -- the stream kernel zeroes the counters, the a = 1
        // decode folds the rms tree and the activity test in, and one CTA
        // compacts.  Same arithmetic, same bits.
        const bool small = tn.latency_path != 0 && aux == stream && !a->rms_in && p.nchunk <= 64 &&
                           (p.L % 32) == 0 && p.L <= NONITER_SEG && p.B <= (tn.latency_path > 0 ? 64 : 8);
        if (small) {
            if ((rc = launch_stream(0, p.B, DecodeScratch{nullptr, 0, wlc, wlc + 64, wlc + 128}))) return rc;
            if (a->ev_stream_end) cudaEventRecord((cudaEvent_t)a->ev_stream_end, stream);
            const ViewSrc src = consecutive_views((const char *)a->x, is_c64, p.n, p.d, 0, (int)p.S);
            rc = launch_fft_views(src, p.B, p.L, a->twiddles, V, (int)p.S, p.L, stream, fft_scratch, 1, nullptr,
                                  nullptr, tn.fft_split);
            if (rc) return rc;
            switch (p.S) {
#define SFDT_SMALL(Sv)                                                                                            \
    rc = launch_decode_small<Sv>(V, p.B, p.L, a->a_max, p.n, partial, p.nchunk, a->zero_threshold, p.d, a->rms, \
                                 thr, status, bloc, bval, wl, wlc, wl2, wlc + 128, tn.decode_coop, stream);
            case 2: SFDT_SMALL(2) break;
            case 4: SFDT_SMALL(4) break;
            case 6: SFDT_SMALL(6) break;
            default: SFDT_SMALL(8) break;
#undef SFDT_SMALL
            }
            if (rc) return rc;
            launch_pdl(k_noniter_small<256>, dim3(1), dim3(256), 0, stream, (const uint8_t *)status,
                       (const int64_t *)bloc, (const cx *)bval, p.B, p.L, a->a_max, (int)p.S, p.d, a->stats,
                       a->entry_offsets, a->unres_offsets, a->dup_offsets, a->locs, (cx *)a->vals, a->unres_bins);
            SFDT_CHECK_LAUNCH();
            launches += fft_view_launches(p.L, tn.fft_split) + 2 +
                        (a->a_max > 1 ? (decode_coop_mode(tn.decode_coop, p.B * p.L, a->a_max) == 2 ? 3 : 1) : 0);
            a->kernel_launches = launches;
            return SFDT_OK;
        }
        for (int64_t c = 0; c < nc; c++) {
            const int64_t c0 = c * bc, nb = (c0 + bc <= p.B) ? bc : p.B - c0;
            // the views need no rms: their gather + FFT (aux) overlaps the
            // HBM stream of the same chunk (main)
            auto launch_fft = [&]() -> int {
                const ViewSrc src = consecutive_views((const char *)a->x + c0 * p.n * (is_c64 ? 8 : 16), is_c64,
                                                      p.n, p.d, 0, (int)p.S);
                return launch_fft_views(src, nb, p.L, a->twiddles, V + c0 * p.S * p.L, (int)p.S, p.L,
                                        aux, fft_scratch ? fft_scratch + c0 * p.S * p.L : nullptr, 1, nullptr,
                                        nullptr, tn.fft_split);
            };
            const bool overlap = aux != stream;
            if (overlap && (rc = launch_fft())) return rc;
            if (!a->rms_in && (rc = launch_stream(c0, nb, no_scratch))) return rc;
            if (c == nc - 1 && a->ev_stream_end) cudaEventRecord((cudaEvent_t)a->ev_stream_end, stream);
            if (aux != stream) {
                cudaEvent_t ev;
                if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess) return SFDT_ECUDA;
                cudaEventRecord(ev, stream);
                cudaStreamWaitEvent(aux, ev, 0);
                cudaEventDestroy(ev);
            }
            // after the rms the FFT epilogue can also mark the active bins;
            // the rms kernel zeroes their flags and the worklist counters
            const bool dense = !overlap;
            uint8_t *actc = dense ? (uint8_t *)(w + p.off_act) + c0 * p.L : nullptr;
            const DecodeScratch zs = dense ? DecodeScratch{actc, p.L, wlc + c, wlc + 64 + c, wlc + 128 + c}
                                           : DecodeScratch{nullptr, 0, nullptr, nullptr, nullptr};
            if (a->rms_in)
                launch_pdl(k_thr_from_rms, dim3((unsigned)((nb + 255) / 256)), dim3(256), 0, aux,
                           (const double *)(a->rms_in + c0), nb, a->zero_threshold, p.d, a->rms + c0, thr + c0, zs);
            else
                launch_rms(partial + c0 * p.nchunk, nb, p.nchunk, p.n, a->zero_threshold, p.d, a->rms + c0,
                           thr + c0, aux, zs);
            SFDT_CHECK_LAUNCH();
            if (!overlap) {
                const ViewSrc src = consecutive_views((const char *)a->x + c0 * p.n * (is_c64 ? 8 : 16), is_c64,
                                                      p.n, p.d, 0, (int)p.S);
                rc = launch_fft_views(src, nb, p.L, a->twiddles, V + c0 * p.S * p.L, (int)p.S, p.L, aux,
                                      fft_scratch ? fft_scratch + c0 * p.S * p.L : nullptr, 1,
                                      thr + c0, actc, tn.fft_split);
                if (rc) return rc;
            }
            int64_t *awlc_p = (int64_t *)(w + p.off_awl) + c0 * p.L;
            const cx *Vc = V + c0 * p.S * p.L;
            uint8_t *stc = status + c0 * p.L;
            int64_t *blc = bloc + c0 * p.L * a->a_max;
            cx *bvc = bval + c0 * p.L * a->a_max;
            switch (p.S) {
            case 2: rc = launch_decode_noniter<2>(Vc, nb, p.L, a->a_max, p.n, thr + c0, stc, blc, bvc, wl + c0 * p.L, wlc + c, aux, actc, awlc_p, wlc + 64 + c, wl2 + c0 * p.L, wlc + 128 + c, tn.decode_coop); break;
            case 4: rc = launch_decode_noniter<4>(Vc, nb, p.L, a->a_max, p.n, thr + c0, stc, blc, bvc, wl + c0 * p.L, wlc + c, aux, actc, awlc_p, wlc + 64 + c, wl2 + c0 * p.L, wlc + 128 + c, tn.decode_coop); break;
            case 6: rc = launch_decode_noniter<6>(Vc, nb, p.L, a->a_max, p.n, thr + c0, stc, blc, bvc, wl + c0 * p.L, wlc + c, aux, actc, awlc_p, wlc + 64 + c, wl2 + c0 * p.L, wlc + 128 + c, tn.decode_coop); break;
            default: rc = launch_decode_noniter<8>(Vc, nb, p.L, a->a_max, p.n, thr + c0, stc, blc, bvc, wl + c0 * p.L, wlc + c, aux, actc, awlc_p, wlc + 64 + c, wl2 + c0 * p.L, wlc + 128 + c, tn.decode_coop); break;
            }
            if (rc) return rc;
            launches += 1 + fft_view_launches(p.L, tn.fft_split) + 1 + (dense ? 1 : 0) +
                        (a->a_max > 1 ? (decode_coop_mode(tn.decode_coop, nb * p.L, a->a_max) == 2 ? 3 : 1) : 0);
        }
        if (aux != stream) {
            if (cudaEventCreateWithFlags(&ev_done, cudaEventDisableTiming) != cudaSuccess) return SFDT_ECUDA;
            cudaEventRecord(ev_done, aux);
            cudaStreamWaitEvent(stream, ev_done, 0);
            cudaEventDestroy(ev_done);
        }
        const int64_t nseg = (p.L + NONITER_SEG - 1) / NONITER_SEG;
        long long *segcnt = (long long *)(w + p.off_seg);
        launch_pdl(k_noniter_count<256>, dim3((unsigned)(p.B * nseg)), dim3(256), 0, stream, (const uint8_t *)status,
                   p.L, a->a_max, nseg, segcnt);
        launch_pdl(k_noniter_fin, dim3((unsigned)((p.B + 255) / 256)), dim3(256), 0, stream,
                   (const long long *)segcnt, p.B, nseg, p.L, (int)p.S, p.d, a->stats);
        SFDT_CHECK_LAUNCH();
        {
            ScanFields f{{SFDT_ST_NENTRIES, SFDT_ST_NUNRESOLVED, 0}, {a->entry_offsets, a->unres_offsets, nullptr}, 2};
            launch_pdl(k_scan_offsets, dim3(1), dim3(1024), 0, stream, (const int64_t *)a->stats, p.B, f);
        }
        SFDT_CHECK_LAUNCH();
        launch_pdl(k_noniter_emit<256>, dim3((unsigned)(p.B * nseg)), dim3(256), 0, stream, (const uint8_t *)status,
                   (const int64_t *)bloc, (const cx *)bval, p.L, a->a_max, (const int64_t *)a->stats,
                   (const int64_t *)a->entry_offsets, (const int64_t *)a->unres_offsets, a->locs, (cx *)a->vals,
                   a->unres_bins, nseg, (const long long *)segcnt);
        SFDT_CHECK_LAUNCH();
        if (a->dup_offsets) cudaMemsetAsync(a->dup_offsets, 0, sizeof(int64_t) * (p.B + 1), stream);
        launches += 4;   // count, fin, scan, emit
        a->kernel_launches = launches;
        return SFDT_OK;
    }

    // iterative: the single pass over x first (all signals), then the passes
    if (a->ev_stream_begin) cudaEventRecord((cudaEvent_t)a->ev_stream_begin, stream);
    if (!a->rms_in && (rc = launch_stream(0, p.B, no_scratch))) return rc;
    if (a->ev_stream_end) cudaEventRecord((cudaEvent_t)a->ev_stream_end, stream);
    if (a->rms_in)
        k_thr_from_rms<<<(unsigned)((p.B + 255) / 256), 256, 0, stream>>>(a->rms_in, p.B, a->zero_threshold,
                                                                          p.d, a->rms, thr,
                                                                          DecodeScratch{nullptr, 0, nullptr, nullptr, nullptr});
    else
        launch_rms(partial, p.B, p.nchunk, p.n, a->zero_threshold, p.d, a->rms, thr, stream);
    SFDT_CHECK_LAUNCH();
    launches += 1;

    // iterative: thresholds per pass (zt * rms * d_l), d_l = min(d0 * 2^l, n)
    IterState st;
    st.V = V;
    st.deferred = (uint8_t *)(w + p.off_def);
    st.slot_loc = (int64_t *)(w + p.off_sloc);
    st.slot_val = (cx *)(w + p.off_sval);
    st.slot_a = (uint8_t *)(w + p.off_sa);
    st.slot_dupmask = (uint8_t *)(w + p.off_sdup);
    st.cnt = (unsigned long long *)(w + p.off_cnt);
    cudaMemsetAsync(st.deferred, 0, size_t(p.B) * p.L, stream);
    cudaMemsetAsync(st.slot_a, 0, size_t(p.B) * 4 * p.L, stream);
    cudaMemsetAsync(st.slot_dupmask, 0, size_t(p.B) * 4 * p.L, stream);
    cudaMemsetAsync(st.cnt, 0, size_t(p.B) * 16 * 8, stream);
    PassInfo pi;
    int64_t *m_of = pi.m, *d_of = pi.d;
    int64_t d = p.d;
    for (int l = 0; l < 4; l++) {
        d_of[l] = d;
        m_of[l] = p.n / d;
        if (l < p.npass && d < p.n) d *= 2;
    }
    // thr layout: [0..B) rms-based base threshold at d0 (from k_rms), then one
    // row per pass with zt*rms*d_l
    for (int l = 0; l < p.npass; l++) {
        k_scale_thr<<<(unsigned)((p.B + 255) / 256), 256, 0, stream>>>(a->rms, p.B, a->zero_threshold,
                                                                      d_of[l], thr + p.B * (l + 1));
        SFDT_CHECK_LAUNCH();
    }
    for (int l = 0; l < p.npass; l++) {
        const int64_t m = m_of[l];
        const ViewSrc src = consecutive_views(a->x, is_c64, p.n, d_of[l], 2 * l, 2);
        rc = launch_fft_views(src, p.B, m, a->twiddles, V + 2 * l * p.L, (int)p.S, p.L, stream,
                              fft_scratch, 1, nullptr, nullptr, tn.fft_split);
        if (rc) return rc;
        const int fold = (l > 0) && (m != m_of[l - 1]);
        const int64_t nb = p.B * m;
        int64_t *awl = (int64_t *)(w + p.off_awl);
        unsigned long long *awlc = (unsigned long long *)(w + p.off_scratch) + 64 + l;
        cudaMemsetAsync(awlc, 0, 8, stream);
        k_iter_prep<<<(unsigned)((nb + 255) / 256), 256, 0, stream>>>(st, p.B, p.L, (int)p.S, a->a_max, l, p.n,
                                                                      m, fold, thr, awl, awlc);
        SFDT_CHECK_LAUNCH();
        {
            int dev = 0, sms = 148;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            (void)sms;
            switch (l) {
#define SFDT_ITD(Lv)                                                                                  \
    k_iter_decode<Lv><<<wl_grid(nb, 128, one_wave(k_iter_decode<Lv>, 128)), 128, 0, stream>>>(          \
        st, p.L, (int)p.S, a->a_max, p.n, m, awl, awlc);
            case 0: SFDT_ITD(0) break;
            case 1: SFDT_ITD(1) break;
            case 2: SFDT_ITD(2) break;
            default: SFDT_ITD(3) break;
#undef SFDT_ITD
            }
            SFDT_CHECK_LAUNCH();
        }
    }
    double *resid = (double *)(w + p.off_resid);
    int64_t *ndef = (int64_t *)(w + p.off_ndef);
    const int64_t m_final = m_of[p.npass - 1];
    k_iter_final<<<(unsigned)p.B, 256, 0, stream>>>(V, st.deferred, p.L, (int)p.S, m_final, resid, ndef);
    SFDT_CHECK_LAUNCH();
    k_iter_count<256><<<(unsigned)p.B, 256, 0, stream>>>(st, p.L, (int)p.S, a->a_max, (int)p.npass,
                                                         pi, resid,
                                                         thr + p.B * p.npass, ndef, a->stats);
    SFDT_CHECK_LAUNCH();
    {
        ScanFields f{{SFDT_ST_NENTRIES, SFDT_ST_NUNRESOLVED, SFDT_ST_NDUP},
                     {a->entry_offsets, a->unres_offsets, a->dup_offsets}, a->dup_offsets ? 3 : 2};
        k_scan_offsets<<<1, 1024, 0, stream>>>(a->stats, p.B, f);
    }
    SFDT_CHECK_LAUNCH();
    k_iter_emit<256><<<(unsigned)((p.B + 7) / 8), 256, 0, stream>>>(st, p.B, p.L, a->a_max, (int)p.npass, pi,
                                                        m_final, a->entry_offsets, a->unres_offsets,
                                                        a->dup_offsets ? a->dup_offsets : nullptr,
                                                        a->locs, (cx *)a->vals, a->unres_bins,
                                                        a->dup_locs);
    SFDT_CHECK_LAUNCH();
    launches += (int)p.npass * (1 + 2 + fft_view_launches(p.L, tn.fft_split)) + 1 + 1 + 1 + 1;   // final, count, scan, emit
    a->kernel_launches = launches;
    return SFDT_OK;
}

// ------------------------------------------------------------ rms mirror
// spectral.py:215-218 rms(x) for a batch of signals: the solver's own HBM
// pass (k_sumsq over 16384-sample chunks, fixed-order tree), so a caller of
// rms() gets exactly the value the solvers threshold with.
extern "C" size_t sfdt_rms_workspace_bytes(int64_t batch, int64_t n) {
    if (batch < 1 || n < 1) return 256;
    const int64_t CH = n < 16384 ? n : 16384;
    return size_t(batch) * size_t((n + CH - 1) / CH) * 8 + size_t(batch) * 8 + 256;
}

extern "C" int sfdt_rms(const void *x, int32_t x_dtype, int64_t batch, int64_t n, double *out, void *ws,
                        size_t ws_bytes, sfdt_stream_t stream_) {
    if (batch < 0 || n < 2 || (n & (n - 1)) || (x_dtype != SFDT_C128 && x_dtype != SFDT_C64)) return SFDT_EINVAL;
    if (batch == 0) return SFDT_OK;
    if (!ws || ws_bytes < sfdt_rms_workspace_bytes(batch, n)) return SFDT_EWORKSPACE;
    cudaStream_t stream = (cudaStream_t)stream_;
    const int64_t CH = n < 16384 ? n : 16384, nchunk = n / CH;
    double *partial = (double *)ws;
    double *thr = partial + batch * nchunk;
    constexpr int TH = 512, UN = 4;
    const dim3 grid((unsigned)nchunk, (unsigned)batch);
    if (x_dtype == SFDT_C64)
        k_sumsq<1, TH, UN><<<grid, TH, 0, stream>>>(x, n, CH, partial, DecodeScratch{nullptr, 0, nullptr, nullptr, nullptr});
    else
        k_sumsq<0, TH, UN><<<grid, TH, 0, stream>>>(x, n, CH, partial, DecodeScratch{nullptr, 0, nullptr, nullptr, nullptr});
    SFDT_CHECK_LAUNCH();
    launch_rms(partial, batch, nchunk, n, 0.0, 1, out, thr, stream);
    SFDT_CHECK_LAUNCH();
    return SFDT_OK;
}
