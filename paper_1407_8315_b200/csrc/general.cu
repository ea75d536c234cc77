// general.cu -- sm_100a kernels of the generally-K-sparse path
// (general.py:272-372, solve_general).
//
//   views        2*a_max consecutive + r_eff random-shift views gathered from
//                x and FFT'd in shared memory (fft.cuh), bit-exact
//   k_gen_svd    thread per bin: singular values of the a_max x a_max Hankel
//                matrix (one-sided Jacobi, _core.pyx:353-433) + |syn|^2 partials
//   k_gen_vote   CTA per signal: the pooled top-K vote of estimate_collisions
//                (general.py:131-155): exact radix select of the K-th largest
//                singular value, ties by (bin, rank) ascending, zero-vote guard,
//                cap, histogram, worklist of voted bins
//   k_gen_bins   thread per voted bin: descending-order Hankel fit, candidate
//                evaluation |P(z_t)| over the d candidates (prune_eval), the
//                correlation fallback, matched-filter union (general.py:313-351)
//                and subspace pursuit with gelsd-semantics least squares
//                (general.py:224-269, 357-366)
//   count/scan/emit  compact (loc, value) lists in dict insertion order
//                (vote class a ascending, bin ascending, column ascending)
#include <climits>
#include <mutex>
#include <cstdlib>
#include <type_traits>

#ifndef SFDT_SP_TMAX
#define SFDT_SP_TMAX 4   // largest least-squares support with a register-resident instance
#endif

#include "common.cuh"
#include "decode.cuh"
#include "fft.cuh"
#include "general.cuh"
#ifdef SFDT_BINS_PROFILE
#include <cstdio>
#endif

namespace sfdt {

struct GenParams {
    int64_t n, d, L, k;
    int a_max, r_eff, keep, prune, S, nv;
    double zvr;
    const int64_t *shifts;
    int64_t shift_stride;
    const cx *base_phi;
    int64_t phi_stride;
    // view slot of random view j of signal b: vslot[b * r_eff + j] (< S when
    // its shift equals a consecutive shift, whose view it then shares)
    const int32_t *vslot;
};

// row of random view j (shift shifts[j]) of signal b at bin kb
__device__ __forceinline__ const cx *rview(const cx *V, const GenParams &p, int64_t b, int j, int64_t kb) {
    return V + (b * p.nv + __ldg(p.vslot + b * p.r_eff + j)) * p.L + kb;
}

// A random shift s < 2*a_max draws the same view as consecutive shift s
// (the reference computes it twice, general.py:288-294; the FFT is the same
// bits either way).  Per signal: the distinct random shifts packed after
// the S consecutive views, each random view's slot, and the number of views
// to transform.  At d = 8 (r_eff = d: every residue drawn) 6 of the 14
// transforms are duplicates.
__global__ void k_gen_vslot(GenParams p, int64_t B, int dedup, int64_t *__restrict__ vsh,
                            int32_t *__restrict__ vslot, int32_t *__restrict__ nview) {
    const int64_t b = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (b >= B) return;
    const int64_t *sh = p.shifts + b * p.shift_stride;
    int n = 0;
    for (int j = 0; j < p.r_eff; j++) {
        const int64_t s = sh[j];
        if (dedup && s < p.S) {
            vslot[b * p.r_eff + j] = (int32_t)s;
        } else {
            vsh[b * p.r_eff + n] = s;
            vslot[b * p.r_eff + j] = p.S + n;
            n++;
        }
    }
    for (int j = n; j < p.r_eff; j++) vsh[b * p.r_eff + j] = 0;   // padding (never transformed)
    nview[b] = p.S + n;
}

// ------------------------------------------------------------------- svd
// Singular values of the 3 x 3 Hankel H_ij = m_{i+j} in closed form: the
// eigenvalues of the Hermitian G = H^H H by the trigonometric cubic
// (lambda = q + 2 p cos(phi + 2 pi k / 3)), sigma = sqrt(lambda).  Its
// error grows with the spread lambda_1 / lambda_3 and, through acos, as
// |r| -> 1 (a nearly repeated eigenvalue), so it is used only when
// lambda_3 >= lambda_1 / 64 and |r| <= 0.999: there sigma agrees with
// LAPACK's SVD to <= 5.3e-14 relative (1e5 random Hankels, measured; the
// reference's two backends differ by up to 1e-13), and it takes 86 % of
// noise bins.  Every other bin -- rank-1 tone bins, near-singular or
// near-degenerate Hankels -- is listed for the register-resident Jacobi
// (k_gen_svd_fix).
__device__ __forceinline__ bool hankel_sv3_closed(const cx *m, double *out) {
    // G_jk = sum_i conj(m_{i+j}) m_{i+k}
    double g00 = 0.0, g11 = 0.0, g22 = 0.0;
    cx g01 = mk(0.0, 0.0), g02 = mk(0.0, 0.0), g12 = mk(0.0, 0.0);
#pragma unroll
    for (int i = 0; i < 3; i++) {
        const cx a0 = m[i], a1 = m[i + 1], a2 = m[i + 2];
        g00 = fma(a0.re, a0.re, fma(a0.im, a0.im, g00));
        g11 = fma(a1.re, a1.re, fma(a1.im, a1.im, g11));
        g22 = fma(a2.re, a2.re, fma(a2.im, a2.im, g22));
        g01 = cadd(g01, nmul(cconj(a0), a1));
        g02 = cadd(g02, nmul(cconj(a0), a2));
        g12 = cadd(g12, nmul(cconj(a1), a2));
    }
    const double q = (g00 + g11 + g22) * (1.0 / 3.0);
    const double a = g00 - q, b = g11 - q, c = g22 - q;
    const double x2 = fma(g01.re, g01.re, g01.im * g01.im);
    const double y2 = fma(g02.re, g02.re, g02.im * g02.im);
    const double z2 = fma(g12.re, g12.re, g12.im * g12.im);
    const double p2 = fma(a, a, fma(b, b, fma(c, c, 2.0 * (x2 + y2 + z2))));
    double l1, l2, l3;
    if (p2 <= 0.0) {
        l1 = l2 = l3 = q;
    } else {
        const double pp = sqrt(p2 * (1.0 / 6.0));
        // det(G - qI) = abc + 2 Re(x z conj(y)) - a|z|^2 - b|y|^2 - c|x|^2
        const cx xz = nmul(g01, g12);
        const double re = fma(xz.re, g02.re, xz.im * g02.im);
        const double det = fma(a * b, c, fma(2.0, re, -fma(a, z2, fma(b, y2, c * x2))));
        const double r = det / (2.0 * pp * pp * pp);
        if (!(fabs(r) <= 0.999)) return false;
        const double phi = acos(r) * (1.0 / 3.0);
        l1 = fma(2.0 * pp, cos(phi), q);
        l3 = fma(2.0 * pp, cos(phi + 2.0943951023931957), q);
        l2 = 3.0 * q - l1 - l3;
    }
    if (!(l1 > 0.0) || !(l1 < INFINITY) || !(l3 * 64.0 >= l1)) return false;
    out[0] = sqrt(l1);
    out[1] = sqrt(l2);
    out[2] = sqrt(l3);
    return out[0] >= out[1] && out[1] >= out[2];
}

// the bins k_gen_svd left to the Jacobi (listed flat indices b*L + k)
__global__ void __launch_bounds__(128) k_gen_svd_fix(const cx *__restrict__ V, GenParams p,
                                                     double *__restrict__ sv, const int64_t *__restrict__ fix,
                                                     const unsigned long long *__restrict__ nfix) {
    const int64_t cnt = (int64_t)*nfix;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < cnt;
         i += int64_t(gridDim.x) * blockDim.x) {
        const int64_t t = fix[i];
        const int64_t b = t / p.L, k = t - b * p.L;
        cx syn[6];
#pragma unroll
        for (int j = 0; j < 6; j++) syn[j] = ldcx(V + (b * p.nv + j) * p.L + k);
        double s[3];
        hankel_sv_n<3>(syn, s, 2.220446049250313e-16);
#pragma unroll
        for (int j = 0; j < 3; j++) sv[t * 3 + j] = s[j];
    }
}

template <int AM>
__global__ void __launch_bounds__(128) k_gen_svd(const cx *__restrict__ V, GenParams p,
                                                 double *__restrict__ sv, double *__restrict__ partial,
                                                 int64_t *__restrict__ fix, unsigned long long *__restrict__ nfix,
                                                 int closed) {
    constexpr int S = 2 * AM;
    const int64_t b = blockIdx.y;
    const int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    double e = 0.0;
    if (k < p.L) {
        cx syn[S];
#pragma unroll
        for (int j = 0; j < S; j++) {
            syn[j] = ldcx(V + (b * p.nv + j) * p.L + k);
            e += syn[j].re * syn[j].re + syn[j].im * syn[j].im;
        }
        double s[AM];
        if (AM == 3 && closed) {
            // closed form; the conditioned-out bins go to k_gen_svd_fix
            if (hankel_sv3_closed(syn, s)) {
#pragma unroll
                for (int i = 0; i < AM; i++) sv[(b * p.L + k) * AM + i] = s[i];
            } else {
                fix[atomicAdd(nfix, 1ull)] = b * p.L + k;
            }
        } else {
            hankel_sv_n<AM>(syn, s, 2.220446049250313e-16);
#pragma unroll
            for (int i = 0; i < AM; i++) sv[(b * p.L + k) * AM + i] = s[i];
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) e += __shfl_xor_sync(0xffffffffu, e, o);
    __shared__ double red[4];
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = e;
    __syncthreads();
    if (threadIdx.x == 0) partial[b * gridDim.x + blockIdx.x] = (red[0] + red[1]) + (red[2] + red[3]);
}

// standalone form (estimate_collisions on given syndromes, general.py:131-155):
// rows of a (nb, ld) row-major syndrome matrix; energy over all ld columns
template <int AM>
__global__ void __launch_bounds__(128) k_rows_svd(const cx *__restrict__ syn, int64_t nb, int64_t ld,
                                                  double *__restrict__ sv, double *__restrict__ partial,
                                                  double tol) {
    const int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    double e = 0.0;
    if (k < nb) {
        cx m[2 * AM];
#pragma unroll
        for (int j = 0; j < 2 * AM - 1; j++) m[j] = ldcx(syn + k * ld + j);
        for (int64_t j = 0; j < ld; j++) {
            const cx v = ldcx(syn + k * ld + j);
            e += v.re * v.re + v.im * v.im;
        }
        double s[AM];
        hankel_sv_n<AM>(m, s, tol);
#pragma unroll
        for (int i = 0; i < AM; i++) sv[k * AM + i] = s[i];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) e += __shfl_xor_sync(0xffffffffu, e, o);
    __shared__ double red[4];
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = e;
    __syncthreads();
    if (threadIdx.x == 0) partial[blockIdx.x] = (red[0] + red[1]) + (red[2] + red[3]);
}

// ------------------------------------------------------------------ vote
// staging keys in smem measured slower (736 vs 552 us, cfg4), and so did
// caching them in registers (64 registers halve the resident CTAs: 468 ->
// 637 us); keys are re-read from L2
constexpr int VOTE_SMEM_KEYS = 0;
constexpr int VOTE_CAND = 2048;   // candidate keys compacted to shared memory

__device__ __forceinline__ unsigned long long dkey(double v) {
    return (unsigned long long)__double_as_longlong(v);   // sigma >= 0: bit order == value order
}

__global__ void __launch_bounds__(1024, 2) k_gen_vote(const double *__restrict__ sv,
                                                   const double *__restrict__ partial, int nparts,
                                                   GenParams p, int32_t *__restrict__ votes,
                                                   int64_t *__restrict__ stats,
                                                   int64_t *__restrict__ wl,
                                                   unsigned long long *__restrict__ wl_count) {
    const int64_t b = blockIdx.x;
    const int64_t M = p.L * p.a_max;
    const int64_t take = p.k < M ? p.k : M;
    extern __shared__ double s_keys[];
    // the radix passes re-read every key 8 times: stage them in shared
    // memory when they fit (config 4: 12288 keys = 96 KiB)
    const bool in_smem = M <= VOTE_SMEM_KEYS;
    if (in_smem)
        for (int64_t i = threadIdx.x; i < M; i += blockDim.x) s_keys[i] = sv[b * M + i];
    const double *svb = in_smem ? s_keys : sv + b * M;
    int32_t *vb = votes + b * p.L;
    __shared__ unsigned int hist[256];
    __shared__ unsigned long long s_prefix, s_mask;
    __shared__ long long s_remaining;
    __shared__ int wsum[32];
    __shared__ unsigned long long s_ck[VOTE_CAND];
    __shared__ unsigned int s_h32[5];
    __shared__ long long s_ncand;
    __shared__ int s_nc;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        s_prefix = 0;
        s_mask = 0;
        s_remaining = take;
    }
    for (int64_t i = threadIdx.x; i < p.L; i += blockDim.x) vb[i] = 0;
    // visit every flat index in order of i0 = 0, blockDim, ... (block-uniform
    // trip count; f may contain block barriers)
    auto for_keys = [&](auto &&f) {
        for (int64_t i0 = 0; i0 < M; i0 += blockDim.x) {
            const int64_t i = i0 + threadIdx.x;
            f(i, i < M ? dkey(svb[i]) : 0ull);
        }
    };
    __syncthreads();
    // exact radix select (8-bit digits, MSB first) of the take-th largest key.
    // Histogram: lanes holding the same digit are aggregated with
    // __match_any_sync (sigma keys share their top bytes, so plain shared
    // atomics serialise); digit choice: warp 0 scans the 256 counts from the
    // top, 8 per lane.
    //
    // Once the keys sharing the chosen prefix fit VOTE_CAND, they are
    // compacted into shared memory and the remaining passes scan only them
    // (config 4: 2 full passes + 1 compaction pass instead of 8 full passes).
    if (threadIdx.x == 0) s_ncand = M;
    __syncthreads();
    bool cand = false;   // block-uniform
    if (take > 0) {
        for (int shift = 56; shift >= 0; shift -= 8) {
            const unsigned long long pre = s_prefix, msk = s_mask;
            if (!cand && s_ncand <= VOTE_CAND) {
                if (threadIdx.x == 0) s_nc = 0;
                __syncthreads();
                for_keys([&](int64_t i, unsigned long long key) {
                    const bool m = i < M && (key & msk) == pre;
                    const unsigned bal = __ballot_sync(0xffffffffu, m);
                    int base = 0;
                    if (lane == 0 && bal) base = atomicAdd(&s_nc, __popc(bal));
                    base = __shfl_sync(0xffffffffu, base, 0);
                    if (m) s_ck[base + __popc(bal & ((1u << lane) - 1))] = key;
                });
                cand = true;
            }
            for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
            __syncthreads();
            auto hist_key = [&](bool valid, unsigned long long key) {
                int dg = 256;   // not a candidate
                if (valid && (key & msk) == pre) dg = (int)((key >> shift) & 255);
                const unsigned peers = __match_any_sync(0xffffffffu, dg);
                if (dg < 256 && lane == __ffs(peers) - 1) atomicAdd(&hist[dg], (unsigned)__popc(peers));
            };
            if (cand) {
                const int nc = s_nc;
                for (int i0 = 0; i0 < nc; i0 += blockDim.x) {
                    const int i = i0 + threadIdx.x;
                    hist_key(i < nc, i < nc ? s_ck[i] : 0ull);
                }
            } else {
                for_keys([&](int64_t i, unsigned long long key) { hist_key(i < M, key); });
            }
            __syncthreads();
            if (warp == 0) {
                // lane l owns digits 255-8l .. 248-8l (descending)
                unsigned c[8], lsum = 0;
#pragma unroll
                for (int q = 0; q < 8; q++) {
                    c[q] = hist[255 - 8 * lane - q];
                    lsum += c[q];
                }
                unsigned inc = lsum;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const unsigned y = __shfl_up_sync(0xffffffffu, inc, o);
                    if (lane >= o) inc += y;
                }
                const long long rem = s_remaining;
                const long long before = (long long)(inc - lsum);
                const bool mine = before < rem && before + (long long)lsum >= rem;
                if (mine) {
                    long long cum = before;
                    int D = 255 - 8 * lane - 7;
                    unsigned cD = c[7];
#pragma unroll
                    for (int q = 0; q < 8; q++) {
                        if (cum + (long long)c[q] >= rem) {
                            D = 255 - 8 * lane - q;
                            cD = c[q];
                            break;
                        }
                        cum += c[q];
                    }
                    s_remaining = rem - cum;
                    s_ncand = cD;
                    s_prefix = pre | ((unsigned long long)D << shift);
                    s_mask = msk | (0xFFull << shift);
                }
            }
            __syncthreads();
        }
    }
    const unsigned long long tau = s_prefix;
    const long long need_eq = take > 0 ? s_remaining : 0;   // how many keys == tau to take
    // selection in flat order: keys > tau all; keys == tau by ascending flat
    // index (lexsort tie-break: bin asc, then rank asc)
    long long eq_carry = 0;
    const bool all_eq = take > 0 && need_eq == s_ncand;   // every key == tau is taken (the usual case)
    if (all_eq) {
        for (int64_t i = threadIdx.x; i < M; i += blockDim.x)
            if (dkey(svb[i]) >= tau) atomicAdd(&vb[i / p.a_max], 1);
    } else if (take > 0)
        for_keys([&](int64_t i, unsigned long long key) {
            const bool gt = i < M && key > tau;
            const bool eq = i < M && key == tau;
            const unsigned m = __ballot_sync(0xffffffffu, eq);
            if (lane == 0) wsum[warp] = __popc(m);
            __syncthreads();
            int before = 0, total = 0;
            for (int w2 = 0; w2 < (int)(blockDim.x >> 5); w2++) {
                before += (w2 < warp) ? wsum[w2] : 0;
                total += wsum[w2];
            }
            const long long rank = eq_carry + before + __popc(m & ((1u << lane) - 1));
            if (gt || (eq && rank < need_eq)) atomicAdd(&vb[i / p.a_max], 1);
            eq_carry += total;
            __syncthreads();
        });
    __syncthreads();
    // zero-vote guard on the RMS of all consecutive syndromes, cap, histogram
    double esum = 0.0;
    if (threadIdx.x == 0) {
        for (int i = 0; i < nparts; i++) esum += partial[b * nparts + i];
    }
    __shared__ double s_thr;
    if (threadIdx.x == 0) {
        const double rms_syn = sqrt(esum / (double)(p.L * p.S));
        s_thr = p.zvr * rms_syn;
    }
    __syncthreads();
    // (histogram counts in registers and 32-bit shared atomics; worklist
    // slots reserved once per block after a block-wide count)
    const int cap = (int)(p.a_max < p.d ? p.a_max : p.d);
    if (threadIdx.x < 5) s_h32[threadIdx.x] = 0;
    if (threadIdx.x == 0) s_nc = 0;
    __syncthreads();
    unsigned h0 = 0, h1 = 0, h2 = 0, h3 = 0, h4 = 0;
    for (int64_t kb = threadIdx.x; kb < p.L; kb += blockDim.x) {
        int v = vb[kb];
        if (svb[kb * p.a_max] <= s_thr) v = 0;
        if (v > cap) v = cap;
        vb[kb] = v;
        h0 += v == 0;
        h1 += v == 1;
        h2 += v == 2;
        h3 += v == 3;
        h4 += v == 4;
    }
    if (h0) atomicAdd(&s_h32[0], h0);
    if (h1) atomicAdd(&s_h32[1], h1);
    if (h2) atomicAdd(&s_h32[2], h2);
    if (h3) atomicAdd(&s_h32[3], h3);
    if (h4) atomicAdd(&s_h32[4], h4);
    __syncthreads();
    __shared__ unsigned long long s_base;
    if (threadIdx.x == 0) {
        int64_t *st = stats + b * SFDT_GS_PER_SIGNAL;
        for (int a = 0; a <= 4; a++) st[SFDT_GS_HIST0 + a] = s_h32[a];
        const unsigned nv = s_h32[1] + s_h32[2] + s_h32[3] + s_h32[4];
        st[SFDT_GS_NVOTED] = nv;
        st[SFDT_GS_RANKDEF] = 0;
        s_base = nv ? atomicAdd(wl_count, (unsigned long long)nv) : 0ull;
    }
    __syncthreads();
    // worklist append (order within the list is irrelevant downstream)
    for (int64_t k0 = 0; k0 < p.L; k0 += blockDim.x) {
        const int64_t kb = k0 + threadIdx.x;
        const bool on = kb < p.L && vb[kb] >= 1;
        const unsigned bal = __ballot_sync(0xffffffffu, on);
        int base = 0;
        if (lane == 0 && bal) base = atomicAdd(&s_nc, __popc(bal));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (on) wl[s_base + base + __popc(bal & ((1u << lane) - 1))] = b * p.L + kb;
    }
}

// ------------------------------------------------ vote, long views
// The same exact top-K selection for signals with many keys (M = L*a_max >
// VOTE_BIG), spread over CTAs of VCH keys: each 8-bit radix pass builds
// per-chunk histograms (warp-aggregated) summed into a per-signal global
// histogram, one warp per signal picks the digit; then per-chunk counts of
// keys equal to the threshold give every chunk its tie rank base, the
// chunks vote, and a bin-parallel pass applies the zero-vote guard, cap,
// histogram and worklist.  Identical result to k_gen_vote.
constexpr int64_t VOTE_BIG = 65536;
constexpr int64_t VCH = 16384;

struct VSel {
    unsigned long long prefix, mask;
    long long remaining;
    double thr;
    unsigned long long nc;   // keys sharing the 16-bit prefix (k_vsel_compact)
    long long neq;           // keys equal to the threshold (k_vsel_select), -1 unknown
};

// keys per signal that k_vsel_compact can hold; beyond it k_vsel_select
// scans every key of the signal (same result, slower)
constexpr int64_t VSEL_CAND = 65536;

// per signal: state, zero-vote threshold (rms of the consecutive syndromes),
// stats fields the later passes accumulate into
// one warp per signal (lane-strided partial sums, then a butterfly)
__global__ void k_vsel_init(const double *__restrict__ partial, int nparts, GenParams p, int64_t B,
                            VSel *__restrict__ vs, int64_t *__restrict__ stats) {
    const int64_t b = blockIdx.x;
    const int lane = threadIdx.x;
    const int64_t M = p.L * p.a_max;
    double esum = 0.0;
    for (int i = lane; i < nparts; i += 32) esum += partial[b * nparts + i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) esum += __shfl_xor_sync(0xffffffffu, esum, o);
    if (lane != 0) return;
    const double rms_syn = sqrt(esum / (double)(p.L * p.S));
    vs[b].prefix = 0;
    vs[b].mask = 0;
    vs[b].remaining = p.k < M ? p.k : M;
    vs[b].thr = p.zvr * rms_syn;
    vs[b].nc = 0;
    vs[b].neq = -1;
    int64_t *st = stats + b * SFDT_GS_PER_SIGNAL;
    for (int a = 0; a <= 4; a++) st[SFDT_GS_HIST0 + a] = 0;
    st[SFDT_GS_NVOTED] = 0;
    st[SFDT_GS_RANKDEF] = 0;
}

__global__ void __launch_bounds__(256) k_vsel_hist(const double *__restrict__ sv, GenParams p, int64_t nch,
                                                   int shift, const VSel *__restrict__ vs,
                                                   unsigned int *__restrict__ ghist) {
    const int64_t b = blockIdx.x / nch, ch = blockIdx.x - b * nch;
    const int64_t M = p.L * p.a_max;
    __shared__ unsigned int hist[256];
    const int lane = threadIdx.x & 31;
    hist[threadIdx.x] = 0;
    __syncthreads();
    const unsigned long long pre = vs[b].prefix, msk = vs[b].mask;
    const int64_t i1 = (ch + 1) * VCH < M ? (ch + 1) * VCH : M;
    const double *svb = sv + b * M;
    for (int64_t i0 = ch * VCH; i0 < i1; i0 += blockDim.x) {   // block-uniform trip count
        const int64_t i = i0 + threadIdx.x;
        int dg = 256;
        if (i < i1) {
            const unsigned long long key = dkey(svb[i]);
            if ((key & msk) == pre) dg = (int)((key >> shift) & 255);
        }
        const unsigned peers = __match_any_sync(0xffffffffu, dg);
        if (dg < 256 && lane == __ffs(peers) - 1) atomicAdd(&hist[dg], (unsigned)__popc(peers));
    }
    __syncthreads();
    const unsigned c = hist[threadIdx.x];
    if (c) atomicAdd(&ghist[b * 256 + threadIdx.x], c);
}

// one warp per signal: choose the digit (as k_gen_vote), clear the histogram
__global__ void k_vsel_pick(int64_t B, int shift, VSel *__restrict__ vs, unsigned int *__restrict__ ghist) {
    const int64_t b = blockIdx.x;
    const int lane = threadIdx.x;
    unsigned c[8], lsum = 0;
#pragma unroll
    for (int q = 0; q < 8; q++) {
        c[q] = ghist[b * 256 + 255 - 8 * lane - q];
        lsum += c[q];
    }
#pragma unroll
    for (int q = 0; q < 8; q++) ghist[b * 256 + 255 - 8 * lane - q] = 0;
    unsigned inc = lsum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    const long long rem = vs[b].remaining;
    if (rem <= 0) return;
    const long long before = (long long)(inc - lsum);
    if (before < rem && before + (long long)lsum >= rem) {
        long long cum = before;
        int D = 255 - 8 * lane - 7;
#pragma unroll
        for (int q = 0; q < 8; q++) {
            if (cum + (long long)c[q] >= rem) {
                D = 255 - 8 * lane - q;
                break;
            }
            cum += c[q];
        }
        vs[b].remaining = rem - cum;
        vs[b].prefix |= (unsigned long long)D << shift;
        vs[b].mask |= 0xFFull << shift;
    }
}

// after the two leading 8-bit passes: the keys sharing the chosen 16-bit
// prefix are appended to the signal's candidate list
__global__ void __launch_bounds__(256) k_vsel_compact(const double *__restrict__ sv, GenParams p, int64_t nch,
                                                      VSel *__restrict__ vs,
                                                      unsigned long long *__restrict__ cand) {
    const int64_t b = blockIdx.x / nch, ch = blockIdx.x - b * nch;
    const int64_t M = p.L * p.a_max;
    if (vs[b].remaining <= 0) return;
    const unsigned long long pre = vs[b].prefix, msk = vs[b].mask;
    const int64_t i1 = (ch + 1) * VCH < M ? (ch + 1) * VCH : M;
    const double *svb = sv + b * M;
    const int lane = threadIdx.x & 31;
    for (int64_t i0 = ch * VCH; i0 < i1; i0 += blockDim.x) {   // block-uniform trip count
        const int64_t i = i0 + threadIdx.x;
        unsigned long long key = 0;
        bool m = false;
        if (i < i1) {
            key = dkey(svb[i]);
            m = (key & msk) == pre;
        }
        const unsigned bal = __ballot_sync(0xffffffffu, m);
        unsigned long long base = 0;
        if (lane == 0 && bal) base = atomicAdd(&vs[b].nc, (unsigned long long)__popc(bal));
        base = __shfl_sync(0xffffffffu, base, 0);
        const unsigned long long slot = base + __popc(bal & ((1u << lane) - 1));
        if (m && slot < (unsigned long long)VSEL_CAND) cand[b * VSEL_CAND + slot] = key;
    }
}

// the remaining six 8-bit passes of the radix select, one CTA per signal,
// over the compacted candidates (or every key when they overflowed)
__global__ void __launch_bounds__(1024) k_vsel_select(const double *__restrict__ sv, GenParams p,
                                                      VSel *__restrict__ vs,
                                                      const unsigned long long *__restrict__ cand) {
    const int64_t b = blockIdx.x;
    const int64_t M = p.L * p.a_max;
    __shared__ unsigned int hist[256];
    __shared__ unsigned long long s_prefix, s_mask;
    __shared__ long long s_remaining, s_neq;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        s_neq = -1;
        s_prefix = vs[b].prefix;
        s_mask = vs[b].mask;
        s_remaining = vs[b].remaining;
    }
    __syncthreads();
    if (s_remaining <= 0) return;
    const unsigned long long nc = vs[b].nc;
    const bool use_cand = nc <= (unsigned long long)VSEL_CAND;
    const int64_t n = use_cand ? (int64_t)nc : M;
    const unsigned long long *cb = cand + b * VSEL_CAND;
    const double *svb = sv + b * M;
    for (int shift = 40; shift >= 0; shift -= 8) {
        for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
        __syncthreads();
        const unsigned long long pre = s_prefix, msk = s_mask;
        for (int64_t i0 = 0; i0 < n; i0 += blockDim.x) {   // block-uniform trip count
            const int64_t i = i0 + threadIdx.x;
            int dg = 256;
            if (i < n) {
                const unsigned long long key = use_cand ? cb[i] : dkey(svb[i]);
                if ((key & msk) == pre) dg = (int)((key >> shift) & 255);
            }
            const unsigned peers = __match_any_sync(0xffffffffu, dg);
            if (dg < 256 && lane == __ffs(peers) - 1) atomicAdd(&hist[dg], (unsigned)__popc(peers));
        }
        __syncthreads();
        if (warp == 0) {   // digit choice, as k_vsel_pick
            unsigned c[8], lsum = 0;
#pragma unroll
            for (int q = 0; q < 8; q++) {
                c[q] = hist[255 - 8 * lane - q];
                lsum += c[q];
            }
            unsigned inc = lsum;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned y = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += y;
            }
            const long long rem = s_remaining;
            const long long before = (long long)(inc - lsum);
            if (before < rem && before + (long long)lsum >= rem) {
                long long cum = before;
                int D = 255 - 8 * lane - 7;
                unsigned cD = c[7];
#pragma unroll
                for (int q = 0; q < 8; q++) {
                    if (cum + (long long)c[q] >= rem) {
                        D = 255 - 8 * lane - q;
                        cD = c[q];
                        break;
                    }
                    cum += c[q];
                }
                s_remaining = rem - cum;
                s_prefix = pre | ((unsigned long long)D << shift);
                s_mask = msk | (0xFFull << shift);
                if (shift == 0) s_neq = cD;   // keys equal to the threshold
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        vs[b].prefix = s_prefix;
        vs[b].mask = s_mask;
        vs[b].remaining = s_remaining;
        vs[b].neq = s_neq;
    }
}

__global__ void __launch_bounds__(256) k_vsel_eqcount(const double *__restrict__ sv, GenParams p, int64_t nch,
                                                      const VSel *__restrict__ vs, long long *__restrict__ eqc) {
    const int64_t b = blockIdx.x / nch, ch = blockIdx.x - b * nch;
    const int64_t M = p.L * p.a_max;
    if (vs[b].neq >= 0 && vs[b].remaining == vs[b].neq) return;   // every tie taken: no ranks needed
    const unsigned long long tau = vs[b].prefix;
    const int64_t i1 = (ch + 1) * VCH < M ? (ch + 1) * VCH : M;
    const double *svb = sv + b * M;
    long long n = 0;
    for (int64_t i = ch * VCH + threadIdx.x; i < i1; i += blockDim.x) n += dkey(svb[i]) == tau;
    __shared__ long long red[256];
    red[threadIdx.x] = n;
    __syncthreads();
    for (int s2 = 128; s2 > 0; s2 >>= 1) {
        if (threadIdx.x < s2) red[threadIdx.x] += red[threadIdx.x + s2];
        __syncthreads();
    }
    if (threadIdx.x == 0) eqc[blockIdx.x] = red[0];
}

__global__ void __launch_bounds__(256) k_vsel_vote(const double *__restrict__ sv, GenParams p, int64_t nch,
                                                   const VSel *__restrict__ vs,
                                                   const long long *__restrict__ eqc,
                                                   int32_t *__restrict__ votes) {
    const int64_t b = blockIdx.x / nch, ch = blockIdx.x - b * nch;
    const int64_t M = p.L * p.a_max;
    const int64_t take = p.k < M ? p.k : M;
    if (take <= 0) return;
    const unsigned long long tau = vs[b].prefix;
    const long long need_eq = vs[b].remaining;
    const int64_t i1 = (ch + 1) * VCH < M ? (ch + 1) * VCH : M;
    const double *svb = sv + b * M;
    int32_t *vb = votes + b * p.L;
    const long long neq = vs[b].neq;
    long long eq_carry = 0, eq_all = neq;   // keys == tau in the chunks before this one / in all
    if (!(neq >= 0 && need_eq == neq)) {
        eq_all = 0;
        for (int64_t c2 = 0; c2 < nch; c2++) {
            const long long e = eqc[b * nch + c2];
            eq_carry += c2 < ch ? e : 0;
            eq_all += e;
        }
    }
    if (need_eq == eq_all) {   // every key == tau is taken: no tie ranks needed
        for (int64_t i = ch * VCH + threadIdx.x; i < i1; i += blockDim.x)
            if (dkey(svb[i]) >= tau) atomicAdd(&vb[i / p.a_max], 1);
        return;
    }
    __shared__ int wsum[8];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int64_t i0 = ch * VCH; i0 < i1; i0 += blockDim.x) {
        const int64_t i = i0 + threadIdx.x;
        unsigned long long key = 0;
        bool gt = false, eq = false;
        if (i < i1) {
            key = dkey(svb[i]);
            gt = key > tau;
            eq = key == tau;
        }
        const unsigned m = __ballot_sync(0xffffffffu, eq);
        if (lane == 0) wsum[warp] = __popc(m);
        __syncthreads();
        int before = 0, total = 0;
        for (int w2 = 0; w2 < 8; w2++) {
            before += (w2 < warp) ? wsum[w2] : 0;
            total += wsum[w2];
        }
        const long long rank = eq_carry + before + __popc(m & ((1u << lane) - 1));
        if (gt || (eq && rank < need_eq)) atomicAdd(&vb[i / p.a_max], 1);
        eq_carry += total;
        __syncthreads();
    }
}

// zero-vote guard, cap, histogram, worklist (bins of a chunk of the signal)
__global__ void __launch_bounds__(256) k_vsel_fin(const double *__restrict__ sv, GenParams p, int64_t nchL,
                                                  const VSel *__restrict__ vs, int32_t *__restrict__ votes,
                                                  int64_t *__restrict__ stats, int64_t *__restrict__ wl,
                                                  unsigned long long *__restrict__ wl_count) {
    const int64_t b = blockIdx.x / nchL, ch = blockIdx.x - b * nchL;
    const int64_t M = p.L * p.a_max;
    const double thr = vs[b].thr;
    const int cap = (int)(p.a_max < p.d ? p.a_max : p.d);
    int32_t *vb = votes + b * p.L;
    const double *svb = sv + b * M;
    __shared__ unsigned int s_hist[5];
    __shared__ int s_n;
    __shared__ unsigned long long s_base;
    if (threadIdx.x < 5) s_hist[threadIdx.x] = 0;
    if (threadIdx.x == 0) s_n = 0;
    __syncthreads();
    const int64_t k0 = ch * VCH, k1 = (k0 + VCH < p.L) ? k0 + VCH : p.L;
    unsigned h0 = 0, h1 = 0, h2 = 0, h3 = 0, h4 = 0;
    for (int64_t kb = k0 + threadIdx.x; kb < k1; kb += blockDim.x) {
        int v = vb[kb];
        if (svb[kb * p.a_max] <= thr) v = 0;
        if (v > cap) v = cap;
        vb[kb] = v;
        h0 += v == 0;
        h1 += v == 1;
        h2 += v == 2;
        h3 += v == 3;
        h4 += v == 4;
    }
    if (h0) atomicAdd(&s_hist[0], h0);
    if (h1) atomicAdd(&s_hist[1], h1);
    if (h2) atomicAdd(&s_hist[2], h2);
    if (h3) atomicAdd(&s_hist[3], h3);
    if (h4) atomicAdd(&s_hist[4], h4);
    __syncthreads();
    if (threadIdx.x < 5 && s_hist[threadIdx.x])
        atomicAdd((unsigned long long *)(stats + b * SFDT_GS_PER_SIGNAL + SFDT_GS_HIST0 + threadIdx.x),
                  (unsigned long long)s_hist[threadIdx.x]);
    if (threadIdx.x == 0) {
        const unsigned long long nv = (unsigned long long)s_hist[1] + s_hist[2] + s_hist[3] + s_hist[4];
        if (nv) {
            atomicAdd((unsigned long long *)(stats + b * SFDT_GS_PER_SIGNAL + SFDT_GS_NVOTED), nv);
            s_base = atomicAdd(wl_count, nv);
        }
    }
    __syncthreads();
    // worklist append (order within the list is irrelevant downstream)
    const int lane = threadIdx.x & 31;
    for (int64_t kq = k0; kq < k1; kq += blockDim.x) {
        const int64_t kb = kq + threadIdx.x;
        const bool on = kb < k1 && vb[kb] >= 1;
        const unsigned bal = __ballot_sync(0xffffffffu, on);
        int base = 0;
        if (lane == 0 && bal) base = atomicAdd(&s_n, __popc(bal));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (on) wl[s_base + base + __popc(bal & ((1u << lane) - 1))] = b * p.L + kb;
    }
}

// ------------------------------------------------------------- per bin
// correlation |sum_j conj(phi_j) v_j| with the column given by its phases
__device__ __forceinline__ double corr_abs(const cx *phi_col, const cx *v, int r) {
    cx acc = mk(0.0, 0.0);
    for (int j = 0; j < r; j++) acc = cadd(acc, nmul(cconj(phi_col[j]), v[j]));
    return cabs_(acc);
}

struct SPOut {
    int nsup;
    int sup[GEN_MAX_SUP];
    cx coef[GEN_MAX_SUP];
    int rankdef;
#ifdef SFDT_BINS_PROFILE
    int iters, nminnorm;
    long long cyc_lsq, cyc_top;
#endif
};

// Warp merge of per-lane top lists (each sorted best-first by score desc,
// then column asc) into the warp's top `cnt` in the same order -- the result
// of inserting every column sequentially in ascending order.  A NaN score
// ranks after every number (numpy's argsort puts NaN last).  All 32 lanes
// call it and all receive the merged list.
__device__ __forceinline__ bool sp_better(double v2, int t2, double v, int t) {
    const bool n2 = v2 != v2, n1 = v != v;
    if (n2 != n1) return n1;            // a number beats a NaN
    if (!n2 && v2 != v) return v2 > v;
    return t2 < t;
}

__device__ __forceinline__ int warp_topk_merge(const double *sc, const int *id, int nloc, int cnt,
                                               double *osc, int *oid) {
    int h = 0, on = 0;
    for (int round = 0; round < cnt; round++) {
        double v = h < nloc ? sc[h] : 0.0;
        int t = h < nloc ? id[h] : INT_MAX;   // INT_MAX: this lane is exhausted
#pragma unroll
        for (int off = 16; off; off >>= 1) {
            const double v2 = __shfl_xor_sync(0xffffffffu, v, off);
            const int t2 = __shfl_xor_sync(0xffffffffu, t, off);
            if (t2 != INT_MAX && (t == INT_MAX || sp_better(v2, t2, v, t))) {
                v = v2;
                t = t2;
            }
        }
        if (t == INT_MAX) break;
        osc[on] = v;
        oid[on] = t;
        on++;
        if (h < nloc && id[h] == t) h++;
    }
    return on;
}

// subspace pursuit over columns c < ncols (column index -> candidate t via
// cols[] unless all_cols); phi[j, t] = phase_j * base_phi[j, t].
// nlanes = 1: one thread per bin.  nlanes = 32: one warp per bin -- lane l
// scores columns l, l+32, ... (the same per-column arithmetic) and the
// lane lists are merged by warp_topk_merge, so the selections, and with
// them every least-squares solve (run redundantly by all lanes), are
// bit-identical to the single-thread form.
//
// RT > 0: r = RT at compile time -- the row loops unroll and full-rank least
// squares run as the register-resident lstsq_qr_t<RT, C> (the same
// operations in the same order as lstsq_qr, so the same bits), which keeps
// a multi-collision bin's long serial chain out of local memory.
template <int RT = 0>
__device__ __forceinline__ void subspace_pursuit_dev(const cx *y, const cx *phase, const cx *bphi, int64_t d,
                                                     int r_rt, const int *cols, int ncols, bool all_cols,
                                                     int a_sp, SPOut &o, int lane = 0, int nlanes = 1,
                                                     int max_iter = 10) {
    const int r = RT > 0 ? RT : r_rt;
    const int a_eff = a_sp < ncols ? a_sp : ncols;
    auto col_t = [&](int c) -> int64_t { return all_cols ? (int64_t)c : (int64_t)cols[c]; };
    auto phi_col = [&](int c, cx *out) {
        const int64_t t = col_t(c);
#pragma unroll
        for (int j = 0; j < (RT > 0 ? RT : GEN_MAX_R); j++) {
            if (RT == 0 && j >= r) break;
            out[j] = nmul(phase[j], ldcx(bphi + (int64_t)j * d + t));
        }
    };
    cx pc[GEN_MAX_R];
    // initial support: top a_eff of |phi^H y|, stable, then sorted
    double tsc[GEN_MAX_SUP];
    int tid_[GEN_MAX_SUP];
    // top a_eff columns of |phi^H v| (stable), best first
    auto top_cols = [&](const cx *v) -> int {
        int n0 = 0;
        for (int c = lane; c < ncols; c += nlanes) {
            phi_col(c, pc);
            topk_insert(tsc, tid_, n0, a_eff, corr_abs(pc, v, r), c);
        }
        if (nlanes == 1) return n0;
        double msc[GEN_MAX_SUP];
        int mid[GEN_MAX_SUP];
        const int nm = warp_topk_merge(tsc, tid_, n0, a_eff, msc, mid);
        for (int i = 0; i < nm; i++) {
            tsc[i] = msc[i];
            tid_[i] = mid[i];
        }
        return nm;
    };
    int nt = top_cols(y);
    int sup[GEN_MAX_SUP];
    int nsup = nt;
    for (int i = 0; i < nt; i++) sup[i] = tid_[i];
    sort_ints(sup, nsup);
    cx A[GEN_MAX_R * GEN_MAX_SUP], coef[GEN_MAX_SUP], res[GEN_MAX_R];
    o.rankdef = 0;
#ifdef SFDT_BINS_PROFILE
    o.iters = 0; o.nminnorm = 0; o.cyc_lsq = 0; o.cyc_top = 0;
#endif
    auto lsq = [&](const int *s, int ns, cx *x) {
        if constexpr (RT > 0) {
            cx yy[RT > 0 ? RT : 1];
#pragma unroll
            for (int j = 0; j < RT; j++) yy[j] = y[j];
            bool ok = false;
            auto fixed = [&](auto cc) {
                constexpr int C = decltype(cc)::value;
                cx Af[C][RT], xx[C];
#pragma unroll
                for (int c = 0; c < C; c++) phi_col(s[c], Af[c]);
                ok = lstsq_qr_t<RT, C>(Af, yy, xx);
                if (ok)
#pragma unroll
                    for (int c = 0; c < C; c++) x[c] = xx[c];
            };
            switch (ns) {
#if SFDT_SP_TMAX >= 1
            case 1: fixed(std::integral_constant<int, 1>{}); break;
#endif
#if SFDT_SP_TMAX >= 2
            case 2: fixed(std::integral_constant<int, 2>{}); break;
#endif
#if SFDT_SP_TMAX >= 3
            case 3: fixed(std::integral_constant<int, 3>{}); break;
#endif
#if SFDT_SP_TMAX >= 4
            case 4: fixed(std::integral_constant<int, 4>{}); break;
#endif
#if SFDT_SP_TMAX >= 5
            case 5: fixed(std::integral_constant<int, 5>{}); break;
#endif
#if SFDT_SP_TMAX >= 6
            case 6: fixed(std::integral_constant<int, 6>{}); break;
#endif
            default:   // larger supports (a_max = 4): the runtime-sized form
                for (int c = 0; c < ns; c++) phi_col(s[c], A + c * r);
                if (lstsq_qr(A, r, ns, y, x)) return;
                break;
            }
            if (ok) return;   // full rank: unique LS solution
            for (int c = 0; c < ns; c++) phi_col(s[c], A + c * r);
        } else {
            for (int c = 0; c < ns; c++) phi_col(s[c], A + c * r);
            if (lstsq_qr(A, r, ns, y, x)) return;   // full rank: unique LS solution
        }
#ifdef SFDT_BINS_PROFILE
        o.nminnorm++;
#endif
        const int rk = lstsq_min_norm(A, r, ns, y, x);
        if (rk < ns) o.rankdef++;
    };
    auto residual = [&](const int *s, int ns, const cx *x) -> double {
        for (int j = 0; j < r; j++) res[j] = y[j];
        for (int c = 0; c < ns; c++) {
            phi_col(s[c], pc);
            for (int j = 0; j < r; j++) res[j] = csub(res[j], nmul(pc[j], x[c]));
        }
        double ss = 0.0;
        for (int j = 0; j < r; j++) ss = fma(res[j].re, res[j].re, fma(res[j].im, res[j].im, ss));
        return sqrt(ss);
    };
    // general.py:212-269 as ONE loop with a single least-squares call site
    // (the pursuit's code is mostly the inlined register-resident QR forms;
    // three copies of them -- initial, merged and pruned supports -- tripled
    // the kernel and its instruction-cache misses).  stage 0 solves on the
    // current support and judges the residual; stage 1 solves on the merged
    // support and prunes it.  Same solves, same order.
    double best = 0.0;
    int best_sup[GEN_MAX_SUP], best_n = 0;
    cx best_coef[GEN_MAX_SUP];
    int merged[2 * GEN_MAX_SUP], nm = 0;
    cx mcoef[2 * GEN_MAX_SUP];
    int stage = 0, it = -1;
    for (;;) {
#ifdef SFDT_BINS_PROFILE
        const long long c0_ = clock64();
#endif
        lsq(stage ? merged : sup, stage ? nm : nsup, stage ? mcoef : coef);
#ifdef SFDT_BINS_PROFILE
        o.cyc_lsq += clock64() - c0_;
        o.iters++;
#endif
        if (stage) {
            // support = sorted(merged[top a_eff of |mcoef|, stable])
            int n2 = 0;
            for (int c = 0; c < nm; c++) topk_insert(tsc, tid_, n2, a_eff, cabs_(mcoef[c]), c);
            nsup = n2;
            for (int i = 0; i < n2; i++) sup[i] = merged[tid_[i]];
            sort_ints(sup, nsup);
            stage = 0;
            continue;
        }
        const double nrm = residual(sup, nsup, coef);
        if (it >= 0 && nrm >= best * (1.0 - 1e-12)) break;
        best = nrm;
        best_n = nsup;
        for (int i = 0; i < nsup; i++) {
            best_sup[i] = sup[i];
            best_coef[i] = coef[i];
        }
        if (++it >= max_iter) break;
        // merged = union(support, top a_eff of |phi^H residual|)
        nt = top_cols(res);
        int topc[GEN_MAX_SUP];
        for (int i = 0; i < nt; i++) topc[i] = tid_[i];
        sort_ints(topc, nt);
        nm = union_sorted(sup, nsup, topc, nt, merged);
        stage = 1;
    }
    o.nsup = best_n;
    for (int i = 0; i < best_n; i++) {
        o.sup[i] = (int)col_t(best_sup[i]);
        o.coef[i] = best_coef[i];
    }
}

// ------------------------------------------------- matched filter (warp)
// general.py:345-351: scores_t = |sum_j conj(base_phi[j, t]) w_j| over the d
// candidates, w_j = e^{-2 pi i s_j k / N} y_j; the top min(a, d) columns by
// (score desc, t asc) -- np.argsort(-scores, kind="stable")[:a].  One WARP
// per voted bin: lane l scores candidates t = l, l+32, ... (coalesced
// base_phi rows, same per-candidate arithmetic and j order as the
// sequential form), keeps a register top-4, and the warp merges the lane
// lists by repeated (score, t) arg-best.  A NaN score ranks last (numpy
// sorts NaN to the end).
struct Top4 {
    double sc[4];
    int id[4];
};

// acc + conj(ph) * w with four FMAs (the matched-filter inner product; the
// reference's BLAS zgemm does not fix the rounding either)
__device__ __forceinline__ cx cjmac(cx acc, cx ph, cx w) {
    return mk(fma(ph.re, w.re, fma(ph.im, w.im, acc.re)), fma(ph.re, w.im, fma(-ph.im, w.re, acc.im)));
}

__device__ __forceinline__ bool mf_better(double v, int t, double w, int u) {
    return v > w || (v == w && t < u);
}

// One CTA per (signal, chunk of mfl <= MF_LIST bins): base_phi (r x d) is
// staged in shared memory once per CTA when it fits (every voted bin of the
// chunk re-reads all of it), the chunk's voted bins are listed in shared
// memory, and each warp scores one bin.
constexpr int MF_SMEM_MAX = 160 * 1024;
constexpr int MF_LIST = 4096;

template <int R, bool STAGE>
__global__ void __launch_bounds__(256, 2) k_gen_mf(const cx *__restrict__ V, GenParams p,
                                                const int32_t *__restrict__ votes,
                                                int32_t *__restrict__ mf_top, int64_t nchunk, int mfl) {
    constexpr bool stage = STAGE;
    extern __shared__ cx s_phi[];
    __shared__ int s_list[MF_LIST];
    __shared__ double s_q2[8][256];
    __shared__ int s_n;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    // CTA = (signal, chunk of MF_LIST bins): long views of few signals
    // still fill the GPU
    const int64_t b = blockIdx.x / nchunk, chunk = blockIdx.x - b * nchunk;
    constexpr int r = R;
    const int64_t *sh = p.shifts + b * p.shift_stride;
    const cx *gphi = p.base_phi + b * p.phi_stride;
    if (stage)
        for (int64_t i = threadIdx.x; i < (int64_t)r * p.d; i += blockDim.x) s_phi[i] = ldcx(gphi + i);
    // explicit address spaces: LDS from the staged copy, LDG otherwise
    auto phi_at = [&](int64_t i) -> cx { return stage ? s_phi[i] : ldcx(gphi + i); };
    for (int64_t c0 = chunk * mfl; c0 < p.L && c0 < (chunk + 1) * mfl; c0 += mfl) {
        if (threadIdx.x == 0) s_n = 0;
        __syncthreads();
        const int64_t c1 = p.L < c0 + mfl ? p.L : c0 + mfl;
        for (int64_t k0 = c0; k0 < c1; k0 += blockDim.x) {   // block-uniform trip count
            const int64_t kb = k0 + threadIdx.x;
            const int a = kb < c1 ? votes[b * p.L + kb] : 0;
            const int64_t count = (int64_t)p.keep * a < p.d ? (int64_t)p.keep * a : p.d;
            const bool want = a >= 1 && p.prune && count < p.d;
            const unsigned m = __ballot_sync(0xffffffffu, want);
            int base = 0;
            if (lane == 0 && m) base = atomicAdd(&s_n, __popc(m));
            base = __shfl_sync(0xffffffffu, base, 0);
            if (want) s_list[base + __popc(m & ((1u << lane) - 1))] = (int)kb;
        }
        __syncthreads();
        const int nlist = s_n;
        for (int li = warp; li < nlist; li += nw) {
            const int64_t kb = s_list[li];
            const int64_t t = b * p.L + kb;
            const int a = votes[t];
            cx wj = mk(0.0, 0.0);
            if (lane < r) {
                const cx yj = ldcx(rview(V, p, b, lane, kb));
                const double th = DMUL(-TWO_PI, (double)(sh[lane] * kb)) / (double)p.n;
                wj = nmul(gexp(mk(0.0, th)), yj);
            }
            cx w[R];
#pragma unroll
            for (int j = 0; j < R; j++) {
                w[j].re = __shfl_sync(0xffffffffu, wj.re, j);
                w[j].im = __shfl_sync(0xffffffffu, wj.im, j);
            }
            const int n_top = (int)((int64_t)a < p.d ? a : p.d);
            Top4 top;
#pragma unroll
            for (int i = 0; i < 4; i++) {
                top.sc[i] = -INFINITY;
                top.id[i] = INT_MAX;
            }
            const int d = (int)p.d;
            auto dot = [&](int tt) -> cx {
                cx acc = mk(0.0, 0.0);
#pragma unroll
                for (int j = 0; j < R; j++) {
                    const cx ph = phi_at(j * d + tt);
                    acc = cjmac(acc, ph, w[j]);
                }
                return acc;
            };
            auto offer = [&](double v, int id) {   // lane list insert
                if (v != v) v = -1.0;   // NaN last (scores are >= 0 otherwise)
#pragma unroll
                for (int i = 0; i < 4; i++) {
                    if (i < n_top && mf_better(v, id, top.sc[i], top.id[i])) {
                        const double ts = top.sc[i];
                        const int ti = top.id[i];
                        top.sc[i] = v;
                        top.id[i] = id;
                        v = ts;
                        id = ti;
                    }
                }
            };
            if (d <= 256) {
                // pass 1: |acc|^2 of the lane's <= 8 candidates; the warp's
                // n_top-th largest square S bounds the winners: a top
                // candidate has |acc|^2 >= S (1 - 1e-13) (hypot and the
                // square agree to a few ulp), so only those get hypot
                double *q2 = s_q2[warp];
                // four candidates per step: independent dot chains give the
                // FP64 pipe ILP (one chain alone waits on every add)
#pragma unroll
                for (int i0 = 0; i0 < 8; i0 += 4) {
                    cx acc[4];
#pragma unroll
                    for (int u = 0; u < 4; u++) acc[u] = mk(0.0, 0.0);
                    const int tb = lane + 32 * i0;
                    if (tb < d) {   // d is a multiple of 32 here or < 32
#pragma unroll
                        for (int j = 0; j < R; j++) {
#pragma unroll
                            for (int u = 0; u < 4; u++) {
                                const int tt = tb + 32 * u;
                                const int tc = tt < d ? tt : tb;
                                const cx ph = phi_at(j * d + tc);
                                acc[u] = cjmac(acc[u], ph, w[j]);
                            }
                        }
                    }
#pragma unroll
                    for (int u = 0; u < 4; u++) {
                        const int tt = tb + 32 * u;
                        double qv = -1.0;
                        if (tt < d) {
                            const double s2 = acc[u].re * acc[u].re + acc[u].im * acc[u].im;
                            qv = (s2 == s2) ? s2 : INFINITY;   // NaN: always re-checked
                        }
                        q2[tt] = qv;
                    }
                }
                double S = INFINITY;
                {
                    uint32_t used = 0;
                    for (int q = 0; q < n_top; q++) {
                        double bv = -2.0;
                        int bi = -1;
#pragma unroll
                        for (int i = 0; i < 8; i++)
                            if (!(used & (1u << i)) && q2[lane + 32 * i] > bv) {
                                bv = q2[lane + 32 * i];
                                bi = i;
                            }
                        double wv = bv;
                        int wl_ = lane;
#pragma unroll
                        for (int o = 16; o > 0; o >>= 1) {
                            const double ov = __shfl_xor_sync(0xffffffffu, wv, o);
                            const int ol = __shfl_xor_sync(0xffffffffu, wl_, o);
                            if (ov > wv || (ov == wv && ol < wl_)) {
                                wv = ov;
                                wl_ = ol;
                            }
                        }
                        if (wl_ == lane && bi >= 0) used |= 1u << bi;
                        S = wv;
                    }
                }
                const double cut = (S > 1e-150 && S < INFINITY) ? S * (1.0 - 1e-13) : -INFINITY;
#pragma unroll
                for (int i = 0; i < 8; i++) {
                    const int tt = lane + 32 * i;
                    if (tt < d && q2[tt] >= cut) offer(cabs_(dot(tt)), tt);
                }
            } else {
                // four of the lane's candidates per step: independent dot
                // chains (and their loads) in flight; same per-candidate
                // arithmetic, offered in the same ascending order
                int tt = lane;
                for (; tt + 96 < d; tt += 128) {
                    cx acc[4];
#pragma unroll
                    for (int u = 0; u < 4; u++) acc[u] = mk(0.0, 0.0);
#pragma unroll
                    for (int j = 0; j < R; j++) {
#pragma unroll
                        for (int u = 0; u < 4; u++) acc[u] = cjmac(acc[u], phi_at(j * d + tt + 32 * u), w[j]);
                    }
#pragma unroll
                    for (int u = 0; u < 4; u++) offer(cabs_(acc[u]), tt + 32 * u);
                }
                for (; tt < d; tt += 32) offer(cabs_(dot(tt)), tt);
            }
            // warp merge: n_top rounds of arg-best over the lane heads
            int sel[4];
#pragma unroll
            for (int q = 0; q < 4; q++) {
                sel[q] = INT_MAX;
                if (q < n_top) {
                    double bv = top.sc[0];
                    int bi = top.id[0];
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) {
                        const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
                        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
                        if (mf_better(ov, oi, bv, bi)) {
                            bv = ov;
                            bi = oi;
                        }
                    }
                    sel[q] = bi;
                    if (top.id[0] == bi) {   // pop the winning lane's head
#pragma unroll
                        for (int i = 0; i < 3; i++) {
                            top.sc[i] = top.sc[i + 1];
                            top.id[i] = top.id[i + 1];
                        }
                        top.sc[3] = -INFINITY;
                        top.id[3] = INT_MAX;
                    }
                }
            }
            if (lane == 0) {
                // sorted ascending (np.sort of the chosen columns)
#pragma unroll
                for (int i = 1; i < 4; i++)
#pragma unroll
                    for (int j2 = 3; j2 >= i; j2--)
                        if (sel[j2 - 1] > sel[j2]) {
                            const int tmp = sel[j2 - 1];
                            sel[j2 - 1] = sel[j2];
                            sel[j2] = tmp;
                        }
                *reinterpret_cast<int4 *>(mf_top + t * 4) = make_int4(sel[0], sel[1], sel[2], sel[3]);
            }
        }
        __syncthreads();
    }
}

// r_eff values with a register-resident pursuit instance: 3*a_max, or d
// when d < 3*a_max
__host__ __device__ __forceinline__ bool sp1_r(int r) {
    return r == 1 || r == 2 || r == 3 || r == 4 || r == 6 || r == 8 || r == 9 || r == 12;
}

__device__ __forceinline__ bool sp1_item(int a, int r, int nc8) {
    return a == 1 && nc8 >= 1 && nc8 <= 4 && sp1_r(r);
}

// Matched filter for short candidate lists (d <= 32): G = max(d, r_eff)
// lanes (a power of two) per voted bin, 32/G bins per warp, lane t scoring
// candidate t with the same per-candidate arithmetic as k_gen_mf (so the
// same scores), the group's top min(a, d) by (score desc, t asc) picked by
// arg-best over the group.  At d = 8 the warp-per-bin form left 24 of 32
// lanes idle.
template <int R, int G>
__global__ void __launch_bounds__(256) k_gen_mf_small(const cx *__restrict__ V, GenParams p,
                                                      const int32_t *__restrict__ votes,
                                                      int32_t *__restrict__ mf_top, int64_t nchunk) {
    __shared__ int s_list[MF_LIST];
    __shared__ int s_n;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int gl = lane & (G - 1), sub = lane / G;
    constexpr int PER_WARP = 32 / G;
    const int64_t b = blockIdx.x / nchunk, chunk = blockIdx.x - b * nchunk;
    const int64_t *sh = p.shifts + b * p.shift_stride;
    const cx *gphi = p.base_phi + b * p.phi_stride;
    const int d = (int)p.d;
    for (int64_t c0 = chunk * MF_LIST; c0 < p.L && c0 < (chunk + 1) * MF_LIST; c0 += MF_LIST) {
        if (threadIdx.x == 0) s_n = 0;
        __syncthreads();
        const int64_t c1 = p.L < c0 + MF_LIST ? p.L : c0 + MF_LIST;
        for (int64_t k0 = c0; k0 < c1; k0 += blockDim.x) {
            const int64_t kb = k0 + threadIdx.x;
            const int a = kb < c1 ? votes[b * p.L + kb] : 0;
            const int64_t count = (int64_t)p.keep * a < p.d ? (int64_t)p.keep * a : p.d;
            const bool want = a >= 1 && p.prune && count < p.d;
            const unsigned m = __ballot_sync(0xffffffffu, want);
            int base = 0;
            if (lane == 0 && m) base = atomicAdd(&s_n, __popc(m));
            base = __shfl_sync(0xffffffffu, base, 0);
            if (want) s_list[base + __popc(m & ((1u << lane) - 1))] = (int)kb;
        }
        __syncthreads();
        const int nlist = s_n;
        // every group of the warp walks the list in lockstep (uniform trips)
        for (int l0 = warp * PER_WARP; l0 < nlist; l0 += nw * PER_WARP) {
            const int li = l0 + sub;
            const bool valid = li < nlist;
            const int64_t kb = valid ? s_list[li] : 0;
            const int64_t t = b * p.L + kb;
            const int a = valid ? votes[t] : 1;
            cx wj = mk(0.0, 0.0);
            if (valid && gl < R) {
                const cx yj = ldcx(rview(V, p, b, gl, kb));
                const double th = DMUL(-TWO_PI, (double)(sh[gl] * kb)) / (double)p.n;
                wj = nmul(gexp(mk(0.0, th)), yj);
            }
            cx acc = mk(0.0, 0.0);
#pragma unroll
            for (int j = 0; j < R; j++) {
                const cx w = mk(__shfl_sync(0xffffffffu, wj.re, j, G), __shfl_sync(0xffffffffu, wj.im, j, G));
                const cx ph = gl < d ? ldcx(gphi + (int64_t)j * d + gl) : mk(0.0, 0.0);
                acc = cjmac(acc, ph, w);
            }
            double v = -INFINITY;
            if (valid && gl < d) {
                v = cabs_(acc);
                if (v != v) v = -1.0;   // NaN last (scores are >= 0 otherwise)
            }
            int id = gl < d ? gl : INT_MAX;
            const int n_top = (int)((int64_t)a < p.d ? a : p.d);
            int sel[4];
#pragma unroll
            for (int q = 0; q < 4; q++) {
                sel[q] = INT_MAX;
                double bv = v;
                int bi = id;
#pragma unroll
                for (int o = G / 2; o > 0; o >>= 1) {
                    const double ov = __shfl_xor_sync(0xffffffffu, bv, o, G);
                    const int oi = __shfl_xor_sync(0xffffffffu, bi, o, G);
                    if (mf_better(ov, oi, bv, bi)) {
                        bv = ov;
                        bi = oi;
                    }
                }
                if (q < n_top) {
                    sel[q] = bi;
                    if (id == bi) {   // the winner leaves the race
                        v = -INFINITY;
                        id = INT_MAX;
                    }
                }
            }
            if (valid && gl == 0) {
#pragma unroll
                for (int i = 1; i < 4; i++)
#pragma unroll
                    for (int j2 = 3; j2 >= i; j2--)
                        if (sel[j2 - 1] > sel[j2]) {
                            const int tmp = sel[j2 - 1];
                            sel[j2 - 1] = sel[j2];
                            sel[j2] = tmp;
                        }
                *reinterpret_cast<int4 *>(mf_top + t * 4) = make_int4(sel[0], sel[1], sel[2], sel[3]);
            }
        }
        __syncthreads();
    }
}

// Pruning per voted bin (general.py:313-351): descending-order Hankel fit,
// prune_eval over the d candidates with the reference's recurrence (or the
// correlation fallback), union with the matched-filter columns (k_gen_mf).
// Writes the kept column list for k_gen_bins; ncols = -1 means "all d
// columns" (no pruning).  Split from the pursuit so each kernel keeps its
// own registers, stack and instruction footprint.
// LANES = 4 (d >= 1024, d % 512 == 0): four lanes per bin, lane l scoring
// the 512-candidate segments l, l + 4, ... (the recurrence re-seeds at every
// segment start, so each segment's values are the same bits), then lane 0
// merges the four bottom-k lists in the (value, index) order the serial
// scan keeps.  For the few-bins, large-d shapes (config 5 general, K = 64).
template <int LANES>
__global__ void __launch_bounds__(128) k_gen_prune(const cx *__restrict__ V, GenParams p,
                                                   const int32_t *__restrict__ votes,
                                                   const int64_t *__restrict__ wl,
                                                   const unsigned long long *__restrict__ wl_count,
                                                   const int32_t *__restrict__ mf_top,
                                                   int32_t *__restrict__ cols_out, int8_t *__restrict__ ncols_out,
                                                   int heavy_flags, int64_t *__restrict__ hl,
                                                   unsigned long long *__restrict__ hlc, int64_t hl_cap,
                                                   unsigned long long *__restrict__ hlc_hi, int split_a) {
    const int64_t cnt = (int64_t)*wl_count;
    const int sub = LANES > 1 ? (int)(threadIdx.x & (LANES - 1)) : 0;
    for (int64_t it = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) / LANES; it < cnt;
         it += int64_t(gridDim.x) * blockDim.x / LANES) {
        const int64_t t = wl[it];
        const int a = votes[t];
        const int64_t b = t / p.L, kb = t - b * p.L;
        const int r = p.r_eff;
        const int64_t *sh = p.shifts + b * p.shift_stride;
        cx syn[8], y[GEN_MAX_R];
        for (int j = 0; j < p.S; j++) syn[j] = ldcx(V + (b * p.nv + j) * p.L + kb);
        for (int j = 0; j < r; j++) y[j] = ldcx(rview(V, p, b, j, kb));
        const int64_t count = (int64_t)p.keep * a < p.d ? (int64_t)p.keep * a : p.d;
        int cols[GEN_MAX_COLS];
        int ncols = 0;
        bool all_cols = true;
        if (p.prune && count < p.d) {
            all_cols = false;
            // descending-order Hankel fit (general.py:324-337)
            cx c[4];
            int order = 0;
            for (int o2 = p.a_max; o2 >= 1; o2--) {
                double scale = 0.0;
                for (int l = 0; l < 2 * o2; l++) scale = nanmax2(scale, cabs_(syn[l]));
                scale = nanmax2(scale, TINY);
                const cx cd = hankel_solve1(syn, o2, c);
                if (cabs_(cd) > DMUL(SINGULARITY_RTOL, powa(scale, o2))) {
                    order = o2;
                    break;
                }
            }
            double ks[GEN_MAX_COLS];
            int kp[GEN_MAX_COLS], nk = 0;
            const int cnti = (int)count;
            if (order > 0) {
                // prune_eval (_core.pyx:319-346) with the same recurrence
                const cx base = gexp(mk(0.0, DMUL(TWO_PI, (double)kb) / (double)p.n));
                const cx wd = gexp(mk(0.0, TWO_PI / (double)p.d));
                cx zt = base;
                // |acc|^2 pre-filter: once the kept list is full, a candidate
                // whose squared magnitude exceeds cut^2 (1 + 1e-13) is
                // certainly not below the cut (hypot and the square differ by
                // a few ulps), so the hypot and the insertion are skipped
                double cut2 = INFINITY;
                // Horner in descending order with the coefficients in
                // registers (constant indices, predicated on the order)
                const cx cr[4] = {c[0], order > 1 ? c[1] : mk(0.0, 0.0), order > 2 ? c[2] : mk(0.0, 0.0),
                                  order > 3 ? c[3] : mk(0.0, 0.0)};
                auto horner = [&](cx z) -> cx {
                    cx acc = mk(1.0, 0.0);
#pragma unroll
                    for (int j = 3; j >= 0; j--)
                        if (j < order) acc = cadd(gmul(acc, z), cr[j]);
                    return acc;
                };
                auto offer = [&](cx acc, int tt) {
                    const double q = acc.re * acc.re + acc.im * acc.im;
                    if (!(q > cut2)) {
                        botk_insert(ks, kp, nk, cnti, cabs_(acc), tt);
                        if (nk == cnti) cut2 = ks[cnti - 1] * ks[cnti - 1] * (1.0 + 1e-13);
                    }
                };
                // the recurrence z *= wd, re-seeded at every 512th candidate
                auto advance = [&](cx z, int64_t tt) -> cx {
                    return ((tt & 511) == 511)
                        ? gmul(base, gexp(mk(0.0, DMUL(TWO_PI, (double)(tt + 1)) / (double)p.d)))
                        : gmul(z, wd);
                };
                if (LANES > 1) {
                    // this lane's 512-candidate segments, each from its re-seed
                    for (int64_t s0 = (int64_t)sub * 512; s0 < p.d; s0 += (int64_t)LANES * 512) {
                        zt = s0 == 0 ? base : gmul(base, gexp(mk(0.0, DMUL(TWO_PI, (double)s0) / (double)p.d)));
                        for (int64_t tt = s0; tt < s0 + 512; tt += 4) {
                            const cx z0 = zt, z1 = advance(z0, tt), z2 = advance(z1, tt + 1),
                                     z3 = advance(z2, tt + 2);
                            zt = advance(z3, tt + 3);
                            const cx a0 = horner(z0), a1 = horner(z1), a2 = horner(z2), a3 = horner(z3);
                            offer(a0, (int)tt);
                            offer(a1, (int)tt + 1);
                            offer(a2, (int)tt + 2);
                            offer(a3, (int)tt + 3);
                        }
                    }
                } else if ((p.d & 3) == 0) {
                    // four candidates per step: independent Horner chains
                    for (int64_t tt = 0; tt < p.d; tt += 4) {
                        const cx z0 = zt, z1 = advance(z0, tt), z2 = advance(z1, tt + 1),
                                 z3 = advance(z2, tt + 2);
                        zt = advance(z3, tt + 3);
                        const cx a0 = horner(z0), a1 = horner(z1), a2 = horner(z2), a3 = horner(z3);
                        offer(a0, (int)tt);
                        offer(a1, (int)tt + 1);
                        offer(a2, (int)tt + 2);
                        offer(a3, (int)tt + 3);
                    }
                } else {
                    for (int64_t tt = 0; tt < p.d; tt++) {
                        offer(horner(zt), (int)tt);
                        zt = advance(zt, tt);
                    }
                }
            } else if (sub == 0) {
                // _correlation_keep (general.py:158-165)
                const int64_t m = p.L;
                for (int64_t tt = 0; tt < p.d; tt++) {
                    const int64_t loc = (kb + tt * m) & (p.n - 1);
                    cx acc = mk(0.0, 0.0);
                    for (int j = 0; j < r; j++) {
                        const double th = DMUL(TWO_PI, (double)(sh[j] * loc)) / (double)p.n;
                        acc = cadd(acc, nmul(cconj(gexp(mk(0.0, th))), y[j]));
                    }
                    topk_insert(ks, kp, nk, cnti, cabs_(acc), (int)tt);
                }
            }
            if (LANES > 1) {
                // lane 0 merges lanes 1..3: lexicographic (value, index)
                // bottom-k, what the serial ascending-index scan keeps
                const unsigned gm = 0xFu << (threadIdx.x & 28);
                const int base_lane = (int)(threadIdx.x & 28);
                for (int l = 1; l < LANES; l++) {
                    const int nl = __shfl_sync(gm, nk, base_lane + l);
                    for (int e = 0; e < cnti; e++) {
                        const double v = __shfl_sync(gm, e < nk ? ks[e] : 0.0, base_lane + l);
                        const int tv = __shfl_sync(gm, e < nk ? kp[e] : 0, base_lane + l);
                        if (sub != 0 || e >= nl) continue;
                        // (value, index) order with NaN last -- botk_insert's order
                        auto before = [&](double w, int tw) {
                            return score_before_asc(v, w) || ((v == w || (v != v && w != w)) && tv < tw);
                        };
                        if (nk == cnti && !before(ks[cnti - 1], kp[cnti - 1])) continue;
                        int pos = (nk < cnti) ? nk++ : cnti - 1;
                        while (pos > 0 && before(ks[pos - 1], kp[pos - 1])) {
                            ks[pos] = ks[pos - 1];
                            kp[pos] = kp[pos - 1];
                            pos--;
                        }
                        ks[pos] = v;
                        kp[pos] = tv;
                    }
                }
            }
            sort_ints(kp, nk);
            // matched-filter augmentation (general.py:345-351): k_gen_mf
            const int nt = (int)((int64_t)a < p.d ? a : p.d);
            const int4 mft = *reinterpret_cast<const int4 *>(mf_top + t * 4);
            const int tp[4] = {mft.x, mft.y, mft.z, mft.w};
            ncols = union_sorted(kp, nk, tp, nt, cols);
        } else {
            ncols = (int)p.d;
        }
        if (sub != 0) continue;   // lane 0 of the group writes
        if (!all_cols) {
            for (int c2 = 0; c2 < ncols; c2++) cols_out[it * GEN_MAX_COLS + c2] = cols[c2];
            ncols_out[it] = (int8_t)ncols;
        } else {
            ncols_out[it] = -1;
        }
        // the bins k_gen_bins pursues go to a separate list so that each gets
        // its own warp there (bit 0: k_gen_sp1 takes its items, bit 1:
        // k_gen_bins_warp takes the all-column bins)
        const int nc = all_cols ? -1 : ncols;
        const bool heavy = !((heavy_flags & 1) && sp1_item(a, r, nc)) && !((heavy_flags & 2) && nc < 0);
        // bins with a >= split_a (the longer pursuits) fill the list from
        // its end, so k_gen_bins can deal them first
        if (heavy) {
            if (split_a > 0 && a >= split_a) hl[hl_cap - 1 - (int64_t)atomicAdd(hlc_hi, 1ull)] = it;
            else hl[atomicAdd(hlc, 1ull)] = it;
        }
    }
}

// ------------------------------------------- subspace pursuit, a_sp = 1
// Register-resident pursuit for the dominant case -- a single-collision bin
// on a pruned list of <= 4 columns -- in its own kernel (k_gen_sp1), so its
// registers do not inflate the generic kernel.  Same operations in the same
// order as subspace_pursuit_dev with a_eff = 1: stable first-max
// selections, Householder least squares with the min-norm fallback, the
// 1e-12 stopping rule.  A is overwritten (rebuilt for the fallback).
template <int R>
__device__ __forceinline__ void sp_a1_t(const cx (&y)[R], const cx (&phase)[R], const cx *bphi, int64_t d,
                                        const int *cols, int ncols, SPOut &o) {
    auto phi_col = [&](int c, cx (&out)[R]) {
        const int64_t t = (int64_t)cols[c];
#pragma unroll
        for (int j = 0; j < R; j++) out[j] = nmul(phase[j], ldcx(bphi + (int64_t)j * d + t));
    };
    // first max of |phi_c^H v| over the columns (topk_insert with cnt = 1)
    auto argmax_cols = [&](const cx (&v)[R]) -> int {
        int bi = -1;
        double bv = 0.0;
        for (int c = 0; c < ncols; c++) {
            cx pc[R];
            phi_col(c, pc);
            cx acc = mk(0.0, 0.0);
#pragma unroll
            for (int j = 0; j < R; j++) acc = cadd(acc, nmul(cconj(pc[j]), v[j]));
            const double sc = cabs_(acc);
            if (bi < 0 || sc > bv) {
                bv = sc;
                bi = c;
            }
        }
        return bi;
    };
    o.rankdef = 0;
    auto lsq1 = [&](int c0, cx &x) {
        cx A[1][R], xx[1];
        phi_col(c0, A[0]);
        if (lstsq_qr_t<R, 1>(A, y, xx)) {
            x = xx[0];
            return;
        }
        cx Af[R];
        phi_col(c0, A[0]);
#pragma unroll
        for (int i = 0; i < R; i++) Af[i] = A[0][i];
        if (lstsq_min_norm(Af, R, 1, y, xx) < 1) o.rankdef++;
        x = xx[0];
    };
    auto lsq2 = [&](int c0, int c1, cx &x0, cx &x1) {
        cx A[2][R], xx[2];
        phi_col(c0, A[0]);
        phi_col(c1, A[1]);
        if (!lstsq_qr_t<R, 2>(A, y, xx)) {
            phi_col(c0, A[0]);
            phi_col(c1, A[1]);
            cx Af[2 * R];
#pragma unroll
            for (int i = 0; i < R; i++) {
                Af[i] = A[0][i];
                Af[R + i] = A[1][i];
            }
            if (lstsq_min_norm(Af, R, 2, y, xx) < 2) o.rankdef++;
        }
        x0 = xx[0];
        x1 = xx[1];
    };
    cx res[R];
    auto residual = [&](int c0, cx x) -> double {
        cx pc[R];
        phi_col(c0, pc);
        double ss = 0.0;
#pragma unroll
        for (int j = 0; j < R; j++) {
            res[j] = csub(y[j], nmul(pc[j], x));
            ss = fma(res[j].re, res[j].re, fma(res[j].im, res[j].im, ss));
        }
        return sqrt(ss);
    };
    int sup = argmax_cols(y);
    cx coef;
    lsq1(sup, coef);
    double best = residual(sup, coef);
    int best_sup = sup;
    cx best_coef = coef;
    for (int it = 0; it < 10; it++) {
        const int topc = argmax_cols(res);
        if (topc == sup) {
            cx mc;
            lsq1(sup, mc);   // the merged solve (its rank counts, its value is unused)
        } else {
            const int m0 = sup < topc ? sup : topc, m1 = sup < topc ? topc : sup;
            cx mc0, mc1;
            lsq2(m0, m1, mc0, mc1);
            sup = (cabs_(mc1) > cabs_(mc0)) ? m1 : m0;   // top 1 of |mcoef|, first max
        }
        lsq1(sup, coef);
        const double nrm = residual(sup, coef);
        if (nrm >= best * (1.0 - 1e-12)) break;
        best = nrm;
        best_sup = sup;
        best_coef = coef;
    }
    o.nsup = 1;
    o.sup[0] = cols[best_sup];
    o.coef[0] = best_coef;
}

template <int R>
__global__ void __launch_bounds__(128) k_gen_sp1(const cx *__restrict__ V, GenParams p,
                                                 const int32_t *__restrict__ votes,
                                                 const int64_t *__restrict__ wl,
                                                 const unsigned long long *__restrict__ wl_count,
                                                 const int32_t *__restrict__ cols_in,
                                                 const int8_t *__restrict__ ncols_in,
                                                 uint8_t *__restrict__ nent, int64_t *__restrict__ sloc,
                                                 cx *__restrict__ sval, int64_t *__restrict__ stats) {
    const int64_t cnt = (int64_t)*wl_count;
    for (int64_t it = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; it < cnt;
         it += int64_t(gridDim.x) * blockDim.x) {
        const int64_t t = wl[it];
        const int a = votes[t];
        const int nc8 = ncols_in[it];
        if (!sp1_item(a, R, nc8)) continue;
        const int64_t b = t / p.L, kb = t - b * p.L;
        const int64_t *sh = p.shifts + b * p.shift_stride;
        const cx *bphi = p.base_phi + b * p.phi_stride;
        cx y[R], phase[R];
        const double tk = DMUL(TWO_PI, (double)kb);
#pragma unroll
        for (int j = 0; j < R; j++) {
            y[j] = ldcx(rview(V, p, b, j, kb));
            phase[j] = gexp(mk(0.0, DMUL(tk, (double)sh[j]) / (double)p.n));
        }
        int cols[4];
#pragma unroll
        for (int c2 = 0; c2 < 4; c2++) cols[c2] = c2 < nc8 ? cols_in[it * GEN_MAX_COLS + c2] : 0;
        SPOut o;
        sp_a1_t<R>(y, phase, bphi, p.d, cols, nc8, o);
        int ne = 0;
        if (!(o.coef[0].re == 0.0 && o.coef[0].im == 0.0)) {   // np.nonzero(coef)
            sloc[t * p.a_max] = (kb + (int64_t)o.sup[0] * p.L) & (p.n - 1);
            stcx(sval + t * p.a_max, o.coef[0]);
            ne = 1;
        }
        nent[t] = (uint8_t)ne;
        if (o.rankdef)
            atomicAdd((unsigned long long *)(stats + b * SFDT_GS_PER_SIGNAL + SFDT_GS_RANKDEF),
                      (unsigned long long)o.rankdef);
    }
}

// Subspace pursuit per voted bin on the kept columns (general.py:357-366),
// for the bins on k_gen_prune's list (multi-collision bins and the rest
// k_gen_sp1 / k_gen_bins_warp do not take).  Each bin is a long serial FP64
// chain (~1e5 cycles, measured), so the list is dealt out lane-major: item q
// goes to lane q / nwarps of warp q % nwarps -- with fewer items than warps
// no two chains share a warp (divergent lanes would run them one after the
// other).
#ifndef SFDT_BINS_MINB
#define SFDT_BINS_MINB 2   // resident CTAs per SM (255 registers; 3 / 4 spill -- measured, profiles/r02_bins_minb)
#endif
template <int RT>
__global__ void __launch_bounds__(128, SFDT_BINS_MINB) k_gen_bins(const cx *__restrict__ V, GenParams p,
                                                  const int32_t *__restrict__ votes,
                                                  const int64_t *__restrict__ wl,
                                                  const int64_t *__restrict__ hl,
                                                  const unsigned long long *__restrict__ hl_count,
                                                  const int32_t *__restrict__ cols_in,
                                                  const int8_t *__restrict__ ncols_in,
                                                  uint8_t *__restrict__ nent, int64_t *__restrict__ sloc,
                                                  cx *__restrict__ sval, int64_t *__restrict__ stats,
                                                  unsigned long long *__restrict__ hl_next, int deal_max,
                                                  const unsigned long long *__restrict__ hl_hi_count,
                                                  int64_t hl_cap) {
    // item q < cnt_hi: the a >= split_a bins (hl's tail, longer chains);
    // then the rest from hl's head
    const int64_t cnt_hi = (int64_t)*hl_hi_count;
    const int64_t cnt = (int64_t)*hl_count + cnt_hi;
    const int64_t nwarps = int64_t(gridDim.x) * (blockDim.x >> 5);
    const int64_t gw = int64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    // up to deal_max bins per warp: dealt lane-major (item q to lane
    // q / nwarps of warp q % nwarps), so every warp of the wave holds at
    // most ceil(cnt / nwarps) chains -- one when cnt <= nwarps.  Beyond
    // that (no pruning: every voted bin) every thread takes the next bin
    // from a counter, so the long and short chains balance dynamically.
    // (A counter at a few bins per warp hands each warp 32 consecutive
    // items: the chains would pile into cnt / 32 warps.)
    // Lanes >= 1 take their items in reverse warp order, so the first
    // (longest) items on lane 0 of the low warps pair with the last ones.
    const bool dealt = cnt <= (int64_t)deal_max * nwarps;
    if (dealt && (int64_t)lane * nwarps >= cnt) return;
    for (int64_t q = dealt ? (lane ? nwarps - 1 - gw : gw) + lane * nwarps : (int64_t)atomicAdd(hl_next, 1ull);
         q < cnt; q = dealt ? cnt : (int64_t)atomicAdd(hl_next, 1ull)) {
        const int64_t it = q < cnt_hi ? hl[hl_cap - 1 - q] : hl[q - cnt_hi];
        const int64_t t = wl[it];
        const int a = votes[t];
        const int r = RT > 0 ? RT : p.r_eff;
        const int64_t b = t / p.L, kb = t - b * p.L;
        const int64_t *sh = p.shifts + b * p.shift_stride;
        const cx *bphi = p.base_phi + b * p.phi_stride;
        cx y[GEN_MAX_R];
#pragma unroll
        for (int j = 0; j < (RT > 0 ? RT : GEN_MAX_R); j++) {
            if (RT == 0 && j >= r) break;
            y[j] = ldcx(rview(V, p, b, j, kb));
        }
        int cols[GEN_MAX_COLS];
        const int nc8 = ncols_in[it];
        const bool all_cols = nc8 < 0;
        const int ncols = all_cols ? (int)p.d : nc8;
        for (int c2 = 0; c2 < (all_cols ? 0 : ncols); c2++) cols[c2] = cols_in[it * GEN_MAX_COLS + c2];
        // subspace pursuit on this bin's columns (general.py:357-366)
        cx phase[GEN_MAX_R];
        const double tk = DMUL(TWO_PI, (double)kb);
#pragma unroll
        for (int j = 0; j < (RT > 0 ? RT : GEN_MAX_R); j++) {
            if (RT == 0 && j >= r) break;
            phase[j] = gexp(mk(0.0, DMUL(tk, (double)sh[j]) / (double)p.n));
        }
        const int a_sp = a < r ? a : r;
        SPOut o;
#ifdef SFDT_BINS_PROFILE
        const long long c0 = clock64();
#endif
        subspace_pursuit_dev<RT>(y, phase, bphi, p.d, r, cols, ncols, all_cols, a_sp, o);
#ifdef SFDT_BINS_PROFILE
        {
            const long long dc = clock64() - c0;
            if (dc > 150000 || (q & 63) == 0)
                printf("BIN q=%lld a=%d ncols=%d nsup=%d lsqcalls=%d minnorm=%d rankdef=%d cyc=%lld cyc_lsq=%lld lane=%d\n", (long long)q, a, ncols, o.nsup,
                       o.iters, o.nminnorm, o.rankdef, dc, o.cyc_lsq, lane);
        }
#endif
        int ne = 0;
        for (int i = 0; i < o.nsup; i++) {
            if (o.coef[i].re == 0.0 && o.coef[i].im == 0.0) continue;   // np.nonzero(coef)
            sloc[t * p.a_max + ne] = (kb + (int64_t)o.sup[i] * p.L) & (p.n - 1);
            stcx(sval + t * p.a_max + ne, o.coef[i]);
            ne++;
        }
        nent[t] = (uint8_t)ne;
        if (o.rankdef)
            atomicAdd((unsigned long long *)(stats + b * SFDT_GS_PER_SIGNAL + SFDT_GS_RANKDEF),
                      (unsigned long long)o.rankdef);
    }
}

// One WARP per bin for the bins whose pursuit scores all d columns (no
// pruning, general.py:352-354): the column scans of subspace pursuit are
// spread over the lanes (k_gen_bins skips these bins).
__global__ void __launch_bounds__(256) k_gen_bins_warp(const cx *__restrict__ V, GenParams p,
                                                       const int32_t *__restrict__ votes,
                                                       const int64_t *__restrict__ wl,
                                                       const unsigned long long *__restrict__ wl_count,
                                                       const int8_t *__restrict__ ncols_in,
                                                       uint8_t *__restrict__ nent, int64_t *__restrict__ sloc,
                                                       cx *__restrict__ sval, int64_t *__restrict__ stats) {
    const int64_t cnt = (int64_t)*wl_count;
    const int lane = threadIdx.x & 31;
    const int64_t nw = int64_t(gridDim.x) * (blockDim.x >> 5);
    for (int64_t it = int64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); it < cnt; it += nw) {
        if (ncols_in[it] >= 0) continue;   // pruned bins: k_gen_sp1 / k_gen_bins
        const int64_t t = wl[it];
        const int a = votes[t];
        const int r = p.r_eff;
        const int64_t b = t / p.L, kb = t - b * p.L;
        const int64_t *sh = p.shifts + b * p.shift_stride;
        const cx *bphi = p.base_phi + b * p.phi_stride;
        cx y[GEN_MAX_R], phase[GEN_MAX_R];
        const double tk = DMUL(TWO_PI, (double)kb);
        for (int j = 0; j < r; j++) {
            y[j] = ldcx(rview(V, p, b, j, kb));
            phase[j] = gexp(mk(0.0, DMUL(tk, (double)sh[j]) / (double)p.n));
        }
        const int a_sp = a < r ? a : r;
        SPOut o;
        subspace_pursuit_dev(y, phase, bphi, p.d, r, nullptr, (int)p.d, true, a_sp, o, lane, 32);
        if (lane == 0) {
            int ne = 0;
            for (int i = 0; i < o.nsup; i++) {
                if (o.coef[i].re == 0.0 && o.coef[i].im == 0.0) continue;   // np.nonzero(coef)
                sloc[t * p.a_max + ne] = (kb + (int64_t)o.sup[i] * p.L) & (p.n - 1);
                stcx(sval + t * p.a_max + ne, o.coef[i]);
                ne++;
            }
            nent[t] = (uint8_t)ne;
            if (o.rankdef)
                atomicAdd((unsigned long long *)(stats + b * SFDT_GS_PER_SIGNAL + SFDT_GS_RANKDEF),
                          (unsigned long long)o.rankdef);
        }
    }
}

// -------------------------------------------------------------- compaction
// A signal's bins are split into segments of GEN_SEG bins (one CTA each) so
// long views of few signals fill the GPU: per-segment class counts, folded
// per signal, and each segment emitted at its signal's class bases plus
// the counts of the segments before it.
constexpr int64_t GEN_SEG = 8192;

__global__ void __launch_bounds__(256) k_gen_count(const int32_t *__restrict__ votes,
                                                   const uint8_t *__restrict__ nent, int64_t L,
                                                   int64_t nseg, long long *__restrict__ segcnt) {
    const int64_t b = blockIdx.x / nseg, g = blockIdx.x - b * nseg;
    const int64_t k0 = g * GEN_SEG, k1 = (k0 + GEN_SEG < L) ? k0 + GEN_SEG : L;
    long long c[4] = {0, 0, 0, 0};
    for (int64_t kb = k0 + threadIdx.x; kb < k1; kb += blockDim.x) {
        const int v = votes[b * L + kb];
        if (v >= 1) c[v - 1] += nent[b * L + kb];
    }
    __shared__ long long red[4][256];
    for (int q = 0; q < 4; q++) red[q][threadIdx.x] = c[q];
    __syncthreads();
    for (int s = 128; s > 0; s >>= 1) {
        if (threadIdx.x < s)
            for (int q = 0; q < 4; q++) red[q][threadIdx.x] += red[q][threadIdx.x + s];
        __syncthreads();
    }
    if (threadIdx.x < 4) segcnt[blockIdx.x * 4 + threadIdx.x] = red[threadIdx.x][0];
}

__global__ void k_gen_fin(const long long *__restrict__ segcnt, int64_t B, int64_t nseg,
                          int64_t *__restrict__ stats) {
    const int64_t b = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (b >= B) return;
    long long r[4] = {0, 0, 0, 0};
    for (int64_t g = 0; g < nseg; g++)
        for (int q = 0; q < 4; q++) r[q] += segcnt[(b * nseg + g) * 4 + q];
    int64_t *st = stats + b * SFDT_GS_PER_SIGNAL;
    long long tot = 0;
    for (int q = 0; q < 4; q++) {
        st[SFDT_GS_CLASS0 + q] = r[q];
        tot += r[q];
    }
    st[SFDT_GS_NENTRIES] = tot;
}

__global__ void k_gen_scan(const int64_t *__restrict__ stats, int64_t B, int64_t *__restrict__ offsets) {
    __shared__ long long buf[1024];
    __shared__ long long carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int64_t base = 0; base < B; base += 1024) {
        const int64_t i = base + threadIdx.x;
        const long long v = (i < B) ? stats[i * SFDT_GS_PER_SIGNAL + SFDT_GS_NENTRIES] : 0;
        buf[threadIdx.x] = v;
        __syncthreads();
        for (int s = 1; s < 1024; s <<= 1) {
            const long long add = (threadIdx.x >= s) ? buf[threadIdx.x - s] : 0;
            __syncthreads();
            buf[threadIdx.x] += add;
            __syncthreads();
        }
        if (i < B) offsets[i] = carry + buf[threadIdx.x] - v;
        __syncthreads();
        if (threadIdx.x == 1023) carry += buf[1023];
        __syncthreads();
    }
    if (threadIdx.x == 0) offsets[B] = carry;
}

// entries in (vote class asc, bin asc, column asc) order; per tile one block
// scan of 4 x 13-bit packed per-class entry counts
__global__ void __launch_bounds__(256) k_gen_emit(const int32_t *__restrict__ votes,
                                                  const uint8_t *__restrict__ nent,
                                                  const int64_t *__restrict__ sloc,
                                                  const cx *__restrict__ sval, int64_t L, int a_max,
                                                  const int64_t *__restrict__ stats,
                                                  const int64_t *__restrict__ eoff,
                                                  int64_t *__restrict__ locs, cx *__restrict__ vals,
                                                  int64_t nseg, const long long *__restrict__ segcnt) {
    __shared__ unsigned long long wtot[8];
    const int64_t b = blockIdx.x / nseg, g = blockIdx.x - b * nseg;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t *st = stats + b * SFDT_GS_PER_SIGNAL;
    long long base[4];
    base[0] = eoff[b];
    for (int c = 1; c < 4; c++) base[c] = base[c - 1] + st[SFDT_GS_CLASS0 + c - 1];
    for (int64_t g2 = 0; g2 < g; g2++)
        for (int c = 0; c < 4; c++) base[c] += segcnt[(b * nseg + g2) * 4 + c];
    long long carry[4] = {0, 0, 0, 0};
    const int64_t k0 = g * GEN_SEG, k1 = (k0 + GEN_SEG < L) ? k0 + GEN_SEG : L;
    for (int64_t t0 = k0; t0 < k1; t0 += 1024) {
        int ci[4], ne[4];
        unsigned long long packed = 0;
#pragma unroll
        for (int u = 0; u < 4; u++) {
            const int64_t kb = t0 + 4 * threadIdx.x + u;
            ci[u] = -1;
            ne[u] = 0;
            if (kb < k1) {
                const int v = votes[b * L + kb];
                if (v >= 1) {
                    ci[u] = v - 1;
                    ne[u] = nent[b * L + kb];
                    packed += (unsigned long long)ne[u] << (13 * ci[u]);
                }
            }
        }
        unsigned long long inc = packed;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += y;
        }
        if (lane == 31) wtot[warp] = inc;
        __syncthreads();
        unsigned long long before = 0, total = 0;
        for (int w2 = 0; w2 < 8; w2++) {
            before += (w2 < warp) ? wtot[w2] : 0;
            total += wtot[w2];
        }
        __syncthreads();
        const unsigned long long pre = before + inc - packed;
#pragma unroll
        for (int u = 0; u < 4; u++) {
            const int c = ci[u];
            if (c < 0) continue;
            long long pos = base[c] + carry[c] + (long long)((pre >> (13 * c)) & 0x1FFF);
            for (int u2 = 0; u2 < u; u2++)
                if (ci[u2] == c) pos += ne[u2];
            const int64_t t = b * L + t0 + 4 * threadIdx.x + u;
            for (int j = 0; j < ne[u]; j++) {
                locs[pos + j] = sloc[t * a_max + j];
                stcx(vals + pos + j, sval[t * a_max + j]);
            }
        }
#pragma unroll
        for (int c = 0; c < 4; c++) carry[c] += (long long)((total >> (13 * c)) & 0x1FFF);
    }
}

// --------------------------------------------------------------- host side
struct GenPlan {
    int64_t B, n, d, L, nv, nparts;
    int S;
    size_t off_V, off_sv, off_part, off_votes, off_nent, off_sloc, off_sval, off_wl, off_cnt,
        off_fft, off_mf, off_cols, off_ncols, off_hl, off_vsh, off_vslot, off_nview, off_fix, off_cand, off_seg, off_vsel, off_ghist, off_eqc, off_win, off_winf, total;
    int win;   // window-ring look-ahead in signals (0: each view gathers its own samples)
    int x_host;   // the signals live in host-mapped memory
    int wing;     // window gather kernel + FFT from its buffer (host-mapped signals, L != 4096)
};

static int make_gen_plan(const sfdt_general_args *a, GenPlan &p) {
    if (!a || a->batch < 1 || a->n < 2 || (a->n & (a->n - 1))) return SFDT_EINVAL;
    if (a->a_max < 1 || a->a_max > 4 || a->d < 1 || a->d > a->n || (a->d & (a->d - 1))) return SFDT_EINVAL;
    if (a->r_eff < 1 || a->r_eff > GEN_MAX_R || a->r_eff > a->d || a->k < 1) return SFDT_EINVAL;
    if (a->keep_per_collision < 1 || a->keep_per_collision * a->a_max + a->a_max > GEN_MAX_COLS)
        return SFDT_EINVAL;
    if (2 * a->a_max + a->r_eff > MAX_VIEWS) return SFDT_EINVAL;
    if (a->x_dtype != SFDT_C128 && a->x_dtype != SFDT_C64) return SFDT_EINVAL;
    {
        // the A/B switches, validated before anything is enqueued
        const sfdt_tuning t = tuning_or_default(a->tuning);
        if (t.gen_mf_list != 0 && (t.gen_mf_list < 32 || t.gen_mf_list > MF_LIST)) return SFDT_EINVAL;
        if (t.gen_prune_lanes != 0 && t.gen_prune_lanes != 1 && t.gen_prune_lanes != 4) return SFDT_EINVAL;
        if (t.gen_warp < -1 || t.gen_warp > 1 || t.gen_deal < 0 || t.gen_split_a < 0) return SFDT_EINVAL;
        if (t.gen_window < -4 || t.gen_window > 256) return SFDT_EINVAL;
    }
    p.B = a->batch;
    p.n = a->n;
    p.d = a->d;
    p.L = a->n / a->d;
    p.S = 2 * a->a_max;
    p.nv = p.S + a->r_eff;
    p.nparts = (p.L + 127) / 128;
    size_t o = 0;
    auto take = [&](size_t bytes) { size_t r = o; o = (o + bytes + 255) & ~size_t(255); return r; };
    p.off_V = take(size_t(p.B) * p.nv * p.L * 16);
    p.off_sv = take(size_t(p.B) * p.L * a->a_max * 8);
    p.off_part = take(size_t(p.B) * p.nparts * 8);
    p.off_votes = take(size_t(p.B) * p.L * 4);
    p.off_nent = take(size_t(p.B) * p.L);
    p.off_sloc = take(size_t(p.B) * p.L * a->a_max * 8);
    p.off_sval = take(size_t(p.B) * p.L * a->a_max * 16);
    p.off_wl = take(size_t(p.B) * p.L * 8);
    p.off_cnt = take(64);   // worklist count, heavy-list count
    p.off_mf = take(size_t(p.B) * p.L * 16);
    {
        // voted bins per signal <= min(k, L) (each vote is one of the top k keys)
        const int64_t cap = p.B * (a->k < p.L ? a->k : p.L);
        p.off_cols = take(size_t(cap) * GEN_MAX_COLS * 4);
        p.off_ncols = take(size_t(cap));
        p.off_hl = take(size_t(cap) * 8);
    }
    p.off_seg = take(size_t(p.B) * ((p.L + GEN_SEG - 1) / GEN_SEG) * 4 * 8);
    p.off_vsel = take(size_t(p.B) * sizeof(VSel));
    p.off_ghist = take(size_t(p.B) * 256 * 4);
    p.off_cand = (p.L * a->a_max > VOTE_BIG) ? take(size_t(p.B) * VSEL_CAND * 8) : 0;
    p.off_eqc = take(size_t(p.B) * ((p.L * a->a_max + VCH - 1) / VCH) * 8);
    p.off_vsh = take(size_t(p.B) * a->r_eff * 8);
    p.off_vslot = take(size_t(p.B) * a->r_eff * 4);
    p.off_nview = take(size_t(p.B) * 4);
    p.off_fix = (a->a_max == 3) ? take(size_t(p.B) * p.L * 8) : 0;
    p.off_fft = (p.L > FFT_SMEM_MAX) ? take(size_t(p.B) * p.nv * p.L * 16) : 0;
    {
        // gen_window < 0 (auto): the window ring for host-mapped signals (zero-copy
        // end-to-end path: a d-block's six consecutive shifts become one PCIe read
        // instead of six from six CTAs, config 4 e2e 6.4k -> 14.7k signals/s), each
        // view gathering its own samples for signals in HBM (0.95 vs 1.55 ms)
        int look = tuning_or_default(a->tuning).gen_window;
        p.x_host = 0;
        {
            cudaPointerAttributes at;
            if (cudaPointerGetAttributes(&at, a->x) == cudaSuccess) p.x_host = at.type == cudaMemoryTypeHost;
            else cudaGetLastError();
        }
        const int req = look;
        if (look < 0) look = (p.x_host && req != -4) ? 16 : 0;
        p.win = win_applicable(p.B, p.L, (int)p.nv, look) ? look : 0;
        // host-mapped signals of any other shape (auto only): window gather as
        // its own kernel into a (B, L, 16|32) buffer, ordinary FFT from it
        p.wing = req < 0 && p.x_host && !p.win && p.L >= 128 && p.nv <= 32;
        p.off_win = p.win ? take(win_ring_bytes(p.win)) : (p.wing ? take(win_gather_bytes(p.B, p.L, (int)p.nv)) : 0);
        p.off_winf = p.win ? take(win_flag_bytes(p.B)) : 0;
    }
    p.total = o;
    return SFDT_OK;
}

}  // namespace sfdt

using namespace sfdt;

extern "C" int sfdt_general_caps(const sfdt_general_args *a, int64_t *entry_cap) {
    GenPlan p;
    int rc = make_gen_plan(a, p);
    if (rc) return rc;
    if (entry_cap) *entry_cap = p.B * p.L * a->a_max;
    return SFDT_OK;
}

extern "C" size_t sfdt_general_workspace_bytes(const sfdt_general_args *a) {
    GenPlan p;
    if (make_gen_plan(a, p)) return 0;
    return p.total;
}

extern "C" int sfdt_general_solve(sfdt_general_args *a, void *ws, size_t ws_bytes, sfdt_stream_t stream_) {
    GenPlan p;
    int rc = make_gen_plan(a, p);
    if (rc) return rc;
    if (!ws || ws_bytes < p.total) return SFDT_EWORKSPACE;
    int64_t ecap;
    sfdt_general_caps(a, &ecap);
    if (a->entry_cap < ecap) return SFDT_ECAPACITY;
    if (!a->shifts || !a->base_phi || !a->twiddles) return SFDT_EINVAL;
    cudaStream_t stream = (cudaStream_t)stream_;
    const sfdt_tuning tn = tuning_or_default(a->tuning);
    char *w = (char *)ws;
    cx *V = (cx *)(w + p.off_V);
    double *sv = a->singular_values ? a->singular_values : (double *)(w + p.off_sv);
    double *part = (double *)(w + p.off_part);
    int32_t *votes = a->votes ? a->votes : (int32_t *)(w + p.off_votes);
    uint8_t *nent = (uint8_t *)(w + p.off_nent);
    int64_t *sloc = (int64_t *)(w + p.off_sloc);
    cx *sval = (cx *)(w + p.off_sval);
    int64_t *wl = (int64_t *)(w + p.off_wl);
    unsigned long long *wlc = (unsigned long long *)(w + p.off_cnt);
    cx *fft_scratch = p.off_fft ? (cx *)(w + p.off_fft) : nullptr;
    const int is_c64 = a->x_dtype == SFDT_C64;
    int launches = 0;

    GenParams gp;
    gp.n = p.n;
    gp.d = p.d;
    gp.L = p.L;
    gp.k = a->k;
    gp.a_max = a->a_max;
    gp.r_eff = a->r_eff;
    gp.keep = a->keep_per_collision;
    gp.prune = a->prune;
    gp.S = p.S;
    gp.nv = (int)p.nv;
    gp.zvr = a->zero_vote_rtol;
    gp.shifts = a->shifts;
    gp.shift_stride = a->shift_stride;
    gp.base_phi = (const cx *)a->base_phi;
    gp.phi_stride = a->phi_stride;

    int64_t *vsh = (int64_t *)(w + p.off_vsh);
    int32_t *vslot = (int32_t *)(w + p.off_vslot);
    int32_t *nview = (int32_t *)(w + p.off_nview);
    {
        const int dedup = tn.gen_dedup != 0;
        k_gen_vslot<<<(unsigned)((p.B + 127) / 128), 128, 0, stream>>>(gp, p.B, dedup, vsh, vslot, nview);
        SFDT_CHECK_LAUNCH();
        launches++;
    }
    gp.vslot = vslot;

    // 1. consecutive + random-shift views (general.py:288-294)
    ViewSrc src = consecutive_views(a->x, is_c64, p.n, p.d, 0, p.S);
    src.nshift = (int)p.nv;
    src.dyn_off = vsh;
    src.dyn_first = p.S;
    src.dyn_stride = a->r_eff;
    src.nview = nview;
    if (a->ev_fft_begin) cudaEventRecord((cudaEvent_t)a->ev_fft_begin, stream);
    if (p.wing)
        rc = launch_fft_from_window(src, p.B, p.L, a->twiddles, V, (int)p.nv, p.L, stream, (cx *)(w + p.off_win),
                                    fft_scratch, tn.gen_window == -2, tn.fft_split);
    else if (p.win)
        rc = launch_fft_win16(src, p.B, a->twiddles, V, (int)p.nv, p.L, stream, p.win, (cx *)(w + p.off_win),
                              (int *)(w + p.off_winf), tn.gen_window == -2 ? 1 : (tn.gen_window == -3 ? 0 : !p.x_host));
    else
        rc = launch_fft_views(src, p.B, p.L, a->twiddles, V, (int)p.nv, p.L, stream, fft_scratch, 1, nullptr,
                              nullptr, tn.fft_split);
    if (rc) return rc;
    if (a->ev_fft_end) cudaEventRecord((cudaEvent_t)a->ev_fft_end, stream);
    launches += fft_view_launches(p.L, tn.fft_split) + (p.wing ? 1 : 0);

    // 2. collision vote (general.py:131-155)
    {
        const dim3 g((unsigned)p.nparts, (unsigned)p.B);
        int64_t *fix = (int64_t *)(w + p.off_fix);
        unsigned long long *nfix = wlc + 2;
        switch (a->a_max) {
        case 1: k_gen_svd<1><<<g, 128, 0, stream>>>(V, gp, sv, part, fix, nfix, 0); break;
        case 2: k_gen_svd<2><<<g, 128, 0, stream>>>(V, gp, sv, part, fix, nfix, 0); break;
        case 3: {
            const int closed = tn.gen_svd_closed != 0;   // 0: the Jacobi for every bin
            cudaMemsetAsync(nfix, 0, 8, stream);
            k_gen_svd<3><<<g, 128, 0, stream>>>(V, gp, sv, part, fix, nfix, closed);
            SFDT_CHECK_LAUNCH();
            k_gen_svd_fix<<<wl_grid(p.B * p.L, 128, one_wave(k_gen_svd_fix, 128)), 128, 0, stream>>>(
                V, gp, sv, fix, nfix);
            launches++;
            break;
        }
        default: k_gen_svd<4><<<g, 128, 0, stream>>>(V, gp, sv, part, fix, nfix, 0); break;
        }
    }
    SFDT_CHECK_LAUNCH();
    cudaMemsetAsync(wlc, 0, 8, stream);
    if (p.L * a->a_max > VOTE_BIG) {
        const int64_t M = p.L * a->a_max;
        const int64_t nch = (M + VCH - 1) / VCH, nchL = (p.L + VCH - 1) / VCH;
        VSel *vs = (VSel *)(w + p.off_vsel);
        unsigned int *ghist = (unsigned int *)(w + p.off_ghist);
        long long *eqc = (long long *)(w + p.off_eqc);
        cudaMemsetAsync(ghist, 0, size_t(p.B) * 256 * 4, stream);
        cudaMemsetAsync(votes, 0, size_t(p.B) * p.L * 4, stream);
        k_vsel_init<<<(unsigned)p.B, 32, 0, stream>>>(part, (int)p.nparts, gp, p.B, vs, a->stats);
        // two full 8-bit passes, then the candidates sharing the 16-bit
        // prefix are compacted and one CTA per signal finishes the select
        for (int shift = 56; shift >= 48; shift -= 8) {
            k_vsel_hist<<<(unsigned)(p.B * nch), 256, 0, stream>>>(sv, gp, nch, shift, vs, ghist);
            k_vsel_pick<<<(unsigned)p.B, 32, 0, stream>>>(p.B, shift, vs, ghist);
        }
        unsigned long long *cand = (unsigned long long *)(w + p.off_cand);
        k_vsel_compact<<<(unsigned)(p.B * nch), 256, 0, stream>>>(sv, gp, nch, vs, cand);
        k_vsel_select<<<(unsigned)p.B, 1024, 0, stream>>>(sv, gp, vs, cand);
        k_vsel_eqcount<<<(unsigned)(p.B * nch), 256, 0, stream>>>(sv, gp, nch, vs, eqc);
        k_vsel_vote<<<(unsigned)(p.B * nch), 256, 0, stream>>>(sv, gp, nch, vs, eqc, votes);
        k_vsel_fin<<<(unsigned)(p.B * nchL), 256, 0, stream>>>(sv, gp, nchL, vs, votes, a->stats, wl, wlc);
        launches += 1 + 4 + 2 + 3 - 1;   // the -1: k_gen_vote is counted below
    } else {
        const int64_t M = p.L * a->a_max;
        const size_t smem = M <= VOTE_SMEM_KEYS ? size_t(M) * 8 : 0;
        cudaFuncSetAttribute(k_gen_vote, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k_gen_vote<<<(unsigned)p.B, 1024, smem, stream>>>(sv, part, (int)p.nparts, gp, votes, a->stats,
                                                          wl, wlc);
    }
    SFDT_CHECK_LAUNCH();
    if (a->ev_vote_end) cudaEventRecord((cudaEvent_t)a->ev_vote_end, stream);
    // 3-4. pruning + subspace pursuit per voted bin
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaMemsetAsync(nent, 0, size_t(p.B) * p.L, stream);
    int32_t *mf_top = (int32_t *)(w + p.off_mf);
    bool mf_small_done = false;
    if (a->prune && p.d <= 32 && tn.gen_mf_small) {
        const int64_t nch = (p.L + MF_LIST - 1) / MF_LIST;
        const unsigned grid = (unsigned)(p.B * nch);
        int G = (int)p.d;
        while (G < a->r_eff) G <<= 1;
        mf_small_done = true;
        switch (a->r_eff * 100 + G) {   // the (r_eff, d) pairs of a_max = 1..4
#define SFDT_MFS(R, G_)                                                                          \
    case R * 100 + G_: k_gen_mf_small<R, G_><<<grid, 256, 0, stream>>>(V, gp, votes, mf_top, nch); break;
            SFDT_MFS(1, 1) SFDT_MFS(2, 2) SFDT_MFS(3, 4) SFDT_MFS(4, 4) SFDT_MFS(6, 8) SFDT_MFS(8, 8)
            SFDT_MFS(9, 16) SFDT_MFS(12, 16) SFDT_MFS(9, 32) SFDT_MFS(12, 32)
#undef SFDT_MFS
        default: mf_small_done = false; break;   // no instance: the warp-per-bin form
        }
        if (mf_small_done) {
            SFDT_CHECK_LAUNCH();
            launches++;
        }
    }
    if (a->prune && !mf_small_done) {
        // bins per CTA: MF_LIST, fewer when that leaves < 2 CTAs per SM
        // (few long-view signals: config 5 general K = 64 had 64 CTAs)
        int mfl = MF_LIST;
        if (tn.gen_mf_list) mfl = tn.gen_mf_list;   // validated by make_gen_plan
        else
            while (mfl > 256 && p.B * ((p.L + mfl - 1) / mfl) < 2 * (int64_t)sms) mfl >>= 1;
        const int64_t nch = (p.L + mfl - 1) / mfl;
        const size_t phi_bytes = size_t(a->r_eff) * p.d * 16;
        const int stage = phi_bytes <= MF_SMEM_MAX;
        const size_t smem = stage ? phi_bytes : 0;
        switch (a->r_eff) {
#define SFDT_MF(R)                                                                                 \
    case R:                                                                                        \
        if (stage) {                                                                               \
            cudaFuncSetAttribute(k_gen_mf<R, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,   \
                                 (int)smem);                                                       \
            k_gen_mf<R, true><<<(unsigned)(p.B * nch), 256, smem, stream>>>(V, gp, votes, mf_top, nch, mfl); \
        } else {                                                                                   \
            k_gen_mf<R, false><<<(unsigned)(p.B * nch), 256, 0, stream>>>(V, gp, votes, mf_top, nch, mfl); \
        }                                                                                          \
        break;
            SFDT_MF(1) SFDT_MF(2) SFDT_MF(3) SFDT_MF(4) SFDT_MF(5) SFDT_MF(6)
            SFDT_MF(7) SFDT_MF(8) SFDT_MF(9) SFDT_MF(10) SFDT_MF(11) SFDT_MF(12)
#undef SFDT_MF
        default: return SFDT_EINVAL;
        }
        SFDT_CHECK_LAUNCH();
        launches++;
    }
    int32_t *colsb = (int32_t *)(w + p.off_cols);
    int8_t *ncolsb = (int8_t *)(w + p.off_ncols);
    // voted bins per signal <= min(K, L): bounds every worklist below
    const int64_t max_voted = p.B * (a->k < p.L ? (int64_t)a->k : p.L);
    const int sp1 = sp1_r(a->r_eff);
    // Bins pursued over all d columns (prune off, or count >= d): one warp
    // per bin while the bins are few -- at most K voted bins per signal, and
    // up to ~224 warps per SM the warp form's shorter chains win (measured
    // at N=2^22, B=64, d=2048/512/128: 7.33 -> 1.33 ms, 3.64 -> 2.19 ms,
    // 2.75 -> 5.53 ms); beyond that, thread per bin (32 bins per warp in
    // lockstep) keeps the FP64 pipe busier than 32 lanes on one bin's
    // redundant least squares.  tuning.gen_warp = 0 / 1 forces either form.
    const bool all_d = !a->prune || p.d <= 2 * (int64_t)a->keep_per_collision * a->a_max;
    const bool few = (int64_t)a->k * p.B <= 224 * (int64_t)sms;
    const int warp_all = all_d && (tn.gen_warp >= 0 ? tn.gen_warp == 1 : few);
    int64_t *hl = (int64_t *)(w + p.off_hl);
    unsigned long long *hlc = wlc + 1;
    cudaMemsetAsync(hlc, 0, 8, stream);
    // wlc[3]: k_gen_bins' take counter, [4]: the a >= split_a count
    cudaMemsetAsync(wlc + 3, 0, 16, stream);
    // heavy bins with a >= split_a dealt first (tuning.gen_split_a; 0: list order)
    const int split_a = tn.gen_split_a;
    // the multi-collision pursuit (k_gen_bins) forks onto the caller's aux
    // stream, when given, beside the single-collision pursuit (k_gen_sp1)
    cudaStream_t side = (cudaStream_t)a->aux_stream;
    if (side == stream) side = nullptr;
    const int hflags = sp1 | (warp_all ? 2 : 0);
    // four lanes per bin when d splits into >= 2 recurrence segments and the
    // bins are few (one lane per bin would leave most of the GPU idle)
    const bool lanes4 = a->prune && p.d >= 1024 && (p.d & 511) == 0 &&
                        (tn.gen_prune_lanes ? tn.gen_prune_lanes == 4 : max_voted <= 64 * (int64_t)sms);
    const unsigned prune_grid = lanes4 ? wl_grid(4 * max_voted, 128, one_wave(k_gen_prune<4>, 128))
                                       : wl_grid(max_voted, 128, one_wave(k_gen_prune<1>, 128));
    if (lanes4)
        k_gen_prune<4><<<prune_grid, 128, 0, stream>>>(V, gp, votes, wl, wlc, mf_top, colsb, ncolsb, hflags, hl,
                                                       hlc, max_voted, wlc + 4, split_a);
    else
        k_gen_prune<1><<<prune_grid, 128, 0, stream>>>(V, gp, votes, wl, wlc, mf_top, colsb, ncolsb, hflags, hl,
                                                       hlc, max_voted, wlc + 4, split_a);
    SFDT_CHECK_LAUNCH();
    if (a->ev_prune_end) cudaEventRecord((cudaEvent_t)a->ev_prune_end, stream);
    // heavy bins (k_gen_bins) fork onto the side stream; the bins of the
    // two pursuits are disjoint (k_gen_prune routes each to one list) and
    // their shared counters are atomics
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    if (side) {
        if (cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming) != cudaSuccess)
            return SFDT_ECUDA;
        cudaEventRecord(ev_fork, stream);
        cudaStreamWaitEvent(side, ev_fork, 0);
    }
    cudaStream_t bstream = side ? side : stream;
    // bins per warp dealt statically in k_gen_bins (tuning.gen_deal; 1: one
    // per warp, 0: the take counter)
    const int deal_max = tn.gen_deal;
    auto launch_bins = [&](cudaStream_t st, const unsigned long long *lo_count, unsigned long long *take,
                           const unsigned long long *hi_count) {
        // one wave; heavy bins dealt over its warps (k_gen_bins)
        switch (a->r_eff) {
#define SFDT_BINS(R)                                                                                    \
    case R:                                                                                             \
        k_gen_bins<R><<<wl_grid(32 * max_voted, 128, one_wave(k_gen_bins<R>, 128)), 128, 0, st>>>(      \
            V, gp, votes, wl, hl, lo_count, colsb, ncolsb, nent, sloc, sval, a->stats, take, deal_max,   \
            hi_count, max_voted);                                                                       \
        break;
            SFDT_BINS(6) SFDT_BINS(8) SFDT_BINS(9) SFDT_BINS(12)
        default:
            SFDT_BINS(0)
#undef SFDT_BINS
        }
    };
    launch_bins(bstream, hlc, wlc + 3, wlc + 4);
    SFDT_CHECK_LAUNCH();
    launches++;
    if (sp1) {
        switch (a->r_eff) {
#define SFDT_SP1(R)                                                                                     \
    case R:                                                                                             \
        k_gen_sp1<R><<<wl_grid(max_voted, 128, one_wave(k_gen_sp1<R>, 128)), 128, 0, stream>>>(        \
            V, gp, votes, wl, wlc, colsb, ncolsb, nent, sloc, sval, a->stats);                          \
        break;
            SFDT_SP1(1) SFDT_SP1(2) SFDT_SP1(3) SFDT_SP1(4) SFDT_SP1(6) SFDT_SP1(8) SFDT_SP1(9) SFDT_SP1(12)
#undef SFDT_SP1
        default: break;
        }
        SFDT_CHECK_LAUNCH();
        launches++;
    }
    if (warp_all) {
        k_gen_bins_warp<<<wl_grid(max_voted, 8, one_wave(k_gen_bins_warp, 256)), 256, 0, stream>>>(
            V, gp, votes, wl, wlc, ncolsb, nent, sloc, sval, a->stats);
        SFDT_CHECK_LAUNCH();
        launches++;
    }
    if (side) {
        cudaEventRecord(ev_join, side);
        cudaStreamWaitEvent(stream, ev_join, 0);
        cudaEventDestroy(ev_fork);   // released once the pending work completes
        cudaEventDestroy(ev_join);
    }
    if (a->ev_pursuit_end) cudaEventRecord((cudaEvent_t)a->ev_pursuit_end, stream);
    const int64_t nseg = (p.L + GEN_SEG - 1) / GEN_SEG;
    long long *segcnt = (long long *)(w + p.off_seg);
    k_gen_count<<<(unsigned)(p.B * nseg), 256, 0, stream>>>(votes, nent, p.L, nseg, segcnt);
    k_gen_fin<<<(unsigned)((p.B + 255) / 256), 256, 0, stream>>>(segcnt, p.B, nseg, a->stats);
    k_gen_scan<<<1, 1024, 0, stream>>>(a->stats, p.B, a->entry_offsets);
    k_gen_emit<<<(unsigned)(p.B * nseg), 256, 0, stream>>>(votes, nent, sloc, sval, p.L, a->a_max, a->stats,
                                                           a->entry_offsets, a->locs, (cx *)a->vals, nseg,
                                                           segcnt);
    SFDT_CHECK_LAUNCH();
    launches += 7;
    a->kernel_launches = launches;
    return SFDT_OK;
}

extern "C" size_t sfdt_estimate_collisions_workspace_bytes(int64_t nb) {
    if (nb < 0) return 0;
    const int64_t nparts = (nb + 127) / 128;
    return size_t(nparts) * 8 + size_t(nb) * 8 + 64 + size_t(SFDT_GS_PER_SIGNAL) * 8 + 1024;
}

extern "C" int sfdt_estimate_collisions(const double *syn, int64_t nb, int64_t ld, int64_t k, int a_max,
                                        int64_t d, double zero_vote_rtol, int32_t *votes, double *sv,
                                        void *ws, size_t ws_bytes, sfdt_stream_t stream_) {
    if (a_max < 1 || a_max > 4 || ld < 2 * a_max - 1 || nb < 0 || k < 1 || d < 1) return SFDT_EINVAL;
    if (nb == 0) return SFDT_OK;
    if (!ws || ws_bytes < sfdt_estimate_collisions_workspace_bytes(nb)) return SFDT_EWORKSPACE;
    cudaStream_t stream = (cudaStream_t)stream_;
    const int64_t nparts = (nb + 127) / 128;
    char *w = (char *)ws;
    double *part = (double *)w;
    int64_t *wl = (int64_t *)(w + ((nparts * 8 + 255) & ~int64_t(255)));
    unsigned long long *wlc = (unsigned long long *)((char *)wl + nb * 8);
    int64_t *stats = (int64_t *)((char *)wlc + 64);
    // the reference runs the Jacobi with its 1e-17 threshold here: this is
    // the kernel-level mirror of estimate_collisions
    switch (a_max) {
    case 1: k_rows_svd<1><<<(unsigned)nparts, 128, 0, stream>>>((const cx *)syn, nb, ld, sv, part, 1e-17); break;
    case 2: k_rows_svd<2><<<(unsigned)nparts, 128, 0, stream>>>((const cx *)syn, nb, ld, sv, part, 1e-17); break;
    case 3: k_rows_svd<3><<<(unsigned)nparts, 128, 0, stream>>>((const cx *)syn, nb, ld, sv, part, 1e-17); break;
    default: k_rows_svd<4><<<(unsigned)nparts, 128, 0, stream>>>((const cx *)syn, nb, ld, sv, part, 1e-17); break;
    }
    SFDT_CHECK_LAUNCH();
    GenParams gp;
    gp.n = nb * d;
    gp.d = d;
    gp.L = nb;
    gp.k = k;
    gp.a_max = a_max;
    gp.r_eff = 1;
    gp.keep = 1;
    gp.prune = 0;
    gp.S = (int)ld;   // the RMS guard averages over every given column
    gp.nv = (int)ld;
    gp.zvr = zero_vote_rtol;
    gp.shifts = nullptr;
    gp.shift_stride = 0;
    gp.base_phi = nullptr;
    gp.phi_stride = 0;
    gp.vslot = nullptr;
    cudaMemsetAsync(wlc, 0, 8, stream);
    {
        const int64_t M = nb * a_max;
        const size_t smem = M <= VOTE_SMEM_KEYS ? size_t(M) * 8 : 0;
        cudaFuncSetAttribute(k_gen_vote, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k_gen_vote<<<1, 1024, smem, stream>>>(sv, part, (int)nparts, gp, votes, stats, wl, wlc);
    }
    SFDT_CHECK_LAUNCH();
    return SFDT_OK;
}

// ------------------------------------------------ drop-in library mirrors
// general.py:109-121 sensing_matrix, :184-221 prune_columns and :224-269
// subspace_pursuit as batched device calls (one thread per bin / problem),
// built from the same device functions as the fused solver kernels.
namespace {

constexpr int PRUNE_MIRROR_MAX = 64;   // keep_per_collision * a supported by the mirror

// Phi[j, t] = exp(2i pi loc_t shifts_j / n), loc_t = (k + col_t * n/d) mod n,
// the phase evaluated as numpy does (2j*pi*outer(shifts, locs)/n)
__device__ __forceinline__ cx sensing_entry(int64_t shift, int64_t loc, int64_t n) {
    return gexp(mk(0.0, DMUL(TWO_PI, (double)(shift * loc)) / (double)n));
}

__global__ void k_sensing_matrix(int64_t n, int64_t d, int64_t k, const int64_t *__restrict__ shifts, int r,
                                  const int64_t *__restrict__ cols, int64_t ncols, cx *__restrict__ out) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= r * ncols) return;
    const int64_t j = i / ncols, c = i - j * ncols;
    const int64_t col = cols ? cols[c] : c;
    const int64_t loc = pmod(k + col * (n / d), n);
    out[i] = sensing_entry(shifts[j], loc, n);
}

// _correlation_keep (general.py:158-165): the `cnt` columns of largest
// |Phi^H y| (stable: ties keep the lower column), returned sorted
__device__ int correlation_keep(const cx *y, const int64_t *sh, int r, int64_t kb, int64_t n, int64_t d, int cnt,
                                int *out) {
    double sc[PRUNE_MIRROR_MAX];
    int id[PRUNE_MIRROR_MAX], nk = 0;
    const int64_t m = n / d;
    for (int64_t t = 0; t < d; t++) {
        const int64_t loc = pmod(kb + t * m, n);
        cx acc = mk(0.0, 0.0);
        for (int j = 0; j < r; j++) acc = cadd(acc, nmul(cconj(sensing_entry(sh[j], loc, n)), y[j]));
        topk_insert(sc, id, nk, cnt, cabs_(acc), (int)t);
    }
    for (int i = 0; i < nk; i++) out[i] = id[i];
    sort_ints(out, nk);
    return nk;
}

// prune_columns for one bin per thread.  nkept[b] = -1: every column kept
// (all fits singular and no fallback) -- np.arange(d).
__global__ void k_prune_columns(const cx *__restrict__ m, int64_t nb, int64_t ld, const int64_t *__restrict__ kbin,
                                int a, int a_max, int64_t n, int64_t d, int keep, const cx *__restrict__ y,
                                int64_t ldy, const int64_t *__restrict__ shifts, int r, int augment,
                                int64_t *__restrict__ kept, int32_t *__restrict__ nkept, int64_t cap) {
    const int64_t b = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (b >= nb) return;
    const int64_t kb = kbin[b];
    const int cnt = (int)((int64_t)keep * a < d ? (int64_t)keep * a : d);
    cx syn[8], yy[GEN_MAX_R], c[4];
    for (int l = 0; l < 2 * a_max; l++) syn[l] = m[b * ld + l];
    if (y)
        for (int j = 0; j < r; j++) yy[j] = y[b * ldy + j];
    // _fit_locator (general.py:168-181): highest non-singular order
    int order = 0;
    for (int o2 = a_max; o2 >= 1; o2--) {
        double scale = 0.0;
        for (int l = 0; l < 2 * o2; l++) scale = nanmax2(scale, cabs_(syn[l]));
        scale = nanmax2(scale, TINY);
        const cx cd = hankel_solve1(syn, o2, c);
        if (cabs_(cd) > DMUL(SINGULARITY_RTOL, powa(scale, o2))) {
            order = o2;
            break;
        }
    }
    int cols[PRUNE_MIRROR_MAX + 4];
    int nc = 0;
    if (order == 0) {
        if (!y) {
            nkept[b] = -1;
            return;
        }
        nc = correlation_keep(yy, shifts, r, kb, n, d, cnt, cols);
    } else {
        // prune_eval (_core.pyx:319-346): recurrence z *= wd re-seeded every
        // 512 candidates, Horner from the leading coefficient; keep the cnt
        // smallest (argpartition then sort: ties to the lower column)
        double ks[PRUNE_MIRROR_MAX];
        int kp[PRUNE_MIRROR_MAX], nk = 0;
        const cx base = gexp(mk(0.0, DMUL(TWO_PI, (double)kb) / (double)n));
        const cx wd = gexp(mk(0.0, TWO_PI / (double)d));
        cx zt = base;
        for (int64_t t = 0; t < d; t++) {
            cx acc = mk(1.0, 0.0);
            for (int j = order - 1; j >= 0; j--) acc = cadd(gmul(acc, zt), c[j]);
            botk_insert(ks, kp, nk, cnt, cabs_(acc), (int)t);
            zt = ((t & 511) == 511) ? gmul(base, gexp(mk(0.0, DMUL(TWO_PI, (double)(t + 1)) / (double)d)))
                                    : gmul(zt, wd);
        }
        for (int i = 0; i < nk; i++) cols[i] = kp[i];
        sort_ints(cols, nk);
        nc = nk;
        if (augment && y && cnt < d) {
            int top[4];
            const int nt = correlation_keep(yy, shifts, r, kb, n, d, a < d ? a : (int)d, top);
            int merged[PRUNE_MIRROR_MAX + 4];
            nc = union_sorted(cols, nk, top, nt, merged);
            for (int i = 0; i < nc; i++) cols[i] = merged[i];
        }
    }
    for (int i = 0; i < nc && i < cap; i++) kept[b * cap + i] = cols[i];
    nkept[b] = nc;
}

// subspace_pursuit on an explicit phi (rows x cols, row-major) per problem:
// subspace_pursuit_dev with unit phases (1 * phi is exact), every column
__global__ void k_subspace_pursuit(const cx *__restrict__ y, const cx *__restrict__ phi, int64_t nb, int rows,
                                   int cols, int a, int max_iter, cx *__restrict__ coef,
                                   int32_t *__restrict__ rankdef) {
    const int64_t b = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (b >= nb) return;
    cx yy[GEN_MAX_R], ones[GEN_MAX_R];
    for (int j = 0; j < rows; j++) {
        yy[j] = y[b * rows + j];
        ones[j] = mk(1.0, 0.0);
    }
    SPOut o;
    subspace_pursuit_dev<0>(yy, ones, phi + b * (int64_t)rows * cols, cols, rows, nullptr, cols, true, a, o, 0, 1,
                            max_iter);
    for (int c2 = 0; c2 < cols; c2++) coef[b * cols + c2] = mk(0.0, 0.0);
    for (int i = 0; i < o.nsup; i++) coef[b * cols + o.sup[i]] = o.coef[i];
    if (rankdef) rankdef[b] = o.rankdef;
}

}  // namespace

extern "C" int sfdt_sensing_matrix(int64_t n, int64_t d, int64_t k, const int64_t *shifts, int r,
                                   const int64_t *columns, int64_t ncols, double *out, sfdt_stream_t stream) {
    if (n < 1 || (n & (n - 1)) || d < 1 || n % d || r < 0 || ncols < 0 || (r && !shifts)) return SFDT_EINVAL;
    if (!r || !ncols) return SFDT_OK;
    const int64_t total = (int64_t)r * ncols;
    k_sensing_matrix<<<(unsigned)((total + 255) / 256), 256, 0, (cudaStream_t)stream>>>(n, d, k, shifts, r, columns,
                                                                                        ncols, (cx *)out);
    SFDT_CHECK_LAUNCH();
    return SFDT_OK;
}

extern "C" int sfdt_prune_columns(const double *m, int64_t nb, int64_t ld, const int64_t *k, int a, int a_max,
                                  int64_t n, int64_t d, int keep, const double *y, int64_t ldy,
                                  const int64_t *shifts, int r, int augment, int64_t *kept, int32_t *nkept,
                                  int64_t cap, sfdt_stream_t stream) {
    if (nb < 0 || a < 1 || a_max < 1 || a_max > 4 || ld < 2 * a_max || n < 1 || (n & (n - 1)) || d < 1 ||
        n % d || keep < 1 || (int64_t)keep * a > PRUNE_MIRROR_MAX || (y && (r < 1 || r > GEN_MAX_R || !shifts)) ||
        cap < (int64_t)keep * a + a || !kept || !nkept)
        return SFDT_EINVAL;
    if (nb == 0) return SFDT_OK;
    k_prune_columns<<<(unsigned)((nb + 63) / 64), 64, 0, (cudaStream_t)stream>>>(
        (const cx *)m, nb, ld, k, a, a_max, n, d, keep, (const cx *)y, ldy, shifts, r, augment, kept, nkept, cap);
    SFDT_CHECK_LAUNCH();
    return SFDT_OK;
}

extern "C" int sfdt_subspace_pursuit(const double *y, const double *phi, int64_t nb, int rows, int cols, int a,
                                     int max_iter, double *coef, int32_t *rankdef, sfdt_stream_t stream) {
    if (nb < 0 || rows < 1 || rows > GEN_MAX_R || cols < 1 || a < 1 || a > rows || max_iter < 0 ||
        2 * (a < cols ? a : cols) > GEN_MAX_SUP || !y || !phi || !coef)
        return SFDT_EINVAL;
    if (nb == 0) return SFDT_OK;
    k_subspace_pursuit<<<(unsigned)((nb + 63) / 64), 64, 0, (cudaStream_t)stream>>>(
        (const cx *)y, (const cx *)phi, nb, rows, cols, a, max_iter, (cx *)coef, rankdef);
    SFDT_CHECK_LAUNCH();
    return SFDT_OK;
}
