// exact.cu -- sm_100a kernels of the exactly-K-sparse path.
//
//   k_stream       one HBM pass over x: per-chunk sum |x|^2 (the rms of
//                  exact.py:176/215) + capture of the 2*a_max-sample shift
//                  window x[d*j .. d*j+S-1] of every d-block (spectral.py:
//                  151-160) into win (B, L, S).  The only kernel that
//                  touches all of x; HBM roofline = 16 B per sample.
//   k_rms          deterministic tree over the chunk partials -> rms, zero
//                  threshold zero_threshold*rms*d.
//   k_fft_views    batched radix-2 DIT FFT of the shifted views, one CTA per
//                  group of views, in shared memory, reproducing the
//                  reference's butterfly arithmetic exactly (fft.cuh).
//   k_decode_noniter  thread-per-bin non-iterative decode (exact.py:184-192)
//   k_iter_pass    one pass l of the iterative solver (exact.py:223-285):
//                  fold, SubFreq, activation, descending-a decode with
//                  retry/deferral, per-bin subtraction of accepted terms.
//   compaction     per-signal scans -> compact (loc, value) lists in the
//                  reference's dict insertion order.
#include "common.cuh"
#include "decode.cuh"
#include "fft.cuh"

namespace sfdt {

// ------------------------------------------------------------- stream pass
// grid (nchunk, B); each CTA streams CH contiguous samples of one signal with
// 16-byte loads (8 in flight per thread), accumulates |x|^2 in a fixed order
// and scatters window samples.  T = double2 (complex128) or float2 (complex64
// storage, upconverted at load).
template <typename T, int THREADS, int UNROLL>
__global__ void __launch_bounds__(THREADS) k_stream(const T *__restrict__ x, int64_t n, int logd,
                                                   int S, int64_t CH, cx *__restrict__ win,
                                                   double *__restrict__ partial) {
    const int64_t b = blockIdx.y;
    const int64_t chunk = blockIdx.x;
    const int64_t d = int64_t(1) << logd;
    const int64_t L = n >> logd;
    const T *xs = x + b * n;
    cx *wb = win + b * L * S;
    double acc = 0.0;
    const int64_t base = chunk * CH;
    for (int64_t off = 0; off < CH; off += int64_t(THREADS) * UNROLL) {
        T v[UNROLL];
#pragma unroll
        for (int u = 0; u < UNROLL; u++) {
            const int64_t e = base + off + int64_t(u) * THREADS + threadIdx.x;
            if constexpr (sizeof(T) == 16) {
                v[u] = (e < base + CH) ? __ldcs(reinterpret_cast<const double2 *>(xs + e)) : T{0, 0};
            } else {
                v[u] = (e < base + CH) ? __ldcs(reinterpret_cast<const float2 *>(xs + e)) : T{0, 0};
            }
        }
#pragma unroll
        for (int u = 0; u < UNROLL; u++) {
            const int64_t e = base + off + int64_t(u) * THREADS + threadIdx.x;
            const double re = (double)v[u].x, im = (double)v[u].y;
            acc = fma(re, re, fma(im, im, acc));
            if (e < base + CH) {
                // window rows j with e = d*j + s (mod n), 0 <= s < S
                int64_t j = e >> logd;
                int64_t s = e & (d - 1);
                while (s < S) {
                    const int64_t jj = j & (L - 1);   // (d*j + s) mod n wraps rows mod L
                    stcx(wb + jj * S + s, mk(re, im));
                    s += d;
                    j -= 1;
                }
            }
        }
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

// rms and threshold per signal: fixed-order pairwise tree over the partials
__global__ void k_rms(const double *__restrict__ partial, int64_t nchunk, int64_t n, double zt,
                      int64_t d, double *__restrict__ rms, double *__restrict__ thr) {
    const int64_t b = blockIdx.x;
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

__global__ void k_scale_thr(const double *__restrict__ rms, int64_t B, double zt, int64_t d,
                            double *__restrict__ out) {
    const int64_t b = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (b < B) out[b] = DMUL(DMUL(zt, rms[b]), (double)d);
}

// --------------------------------------------------- non-iterative decode
// status: 0 inactive, 1..a_max accepted at that a, 0xFF unresolved
__global__ void k_decode_noniter(const cx *__restrict__ V, int64_t B, int64_t L, int S, int a_max,
                                 int64_t n, const double *__restrict__ thr,
                                 uint8_t *__restrict__ status, int64_t *__restrict__ bin_loc,
                                 cx *__restrict__ bin_val) {
    const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= B * L) return;
    const int64_t b = t / L, k = t - b * L;
    cx syn[MAX_SHIFTS];
    const double th = thr[b];
    bool active = false;
    for (int s = 0; s < S; s++) {
        syn[s] = ldcx(V + (b * S + s) * L + k);
        active = active || (cabs_(syn[s]) > th);
    }
    uint8_t st = 0;
    if (active) {
        st = 0xFF;
        Decoded o;
        for (int a = 1; a <= a_max; a++) {
            decode_try(syn, S, a, n, L, k, o);
            if (o.accept) {
                st = (uint8_t)a;
                for (int j = 0; j < a; j++) {
                    bin_loc[t * a_max + j] = o.loc[j];
                    stcx(bin_val + t * a_max + j, o.val[j]);
                }
                break;
            }
        }
    }
    status[t] = st;
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

__global__ void k_iter_pass(IterState st, int64_t B, int64_t L0, int S, int a_max, int l,
                            int64_t n, int64_t m, int fold, const double *__restrict__ thr_base) {
    const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const bool valid = t < B * m;
    const int64_t b = valid ? t / m : 0, k = valid ? t - b * m : 0;
    bool active = false, solved = false, deferred_evt = false;
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
            const int64_t mp = m << (l - p);
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
            (void)mp;
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
        if (active) {
            const int Sl = 2 * l + 2;
            cx syn[MAX_SHIFTS];
            for (int j = 0; j < Sl; j++) syn[j] = Vb[j * L0 + k];
            Decoded o;
            for (int a_try = l + 1; a_try >= 1; a_try--) {
                decode_try(syn, Sl, a_try, n, m, k, o);
                if (o.accept) {
                    solved = true;
                    st.deferred[b * L0 + k] = 0;
                    // duplicate locations overwrite the earlier slot's value
                    uint8_t dupmask = 0;
                    for (int j = 0; j < a_try; j++) {
                        bool found = false;
                        for (int p = 0; p < l && !found; p++) {
                            const int nb = 1 << (l - p);
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
                    for (int j = 0; j < Sl; j++) {
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
        }
    }
    // per-signal counters (warp-aggregated; integer adds are order-free)
    const unsigned mask = 0xffffffffu;
    const int64_t bw = __shfl_sync(mask, b, 0);
    const bool same = __all_sync(mask, !valid || b == bw);
    if (same) {
        const unsigned na = __popc(__ballot_sync(mask, valid && active));
        const unsigned ns = __popc(__ballot_sync(mask, valid && solved));
        const unsigned nd = __popc(__ballot_sync(mask, valid && deferred_evt));
        if ((threadIdx.x & 31) == 0) {
            unsigned long long *c = st.cnt + (bw * 4 + l) * 4;
            if (na) atomicAdd(c + 0, na);
            if (ns) atomicAdd(c + 1, ns);
            if (nd) atomicAdd(c + 2, nd);
        }
    } else if (valid) {
        unsigned long long *c = st.cnt + (b * 4 + l) * 4;
        if (active) atomicAdd(c + 0, 1ull);
        if (solved) atomicAdd(c + 1, 1ull);
        if (deferred_evt) atomicAdd(c + 2, 1ull);
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
// entry offsets; unresolved bins ascending.  One CTA per signal.
template <int THREADS>
__global__ void __launch_bounds__(THREADS) k_noniter_count(const uint8_t *__restrict__ status, int64_t L,
                                                           int a_max, int S, int64_t d,
                                                           int64_t *__restrict__ stats) {
    const int64_t b = blockIdx.x;
    long long cnt[5] = {0, 0, 0, 0, 0};   // entries per a (1..4) and unresolved in [0]
    long long active = 0, tries = 0;
    for (int64_t k = threadIdx.x; k < L; k += THREADS) {
        const uint8_t s = status[b * L + k];
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
    __shared__ long long red[7][THREADS];
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
    if (threadIdx.x == 0) {
        int64_t *st = stats + b * SFDT_ST_PER_SIGNAL;
        const long long nent = red[1][0] + red[2][0] + red[3][0] + red[4][0];
        st[SFDT_ST_NITER] = 1;
        st[SFDT_ST_FULL_SUCCESS] = red[0][0] == 0;
        st[SFDT_ST_NENTRIES] = nent;
        st[SFDT_ST_NUNRESOLVED] = red[0][0];
        st[SFDT_ST_NDUP] = 0;
        st[SFDT_ST_SYNDROMES] = red[6][0] * S;
        st[SFDT_ST_FFT_SAMPLES] = int64_t(S) * L;
        int64_t *it = st + SFDT_ST_ITER0;
        it[0] = d;
        it[1] = red[5][0];                 // attempted
        it[2] = red[5][0] - red[0][0];     // solved
        it[3] = red[0][0];                 // deferred
        it[4] = red[6][0] * S;             // syndromes
        it[5] = int64_t(S) * L;            // fft samples
        // per-a entry counts for the emit pass
        st[24] = red[1][0];
        st[25] = red[2][0];
        st[26] = red[3][0];
        st[27] = red[4][0];
    }
}

// exclusive scan of per-signal counts -> offsets (single CTA, B up to any size)
__global__ void k_scan_offsets(const int64_t *__restrict__ stats, int64_t B, int field,
                               int64_t *__restrict__ offsets) {
    __shared__ long long carry;
    __shared__ long long buf[1024];
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int64_t base = 0; base < B; base += 1024) {
        const int64_t i = base + threadIdx.x;
        long long v = (i < B) ? stats[i * SFDT_ST_PER_SIGNAL + field] : 0;
        buf[threadIdx.x] = v;
        __syncthreads();
        for (int s = 1; s < 1024; s <<= 1) {
            long long add = (threadIdx.x >= s) ? buf[threadIdx.x - s] : 0;
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

// emit entries in (a, bin) order and unresolved bins ascending; one CTA per
// signal, block-wide ordered scan per a-class.
template <int THREADS>
__global__ void __launch_bounds__(THREADS) k_noniter_emit(
    const uint8_t *__restrict__ status, const int64_t *__restrict__ bin_loc,
    const cx *__restrict__ bin_val, int64_t L, int a_max, const int64_t *__restrict__ stats,
    const int64_t *__restrict__ eoff, const int64_t *__restrict__ uoff, int64_t *__restrict__ locs,
    cx *__restrict__ vals, int32_t *__restrict__ ubins) {
    const int64_t b = blockIdx.x;
    __shared__ long long buf[THREADS];
    __shared__ long long carry;
    const int64_t *st = stats + b * SFDT_ST_PER_SIGNAL;
    long long class_base = eoff[b];
    for (int cls = 1; cls <= a_max + 1; cls++) {   // cls a_max+1 = unresolved list
        const bool unres = cls == a_max + 1;
        if (threadIdx.x == 0) carry = unres ? uoff[b] : class_base;
        __syncthreads();
        for (int64_t k0 = 0; k0 < L; k0 += THREADS) {
            const int64_t k = k0 + threadIdx.x;
            const uint8_t s = (k < L) ? status[b * L + k] : 0;
            const long long w = unres ? (s == 0xFF) : ((s == cls) ? cls : 0);
            buf[threadIdx.x] = w;
            __syncthreads();
            for (int o = 1; o < THREADS; o <<= 1) {
                long long add = (threadIdx.x >= o) ? buf[threadIdx.x - o] : 0;
                __syncthreads();
                buf[threadIdx.x] += add;
                __syncthreads();
            }
            const long long pos = carry + buf[threadIdx.x] - w;
            if (w) {
                if (unres) {
                    ubins[pos] = (int32_t)k;
                } else {
                    const int64_t t = b * L + k;
                    for (int j = 0; j < cls; j++) {
                        locs[pos + j] = bin_loc[t * a_max + j];
                        stcx(vals + pos + j, bin_val[t * a_max + j]);
                    }
                }
            }
            __syncthreads();
            if (threadIdx.x == THREADS - 1) carry += buf[THREADS - 1];
            __syncthreads();
        }
        if (!unres) class_base += st[24 + cls - 1];
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
        o[SFDT_ST_NITER] = npass;
        o[SFDT_ST_NENTRIES] = red[0][0];
        o[SFDT_ST_NDUP] = red[1][0];
        o[SFDT_ST_NUNRESOLVED] = ndef[b];
        o[SFDT_ST_SYNDROMES] = syn;
        o[SFDT_ST_FFT_SAMPLES] = fft;
        o[SFDT_ST_FULL_SUCCESS] = (ndef[b] == 0) && (resid[b] <= thr_last[b]);
    }
}

template <int THREADS>
__global__ void __launch_bounds__(THREADS) k_iter_emit(
    const IterState st, int64_t L0, int a_max, int npass, const PassInfo pi,
    int64_t m_final, const int64_t *__restrict__ eoff, const int64_t *__restrict__ uoff,
    const int64_t *__restrict__ doff, int64_t *__restrict__ locs, cx *__restrict__ vals,
    int32_t *__restrict__ ubins, int64_t *__restrict__ dups) {
    const int64_t b = blockIdx.x;
    __shared__ long long bufe[THREADS], bufd[THREADS];
    __shared__ long long carry_e, carry_d;
    if (threadIdx.x == 0) {
        carry_e = eoff[b];
        carry_d = doff ? doff[b] : 0;
    }
    __syncthreads();
    for (int p = 0; p < npass; p++) {
        const int64_t m = pi.m[p];
        for (int a = p + 1; a >= 1; a--) {
            for (int64_t k0 = 0; k0 < m; k0 += THREADS) {
                const int64_t k = k0 + threadIdx.x;
                int64_t si = -1;
                long long we = 0, wd = 0;
                uint8_t dm = 0;
                if (k < m) {
                    si = slot_index(b, p, k, L0);
                    if (st.slot_a[si] == a) {
                        dm = st.slot_dupmask[si];
                        wd = __popc(dm);
                        we = a - wd;
                    }
                }
                bufe[threadIdx.x] = we;
                bufd[threadIdx.x] = wd;
                __syncthreads();
                for (int o = 1; o < THREADS; o <<= 1) {
                    long long ae = (threadIdx.x >= o) ? bufe[threadIdx.x - o] : 0;
                    long long ad = (threadIdx.x >= o) ? bufd[threadIdx.x - o] : 0;
                    __syncthreads();
                    bufe[threadIdx.x] += ae;
                    bufd[threadIdx.x] += ad;
                    __syncthreads();
                }
                long long pe = carry_e + bufe[threadIdx.x] - we;
                long long pd = carry_d + bufd[threadIdx.x] - wd;
                if (we || wd) {
                    for (int j = 0; j < a; j++) {
                        const int64_t loc = st.slot_loc[si * a_max + j];
                        if (dm & (1u << j)) {
                            if (dups) dups[pd] = loc;
                            pd++;
                        } else {
                            locs[pe] = loc;
                            stcx(vals + pe, st.slot_val[si * a_max + j]);
                            pe++;
                        }
                    }
                }
                __syncthreads();
                if (threadIdx.x == THREADS - 1) {
                    carry_e += bufe[THREADS - 1];
                    carry_d += bufd[THREADS - 1];
                }
                __syncthreads();
            }
        }
    }
    // unresolved = deferred bins at the final m, ascending
    if (threadIdx.x == 0) carry_e = uoff[b];
    __syncthreads();
    for (int64_t k0 = 0; k0 < m_final; k0 += THREADS) {
        const int64_t k = k0 + threadIdx.x;
        const long long w = (k < m_final) ? st.deferred[b * L0 + k] : 0;
        bufe[threadIdx.x] = w;
        __syncthreads();
        for (int o = 1; o < THREADS; o <<= 1) {
            long long ae = (threadIdx.x >= o) ? bufe[threadIdx.x - o] : 0;
            __syncthreads();
            bufe[threadIdx.x] += ae;
            __syncthreads();
        }
        if (w) ubins[carry_e + bufe[threadIdx.x] - w] = (int32_t)k;
        __syncthreads();
        if (threadIdx.x == THREADS - 1) carry_e += bufe[THREADS - 1];
        __syncthreads();
    }
}

// ------------------------------------------------------------- host side
static inline size_t align_up(size_t v) { return (v + 255) & ~size_t(255); }

struct ExactPlan {
    int64_t B, n, d, L, S, CH, nchunk, npass;
    int logd;
    size_t off_win, off_V, off_partial, off_thr, off_status, off_bloc, off_bval, off_def,
        off_sloc, off_sval, off_sa, off_sdup, off_cnt, off_resid, off_ndef, off_scratch, off_fft,
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
    p.off_win = take(size_t(p.B) * p.L * p.S * 16);
    p.off_V = take(size_t(p.B) * p.L * p.S * 16);
    p.off_partial = take(size_t(p.B) * p.nchunk * 8);
    p.off_thr = take(size_t(p.B) * 5 * 8);
    if (!a->iterative) {
        p.off_status = take(size_t(p.B) * p.L);
        p.off_bloc = take(size_t(p.B) * p.L * a->a_max * 8);
        p.off_bval = take(size_t(p.B) * p.L * a->a_max * 16);
    } else {
        p.off_def = take(size_t(p.B) * p.L);
        p.off_sloc = take(size_t(p.B) * 4 * p.L * a->a_max * 8);
        p.off_sval = take(size_t(p.B) * 4 * p.L * a->a_max * 16);
        p.off_sa = take(size_t(p.B) * 4 * p.L);
        p.off_sdup = take(size_t(p.B) * 4 * p.L);
        p.off_cnt = take(size_t(p.B) * 16 * 8);
        p.off_resid = take(size_t(p.B) * 8);
        p.off_ndef = take(size_t(p.B) * 8);
    }
    p.off_scratch = take(64 * 8);
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
    char *w = (char *)ws;
    cx *win = (cx *)(w + p.off_win);
    cx *V = (cx *)(w + p.off_V);
    double *partial = (double *)(w + p.off_partial);
    double *thr = (double *)(w + p.off_thr);
    cx *fft_scratch = p.off_fft ? (cx *)(w + p.off_fft) : nullptr;

    int launches = 0;
    // 1. the single pass over x
    {
        if (a->ev_stream_begin) cudaEventRecord((cudaEvent_t)a->ev_stream_begin, stream);
        constexpr int TH = 256, UN = 8;
        dim3 grid((unsigned)p.nchunk, (unsigned)p.B);
        if (a->x_dtype == SFDT_C128)
            k_stream<double2, TH, UN><<<grid, TH, 0, stream>>>((const double2 *)a->x, p.n, p.logd,
                                                               (int)p.S, p.CH, win, partial);
        else
            k_stream<float2, TH, UN><<<grid, TH, 0, stream>>>((const float2 *)a->x, p.n, p.logd,
                                                              (int)p.S, p.CH, win, partial);
        SFDT_CHECK_LAUNCH();
        if (a->ev_stream_end) cudaEventRecord((cudaEvent_t)a->ev_stream_end, stream);
        launches += 1;
        k_rms<<<(unsigned)p.B, 1024, 0, stream>>>(partial, p.nchunk, p.n, a->zero_threshold, p.d,
                                                 a->rms, thr);
        SFDT_CHECK_LAUNCH();
        launches += 1;
    }

    if (!a->iterative) {
        rc = launch_fft_views(win, p.B, p.L, (int)p.S, 1, 0, (int)p.S, p.L, a->twiddles, V,
                              (int)p.S, p.L, stream, fft_scratch);
        if (rc) return rc;
        uint8_t *status = (uint8_t *)(w + p.off_status);
        int64_t *bloc = (int64_t *)(w + p.off_bloc);
        cx *bval = (cx *)(w + p.off_bval);
        const int64_t nbins = p.B * p.L;
        k_decode_noniter<<<(unsigned)((nbins + 127) / 128), 128, 0, stream>>>(
            V, p.B, p.L, (int)p.S, a->a_max, p.n, thr, status, bloc, bval);
        SFDT_CHECK_LAUNCH();
        k_noniter_count<256><<<(unsigned)p.B, 256, 0, stream>>>(status, p.L, a->a_max, (int)p.S,
                                                                p.d, a->stats);
        SFDT_CHECK_LAUNCH();
        k_scan_offsets<<<1, 1024, 0, stream>>>(a->stats, p.B, SFDT_ST_NENTRIES, a->entry_offsets);
        k_scan_offsets<<<1, 1024, 0, stream>>>(a->stats, p.B, SFDT_ST_NUNRESOLVED, a->unres_offsets);
        SFDT_CHECK_LAUNCH();
        k_noniter_emit<256><<<(unsigned)p.B, 256, 0, stream>>>(
            status, bloc, bval, p.L, a->a_max, a->stats, a->entry_offsets, a->unres_offsets,
            a->locs, (cx *)a->vals, a->unres_bins);
        SFDT_CHECK_LAUNCH();
        if (a->dup_offsets) cudaMemsetAsync(a->dup_offsets, 0, sizeof(int64_t) * (p.B + 1), stream);
        launches += (p.L > FFT_SMEM_MAX ? 2 : 1) + 5;
        a->kernel_launches = launches;
        return SFDT_OK;
    }

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
        const int64_t rowstride = d_of[l] / p.d;   // view row j at window row j*rowstride
        rc = launch_fft_views(win, p.B, p.L, (int)p.S, rowstride, 2 * l, 2, m, a->twiddles,
                              V + 2 * l * p.L, (int)p.S, p.L, stream, fft_scratch);
        if (rc) return rc;
        const int fold = (l > 0) && (m != m_of[l - 1]);
        const int64_t nb = p.B * m;
        k_iter_pass<<<(unsigned)((nb + 127) / 128), 128, 0, stream>>>(st, p.B, p.L, (int)p.S, a->a_max,
                                                                      l, p.n, m, fold, thr);
        SFDT_CHECK_LAUNCH();
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
    k_scan_offsets<<<1, 1024, 0, stream>>>(a->stats, p.B, SFDT_ST_NENTRIES, a->entry_offsets);
    k_scan_offsets<<<1, 1024, 0, stream>>>(a->stats, p.B, SFDT_ST_NUNRESOLVED, a->unres_offsets);
    if (a->dup_offsets)
        k_scan_offsets<<<1, 1024, 0, stream>>>(a->stats, p.B, SFDT_ST_NDUP, a->dup_offsets);
    SFDT_CHECK_LAUNCH();
    k_iter_emit<256><<<(unsigned)p.B, 256, 0, stream>>>(st, p.L, a->a_max, (int)p.npass, pi,
                                                        m_final, a->entry_offsets, a->unres_offsets,
                                                        a->dup_offsets ? a->dup_offsets : nullptr,
                                                        a->locs, (cx *)a->vals, a->unres_bins,
                                                        a->dup_locs);
    SFDT_CHECK_LAUNCH();
    launches += (int)p.npass * (1 + 1 + (p.L > FFT_SMEM_MAX ? 2 : 1)) + 1 + 1 + 2 + (a->dup_offsets ? 1 : 0) + 1;
    a->kernel_launches = launches;
    return SFDT_OK;
}
