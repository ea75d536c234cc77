// dropin.cu -- device forms of the reference's per-view and per-bin library
// functions (the drop-in surface around the solvers):
//
//   sfdt_downsample            <- spectral.py:151-160  downsample
//   sfdt_aliased_values        <- spectral.py:163-172  transform_view / aliased_values
//   sfdt_direct_dft            <- spectral.py:110-125  forward_dft_oracle
//   sfdt_decode_bins           <- syndrome.py:69-175   solve_coefficients ->
//                                 roots_closed_form -> solve_values ->
//                                 root_to_location (decode_bin), batched
//   sfdt_poly_residuals        <- syndrome.py:101-106
//   sfdt_reconstruct_syndromes <- syndrome.py:136-144
//
// Same arithmetic as the solver kernels (cx.cuh reproduces gcc / numpy
// complex rounding), one thread per view sample / bin.
#include "common.cuh"
#include "decode.cuh"
#include "fft.cuh"

using namespace sfdt;

namespace {

// out[b, v, j] = x[b, (d*j + shift_v) mod n]
__global__ void k_downsample(const void *__restrict__ x, int is_c64, int64_t B, int64_t n, int64_t d,
                             const int64_t *__restrict__ shifts, int nshift, cx *__restrict__ out) {
    const int64_t L = n / d;
    const int64_t total = B * nshift * L;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
         i += int64_t(gridDim.x) * blockDim.x) {
        const int64_t j = i % L, bv = i / L;
        const int v = (int)(bv % nshift);
        const int64_t b = bv / nshift;
        const int64_t idx = (d * j + shifts[v]) % n;
        if (is_c64) {
            const float2 f = reinterpret_cast<const float2 *>(x)[b * n + idx];
            out[i] = mk((double)f.x, (double)f.y);
        } else {
            out[i] = reinterpret_cast<const cx *>(x)[b * n + idx];
        }
    }
}

// out[b, k] = sum_t x[b, t] * roots[(k t) mod n], roots[q] = e^{-2 pi i q/n}
// (table built as numpy builds it: exp(-2j*pi*arange(n)/n)), then / n.
// One warp per output bin; lanes stride t and the warp reduces.
__global__ void k_direct_dft(const cx *__restrict__ x, int64_t B, int64_t n, const cx *__restrict__ roots,
                             cx *__restrict__ out) {
    const int64_t w = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (w >= B * n) return;
    const int64_t b = w / n, k = w - b * n;
    cx acc = mk(0.0, 0.0);
    for (int64_t t = lane; t < n; t += 32)
        acc = cadd(acc, nmul(roots[(k * t) & (n - 1)], x[b * n + t]));
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        acc.re += __shfl_down_sync(0xffffffffu, acc.re, o);
        acc.im += __shfl_down_sync(0xffffffffu, acc.im, o);
    }
    if (lane == 0) out[w] = cdivr(acc, (double)n);
}

__global__ void k_dft_roots(int64_t n, cx *__restrict__ roots) {
    const int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (q >= n) return;
    // -2j * np.pi * arange(n) / n: (0, -2pi) * q, then complex / n
    roots[q] = gexp(mk(0.0, DMUL(-TWO_PI, (double)q) / (double)n));
}

// decode_bin status codes (Python maps them to the reference's exceptions)
enum { DB_OK = 0, DB_NEAR_SINGULAR = 1, DB_DEGENERATE = 2, DB_ILL_CONDITIONED = 3, DB_ZERO_ROOT = 4 };

// syndrome.py:147-175 for one bin: a = 1 ratio, or Hankel -> closed-form
// roots (residual bound) -> Vandermonde (conditioning bound), then
// root_to_location snapping and the membership flag.  `upto` stops early:
// 1 = coefficients, 2 = + roots, 3 = + values, 4 = full decode.
__global__ void k_decode_bins(const cx *__restrict__ m, int64_t nb, int64_t ld, int a, int64_t n, int64_t d,
                              const int64_t *__restrict__ bins, int upto, int32_t *__restrict__ status,
                              cx *__restrict__ c_out, cx *__restrict__ z_out, cx *__restrict__ p_out,
                              int64_t *__restrict__ loc_out, double *__restrict__ snap_out,
                              int32_t *__restrict__ member_out, double *__restrict__ diag) {
    const int64_t b = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (b >= nb) return;
    cx syn[8], c[4], z[4], p[4];
    for (int l = 0; l < 2 * a; l++) syn[l] = m[b * ld + l];
    int st = DB_OK;
    double dv = 0.0, db = 0.0;   // the failed test's statistic and bound (exception messages)
    double scale = 0.0;
    for (int l = 0; l < 2 * a; l++) scale = nanmax2(scale, cabs_(syn[l]));
    scale = nanmax2(scale, TINY);
    if (a == 1 && upto >= 2) {
        // decode_bin's a = 1 model: z = m1/m0, p = m0 (syndrome.py:160-165)
        dv = cabs_(syn[0]);
        db = DMUL(SINGULARITY_RTOL, scale);
        if (!(dv > db)) st = DB_NEAR_SINGULAR;
        z[0] = ndiv(syn[1], syn[0]);
        p[0] = syn[0];
        c[0] = mk(0.0, 0.0);
    } else {
        // solve_coefficients (syndrome.py:69-83)
        const cx cd = hankel_solve1(syn, a, c);
        dv = cabs_(cd);
        db = DMUL(SINGULARITY_RTOL, powa(scale, a));
        if (!(dv > db)) st = DB_NEAR_SINGULAR;
        if (st == DB_OK && upto >= 2) {
            // roots_closed_form (syndrome.py:86-98): every |P(z)| <= bound
            poly_roots1(c, a, z);
            double cmax = 0.0, resid = 0.0;
            for (int j = 0; j < a; j++) cmax = nanmax2(cmax, cabs_(c[j]));
            const double bound = DMUL(1e-8, nanmax2(1.0, cmax));
            bool bad = false;
            for (int r = 0; r < a; r++) {
                cx acc = mk(1.0, 0.0);
                for (int j = a - 1; j >= 0; j--) acc = cadd(nmul(acc, z[r]), c[j]);
                const double e = cabs_(acc);
                resid = (r == 0) ? e : nanmax2(resid, e);
                bad = bad || e > bound;
            }
            if (bad) {
                st = DB_DEGENERATE;
                dv = resid;
                db = bound;
            }
        }
        if (st == DB_OK && upto >= 3) {
            // solve_values (syndrome.py:109-123)
            const cx pd = vandermonde_solve1(z, syn, a, p);
            double zmax = 0.0;
            for (int j = 0; j < a; j++) zmax = (j == 0) ? cabs_(z[0]) : nanmax2(zmax, cabs_(z[j]));
            dv = cabs_(pd);
            db = DMUL(SINGULARITY_RTOL, powa(nanmax2(1.0, zmax), a));
            if (!(dv > db)) st = DB_ILL_CONDITIONED;
        }
    }
    if (st == DB_OK && upto >= 4) {
        double snap = 0.0;
        bool member = true;
        for (int j = 0; j < a; j++) {
            if (z[j].re == 0.0 && z[j].im == 0.0) {
                st = DB_ZERO_ROOT;
                break;
            }
            // root_to_location (syndrome.py:126-133): rint(angle(z) n / 2pi) mod n
            const double pos = DMUL(atan2(z[j].im, z[j].re), (double)n) / TWO_PI;
            const double sn = rint(pos);
            const int64_t loc = isfinite(sn) ? pmod((int64_t)sn, n) : INT64_MIN;
            loc_out[b * a + j] = loc;
            snap = nanmax2(snap, fabs(DSUB(pos, sn)));
            member = member && loc != INT64_MIN && (loc % (n / d)) == bins[b];
        }
        snap_out[b] = snap;
        member_out[b] = member;
    }
    status[b] = st;
    if (diag) {
        diag[2 * b] = dv;
        diag[2 * b + 1] = db;
    }
    for (int j = 0; j < a; j++) {
        c_out[b * a + j] = c[j];
        if (upto >= 2) z_out[b * a + j] = z[j];
        if (upto >= 3) p_out[b * a + j] = p[j];
    }
}

// |P(z)| (syndrome.py:101-106): Horner from the leading 1, numpy complex ops
__global__ void k_poly_residuals(const cx *__restrict__ c, const cx *__restrict__ z, int64_t nb, int a,
                                 double *__restrict__ out) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= nb * a) return;
    const int64_t b = i / a;
    const cx zz = z[i];
    cx acc = mk(1.0, 0.0);
    for (int j = a - 1; j >= 0; j--) acc = cadd(nmul(acc, zz), c[b * a + j]);
    out[i] = cabs_(acc);
}

// m_l = sum_j p_j z_j^l, l < count (syndrome.py:136-144)
__global__ void k_reconstruct(const cx *__restrict__ z, const cx *__restrict__ p, int64_t nb, int a, int count,
                              cx *__restrict__ out) {
    const int64_t b = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (b >= nb) return;
    cx power[4], terms[4], zz[4], pp[4];
    for (int j = 0; j < a; j++) {
        power[j] = mk(1.0, 0.0);
        zz[j] = z[b * a + j];
        pp[j] = p[b * a + j];
    }
    for (int l = 0; l < count; l++) {
        for (int j = 0; j < a; j++) terms[j] = nmul(pp[j], power[j]);
        out[b * count + l] = npsum(terms, a);
        for (int j = 0; j < a; j++) power[j] = nmul(power[j], zz[j]);
    }
}

inline unsigned grid_for(int64_t items, int threads) {
    int64_t g = (items + threads - 1) / threads;
    if (g > (int64_t(1) << 20)) g = int64_t(1) << 20;
    return (unsigned)(g < 1 ? 1 : g);
}

}  // namespace

extern "C" int sfdt_downsample(const void *x, int32_t x_dtype, int64_t batch, int64_t n, int64_t d,
                               const int64_t *shifts, int32_t nshift, double *out, sfdt_stream_t stream) {
    if (batch < 0 || n < 1 || d < 1 || n % d || nshift < 0 || (x_dtype != SFDT_C128 && x_dtype != SFDT_C64))
        return SFDT_EINVAL;
    if (batch == 0 || nshift == 0) return SFDT_OK;
    const int64_t total = batch * nshift * (n / d);
    k_downsample<<<grid_for(total, 256), 256, 0, (cudaStream_t)stream>>>(x, x_dtype == SFDT_C64, batch, n, d,
                                                                           shifts, nshift, (cx *)out);
    SFDT_CHECK_LAUNCH();
    return SFDT_OK;
}

extern "C" size_t sfdt_aliased_values_workspace_bytes(int64_t batch, int64_t n, int64_t d, int32_t nshift) {
    if (batch < 1 || d < 1 || n < d) return 256;
    const int64_t L = n / d;
    const int per = nshift < MAX_VIEWS ? nshift : MAX_VIEWS;
    return L > FFT_SMEM_MAX ? size_t(batch) * per * L * 16 + 256 : 256;
}

// out[b, v, :] = fft_radix2(x[b, (d*j + shift_v) mod n]) / (n/d): the
// solvers' fused gather + FFT kernels (bit-identical to the reference's
// transform_view), views in groups of MAX_VIEWS per launch.
extern "C" int sfdt_aliased_values(const void *x, int32_t x_dtype, int64_t batch, int64_t n, int64_t d,
                                   const int64_t *shifts, int32_t nshift, const double *twiddles, double *out,
                                   void *ws, size_t ws_bytes, sfdt_stream_t stream) {
    if (batch < 0 || n < 1 || (n & (n - 1)) || d < 1 || n % d || nshift < 0 || !twiddles ||
        (x_dtype != SFDT_C128 && x_dtype != SFDT_C64))
        return SFDT_EINVAL;
    if (batch == 0 || nshift == 0) return SFDT_OK;
    const int64_t L = n / d;
    if (L > FFT_SMEM_MAX && (!ws || ws_bytes < sfdt_aliased_values_workspace_bytes(batch, n, d, nshift)))
        return SFDT_EWORKSPACE;
    if (L > (int64_t(1) << 25)) return SFDT_EINVAL;
    for (int v0 = 0; v0 < nshift; v0 += MAX_VIEWS) {
        const int nv = nshift - v0 < MAX_VIEWS ? nshift - v0 : MAX_VIEWS;
        ViewSrc src = consecutive_views(x, x_dtype == SFDT_C64, n, d, 0, nv);
        src.dyn_off = shifts + v0;   // every view's shift from the table, same for all signals
        src.dyn_first = 0;
        src.dyn_stride = 0;
        src.wrap = n - 1;
        // views land at out[b, v0 + v, :] : view slot v of signal b at
        // (b * SV + v) * ldV with SV = nshift
        const int rc = launch_fft_views(src, batch, L, twiddles, (cx *)out + v0 * L, nshift, L,
                                        (cudaStream_t)stream, L > FFT_SMEM_MAX ? (cx *)ws : nullptr, 1);
        if (rc) return rc;
    }
    return SFDT_OK;
}

extern "C" int sfdt_direct_dft(const double *x, int64_t batch, int64_t n, double *roots_ws, double *out,
                               sfdt_stream_t stream_) {
    if (batch < 0 || n < 1 || (n & (n - 1)) || !roots_ws) return SFDT_EINVAL;
    if (batch == 0) return SFDT_OK;
    cudaStream_t stream = (cudaStream_t)stream_;
    k_dft_roots<<<grid_for(n, 256), 256, 0, stream>>>(n, (cx *)roots_ws);
    const int64_t warps = batch * n;
    k_direct_dft<<<(unsigned)((warps * 32 + 255) / 256), 256, 0, stream>>>((const cx *)x, batch, n,
                                                                             (const cx *)roots_ws, (cx *)out);
    SFDT_CHECK_LAUNCH();
    return SFDT_OK;
}

extern "C" int sfdt_decode_bins(const double *m, int64_t nb, int64_t ld, int a, int64_t n, int64_t d,
                                const int64_t *bins, int upto, int32_t *status, double *c, double *roots,
                                double *vals, int64_t *locs, double *snap, int32_t *member, double *diag,
                                sfdt_stream_t stream) {
    if (a < 1 || a > 4 || ld < 2 * a || nb < 0 || n < 1 || (n & (n - 1)) || d < 1 || n % d || upto < 1 ||
        upto > 4 || !status || !c || (upto >= 2 && !roots) || (upto >= 3 && !vals) ||
        (upto >= 4 && (!locs || !snap || !member || !bins)))
        return SFDT_EINVAL;
    if (nb == 0) return SFDT_OK;
    k_decode_bins<<<grid_for(nb, 128), 128, 0, (cudaStream_t)stream>>>(
        (const cx *)m, nb, ld, a, n, d, bins, upto, status, (cx *)c, (cx *)roots, (cx *)vals, locs, snap, member, diag);
    SFDT_CHECK_LAUNCH();
    return SFDT_OK;
}

extern "C" int sfdt_poly_residuals(const double *c, const double *z, int64_t nb, int a, double *out,
                                   sfdt_stream_t stream) {
    if (a < 1 || nb < 0) return SFDT_EINVAL;
    if (nb == 0) return SFDT_OK;
    k_poly_residuals<<<grid_for(nb * a, 128), 128, 0, (cudaStream_t)stream>>>((const cx *)c, (const cx *)z, nb,
                                                                              a, out);
    SFDT_CHECK_LAUNCH();
    return SFDT_OK;
}

extern "C" int sfdt_reconstruct_syndromes(const double *roots, const double *vals, int64_t nb, int a, int count,
                                          double *out, sfdt_stream_t stream) {
    if (a < 1 || a > 4 || nb < 0 || count < 0) return SFDT_EINVAL;
    if (nb == 0 || count == 0) return SFDT_OK;
    k_reconstruct<<<grid_for(nb, 128), 128, 0, (cudaStream_t)stream>>>((const cx *)roots, (const cx *)vals, nb,
                                                                       a, count, (cx *)out);
    SFDT_CHECK_LAUNCH();
    return SFDT_OK;
}
