// kernels.cu -- batched device mirrors of the reference backend seam
// (_kernels/__init__.py:19-24) behind the C ABI, so the reference's own
// kernel-level known answers can target the B200 code directly.
#include "common.cuh"
#include "decode.cuh"
#include "fft.cuh"
#include "general.cuh"

using namespace sfdt;

namespace {

__global__ void k_hankel(const cx *m, int64_t nb, int64_t ld, int a, cx *c, cx *cd) {
    const int64_t b = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (b >= nb) return;
    cx mm[8], cc[4];
    for (int i = 0; i < 2 * a; i++) mm[i] = m[b * ld + i];
    cd[b] = hankel_solve1(mm, a, cc);
    for (int j = 0; j < a; j++) c[b * a + j] = cc[j];
}

__global__ void k_roots(const cx *c, int64_t nb, int a, cx *z) {
    const int64_t b = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (b >= nb) return;
    cx cc[4], zz[4];
    for (int j = 0; j < a; j++) cc[j] = c[b * a + j];
    poly_roots1(cc, a, zz);
    for (int j = 0; j < a; j++) z[b * a + j] = zz[j];
}

__global__ void k_vand(const cx *z, const cx *m, int64_t nb, int a, int64_t ld, cx *p, cx *pd) {
    const int64_t b = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (b >= nb) return;
    cx zz[4], mm[4], pp[4];
    for (int j = 0; j < a; j++) {
        zz[j] = z[b * a + j];
        mm[j] = m[b * ld + j];
    }
    pd[b] = vandermonde_solve1(zz, mm, a, pp);
    for (int j = 0; j < a; j++) p[b * a + j] = pp[j];
}

__global__ void k_svd(const cx *m, int64_t nb, int64_t ld, int a_max, double *out) {
    const int64_t b = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (b >= nb) return;
    cx mm[7];
    double sv[4];
    for (int i = 0; i < 2 * a_max - 1; i++) mm[i] = m[b * ld + i];
    hankel_singular_values1(mm, a_max, sv);
    for (int j = 0; j < a_max; j++) out[b * a_max + j] = sv[j];
}

// (bin, chunk of 512 candidates) per thread: the reference's recurrence is
// sequential inside each 512-chunk and re-seeded at chunk starts
__global__ void k_prune(const cx *c, const int64_t *k, int64_t nb, int a, int64_t n, int64_t d,
                        double *out) {
    const int64_t nchunk = (d + 511) / 512;
    const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= nb * nchunk) return;
    const int64_t b = t / nchunk, ch = t - b * nchunk;
    cx cc[4];
    for (int j = 0; j < a; j++) cc[j] = c[b * a + j];
    const cx base = gexp(mk(0.0, DMUL(TWO_PI, (double)k[b]) / (double)n));
    const cx wd = gexp(mk(0.0, TWO_PI / (double)d));
    const cx seed = ch ? gexp(mk(0.0, DMUL(TWO_PI, (double)(ch * 512)) / (double)d)) : mk(1.0, 0.0);
    prune_eval_chunk(cc, a, base, wd, seed, ch, d, out + b * d);
}

}  // namespace

extern "C" {

const char *sfdt_strerror(int code) {
    switch (code) {
    case SFDT_OK: return "ok";
    case SFDT_EINVAL: return "invalid argument";
    case SFDT_ECUDA: return "CUDA error";
    case SFDT_EWORKSPACE: return "workspace too small";
    case SFDT_ECAPACITY: return "output capacity too small";
    default: return "unknown error";
    }
}

int sfdt_version(void) { return 10000; }

void sfdt_default_tuning(sfdt_tuning *out) {
    if (out) *out = default_tuning();
}

const char *sfdt_last_cuda_error(void) { return cudaGetErrorString(cudaPeekAtLastError()); }

int sfdt_fft_radix2(const double *x, double *out, int64_t batch, int64_t n, int inverse,
                    const double *twiddles, sfdt_stream_t stream) {
    (void)inverse;   // the table carries the sign
    if (batch < 0 || n < 1 || (n & (n - 1)) || n > (int64_t(1) << 25) || !twiddles) return SFDT_EINVAL;
    if (batch == 0) return SFDT_OK;
    // a (batch, n) array of signals, each its own single view (d = 1); long
    // transforms run the two-pass stage split with `out` as the scratch
    // (pass B reads and writes the same residue-class tile, so in place is safe)
    const ViewSrc src = consecutive_views(x, 0, n, 1, 0, 1);
    return launch_fft_views(src, batch, n, twiddles, (cx *)out, 1, n, (cudaStream_t)stream,
                            (cx *)out, 0);
}

int sfdt_hankel_solve(const double *m, int64_t nb, int64_t ld, int a, double *c, double *cd,
                      sfdt_stream_t stream) {
    if (a < 1 || a > 4 || ld < 2 * a || nb < 0) return SFDT_EINVAL;
    if (!nb) return SFDT_OK;
    k_hankel<<<(unsigned)((nb + 127) / 128), 128, 0, (cudaStream_t)stream>>>((const cx *)m, nb, ld, a,
                                                                             (cx *)c, (cx *)cd);
    SFDT_CHECK_LAUNCH();
    return SFDT_OK;
}

int sfdt_poly_roots(const double *c, int64_t nb, int a, double *z, sfdt_stream_t stream) {
    if (a < 1 || a > 4 || nb < 0) return SFDT_EINVAL;
    if (!nb) return SFDT_OK;
    k_roots<<<(unsigned)((nb + 127) / 128), 128, 0, (cudaStream_t)stream>>>((const cx *)c, nb, a, (cx *)z);
    SFDT_CHECK_LAUNCH();
    return SFDT_OK;
}

int sfdt_vandermonde_solve(const double *z, const double *m, int64_t nb, int a, int64_t ld,
                           double *p, double *pd, sfdt_stream_t stream) {
    if (a < 1 || a > 4 || ld < a || nb < 0) return SFDT_EINVAL;
    if (!nb) return SFDT_OK;
    k_vand<<<(unsigned)((nb + 127) / 128), 128, 0, (cudaStream_t)stream>>>(
        (const cx *)z, (const cx *)m, nb, a, ld, (cx *)p, (cx *)pd);
    SFDT_CHECK_LAUNCH();
    return SFDT_OK;
}

int sfdt_prune_eval(const double *c, const int64_t *k, int64_t nb, int a, int64_t n, int64_t d,
                    double *out, sfdt_stream_t stream) {
    if (a < 1 || a > 4 || nb < 0 || d < 1) return SFDT_EINVAL;
    if (!nb) return SFDT_OK;
    const int64_t nt = nb * ((d + 511) / 512);
    k_prune<<<(unsigned)((nt + 127) / 128), 128, 0, (cudaStream_t)stream>>>((const cx *)c, k, nb, a, n,
                                                                            d, out);
    SFDT_CHECK_LAUNCH();
    return SFDT_OK;
}

int sfdt_hankel_singular_values(const double *m, int64_t nb, int64_t ld, int a_max, double *out,
                                sfdt_stream_t stream) {
    if (a_max < 1 || a_max > 4 || ld < 2 * a_max - 1 || nb < 0) return SFDT_EINVAL;
    if (!nb) return SFDT_OK;
    k_svd<<<(unsigned)((nb + 127) / 128), 128, 0, (cudaStream_t)stream>>>((const cx *)m, nb, ld, a_max,
                                                                          out);
    SFDT_CHECK_LAUNCH();
    return SFDT_OK;
}

}  // extern "C"
