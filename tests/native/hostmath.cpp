// Host build of the device math (paper_1407_8315_b200/csrc/cx.cuh) so that
// tests/test_math.py can check it bit-for-bit against gcc/glibc/numpy.
#include "../../paper_1407_8315_b200/csrc/cx.cuh"
#include <complex.h>

using namespace sfdt;

extern "C" {
void hm_gdiv(const cx *a, const cx *b, cx *o, int64_t n) { for (int64_t i = 0; i < n; i++) o[i] = gdiv(a[i], b[i]); }
void hm_ndiv(const cx *a, const cx *b, cx *o, int64_t n) { for (int64_t i = 0; i < n; i++) o[i] = ndiv(a[i], b[i]); }
void hm_nmul(const cx *a, const cx *b, cx *o, int64_t n) { for (int64_t i = 0; i < n; i++) o[i] = nmul(a[i], b[i]); }
void hm_gmul(const cx *a, const cx *b, cx *o, int64_t n) { for (int64_t i = 0; i < n; i++) o[i] = gmul(a[i], b[i]); }
void hm_gsqrt(const cx *a, cx *o, int64_t n) { for (int64_t i = 0; i < n; i++) o[i] = gsqrt(a[i]); }
void hm_gcbrt(const cx *a, cx *o, int64_t n) { for (int64_t i = 0; i < n; i++) o[i] = gcbrt(a[i]); }
// native gcc/glibc references for the same operations
void hm_ref_div(const double _Complex *a, const double _Complex *b, double _Complex *o, int64_t n) { for (int64_t i = 0; i < n; i++) o[i] = a[i] / b[i]; }
void hm_ref_sqrt(const double _Complex *a, double _Complex *o, int64_t n) { for (int64_t i = 0; i < n; i++) o[i] = csqrt(a[i]); }
void hm_ref_cbrt(const double _Complex *a, double _Complex *o, int64_t n) { for (int64_t i = 0; i < n; i++) o[i] = cpow(a[i], 1.0 / 3.0); }
void hm_hankel(const cx *m, int64_t nb, int64_t ld, int a, cx *c, cx *cd) { for (int64_t b = 0; b < nb; b++) cd[b] = hankel_solve1(m + b * ld, a, c + b * a); }
void hm_roots(const cx *c, int64_t nb, int a, cx *z) { for (int64_t b = 0; b < nb; b++) poly_roots1(c + b * a, a, z + b * a); }
void hm_vand(const cx *z, const cx *m, int64_t nb, int a, int64_t ld, cx *p, cx *pd) { for (int64_t b = 0; b < nb; b++) pd[b] = vandermonde_solve1(z + b * a, m + b * ld, a, p + b * a); }
}
