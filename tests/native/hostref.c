/* gcc/glibc C99 complex references for tests/test_math.py */
#include <complex.h>
#include <stdint.h>
void hr_div(const double _Complex *a, const double _Complex *b, double _Complex *o, int64_t n) { for (int64_t i = 0; i < n; i++) o[i] = a[i] / b[i]; }
void hr_mul(const double _Complex *a, const double _Complex *b, double _Complex *o, int64_t n) { for (int64_t i = 0; i < n; i++) o[i] = a[i] * b[i]; }
void hr_sqrt(const double _Complex *a, double _Complex *o, int64_t n) { for (int64_t i = 0; i < n; i++) o[i] = csqrt(a[i]); }
void hr_cbrt(const double _Complex *a, double _Complex *o, int64_t n) { for (int64_t i = 0; i < n; i++) o[i] = cpow(a[i], 1.0 / 3.0); }
