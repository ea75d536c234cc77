/* twiddle.c -- host-side FFT twiddle tables (C99, built by gcc without FMA
 * contraction, like the reference's extension, pkg/setup.py:14-30).
 *
 * The reference's radix-2 FFT (_core.pyx:61-76) does not use exact
 * twiddles: per butterfly block it runs the recurrence w <- w * wlen from
 * w = 1, re-seeding w = cexp(sign*2i*pi*k/m) every 256 steps.  The values
 * only depend on the stage length m, so one table per (n_max, sign) serves
 * every view length <= n_max.  Stage m occupies [m/2 - 1, m - 1). */
#include <complex.h>
#include <math.h>
#include <stdint.h>

int sfdt_fft_twiddles(int64_t n_max, int inverse, double *host_out)
{
    if (n_max < 1 || (n_max & (n_max - 1)) || !host_out)
        return -1;
    const double sign = inverse ? 1.0 : -1.0;
    const double _Complex two_i = 2.0 * I;
    double _Complex *out = (double _Complex *)host_out;
    for (int64_t m = 2; m <= n_max; m <<= 1) {
        const int64_t half = m >> 1;
        const double _Complex wlen =
            cexp(((double _Complex)sign * two_i * (double _Complex)M_PI) / (double _Complex)(double)m);
        double _Complex w = 1.0;
        for (int64_t k = 0; k < half; k++) {
            if ((k & 255) == 0 && k > 0)
                w = cexp((((double _Complex)sign * two_i * (double _Complex)M_PI) * (double _Complex)(double)k)
                         / (double _Complex)(double)m);
            out[half - 1 + k] = w;
            w = w * wlen;
        }
    }
    return 0;
}
