"""Golden-case definitions shared by make_golden.py and the tests.

Each exact case: (name, n, k, mu, a_max, values, seed, synth).
Each general case: (name, n, k, snr_db, seed, prune).
Small enough that the CPU oracle finishes each in well under a second.
"""

EXACT_CASES = [
    # config 1 exactly: gen_exact(n=2^16, k=64, seed=0), reference radix-2 synthesis
    ("cfg1", 1 << 16, 64, 4, 4, "unit", 0, "radix2"),
    ("n4096_k32_mag", 4096, 32, 4, 4, "mag1_10", 1, "numpy"),
    ("n8192_k128_mu1", 8192, 128, 1, 4, "unit", 2, "numpy"),
    ("n16384_k256_mu2", 16384, 256, 2, 4, "unit", 3, "numpy"),
    ("n16384_k64_gauss", 16384, 64, 4, 4, "gauss", 4, "numpy"),
    ("n1024_k16_mu1", 1024, 16, 1, 4, "unit", 5, "numpy"),
    ("n4096_k64_mu1_a3", 4096, 64, 1, 3, "mag1_10", 6, "numpy"),
    ("n65536_k1024_mu1", 1 << 16, 1024, 1, 4, "unit", 7, "numpy"),
    # |v| = 10^U(-8, 0): the iterative solver re-decodes a location it
    # already wrote -> "duplicate location" warnings, last write wins
    # (exact.py:152-158); seeds chosen by searching with the real reference
    ("dup_n1024_k32_mu1", 1024, 32, 1, 4, "logmag", 19, "numpy"),
    ("dup_n4096_k64_mu1", 4096, 64, 1, 4, "logmag", 36, "numpy"),
    ("dup_n2048_k64_mu2", 2048, 64, 2, 4, "logmag", 0, "numpy"),
    ("dup_n8192_k128_mu1_a3", 8192, 128, 1, 3, "logmag", 19, "numpy"),
]

# cases re-run with the reference's pure-numpy backend (SFFT_DT_PURE_PYTHON=1)
# -- pins oracle/numpy_kernels.py, the envelope backend of the parity tests
NUMPY_BACKEND_CASES = ["cfg1", "n8192_k128_mu1", "dup_n1024_k32_mu1"]
NUMPY_BACKEND_GENERAL = ["g_n16384_k16_20db"]

GENERAL_CASES = [
    ("g_n16384_k16_20db", 16384, 16, 20.0, 11, True),
    ("g_n32768_k32_30db", 32768, 32, 30.0, 12, True),
    ("g_n16384_k8_10db", 16384, 8, 10.0, 13, True),
    ("g_n8192_k4_20db_noprune", 8192, 4, 20.0, 14, False),
    ("g_n65536_k256_30db", 1 << 16, 256, 30.0, 15, True),
]
