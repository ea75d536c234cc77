"""pytest plugin: run the reference's own test suite (baseline/_ref/tests,
staged by tools/stage_reference.sh) against the B200 implementation.

SFDT_REFSUITE_MODE
  stock   the unmodified reference, as staged (the suite's own baseline)
  seam    the reference's Python code with its kernel seam bound to the B200
          library: sfft_dt._kernels.<fn> = paper_1407_8315_b200.kernels.<fn>
          (the six functions of _kernels/__init__.py:19-24, looked up at call
          time by every call site) -- the binding INTEGRATION.md proposes
  dropin  `sfft_dt` IS paper_1407_8315_b200: the suite's
          `from sfft_dt import spectral / syndrome` resolve to the B200
          modules (downsample, transform_view, decode_bin, ... on the GPU)
"""

import os
import sys

_SEAM = ("fft_radix2", "hankel_solve", "poly_roots", "vandermonde_solve", "prune_eval",
         "hankel_singular_values")


def pytest_configure(config):
    mode = os.environ.get("SFDT_REFSUITE_MODE", "stock")
    if mode == "stock":
        return
    import paper_1407_8315_b200 as P
    from paper_1407_8315_b200 import kernels as K
    if mode == "seam":
        from sfft_dt import _kernels
        for name in _SEAM:
            setattr(_kernels, name, getattr(K, name))
        _kernels.BACKEND = "b200"
    elif mode == "dropin":
        from paper_1407_8315_b200 import general, spectral, syndrome
        sys.modules["sfft_dt"] = P
        sys.modules["sfft_dt.spectral"] = spectral
        sys.modules["sfft_dt.syndrome"] = syndrome
        sys.modules["sfft_dt.general"] = general
        sys.modules["sfft_dt._kernels"] = K
    else:
        raise ValueError(f"unknown SFDT_REFSUITE_MODE {mode!r}")


def pytest_report_header(config):
    return f"sfdt refsuite mode: {os.environ.get('SFDT_REFSUITE_MODE', 'stock')}"
