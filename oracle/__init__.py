"""TEST INFRASTRUCTURE ONLY -- the CPU parity oracle for the sFFT-DT hot path.

* ``oracle/kernels.c``  : C restatement of the reference's compiled kernels
  (/root/reference/pkg/src/sfft_dt/_kernels/_core.pyx), bit-identical to them.
* ``oracle/solvers.py`` : numpy restatement of the reference solver drivers
  (exact.py, general.py) over those kernels.
* ``oracle/Makefile``   : builds the C restatement and, when /root/reference is
  present, the reference's own Cython kernels into ``oracle/_ref``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs use
this package, and only as the checker / CPU baseline -- never as the product.
"""
