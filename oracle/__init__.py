"""CPU oracle for the dd Rgemm / Rsyrk hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this package, and
only as the checker / the timed CPU reference -- never as the product path.

* ``dd_oracle.c``  -- bit-exact C restatement of the reference's dd Rgemm /
  Rsyrk (``/root/reference/pkg/src/mpkit/mpblas/level23.py:107-285`` over the
  element kernels of ``mpblas/elem.py:32-78``).  Parity pinned against the
  reference's own outputs in ``tests/golden/`` (made by ``gen_golden.py``).
* ``exact.py``     -- exact rational (Python big-int) values of sampled
  entries of alpha*op(A)*op(B) + beta*C, used to check the error bound of the
  ``fast`` mode, cross-checked against mpmath at 240 bits.
"""
