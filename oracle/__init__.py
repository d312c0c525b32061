"""CPU oracle for the Vecchia hot path -- TEST INFRASTRUCTURE ONLY.

Nothing under ``oracle/`` is imported by the product package
``paper_2407_02740_b200``.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s cpu_baseline / ``--impl reference`` legs may use it, and only as
the checker or the timed CPU baseline.

Modules
-------
vecchia_oracle   ctypes wrapper over ``libvecchia_oracle.so`` (the plain-C
                 restatement in ``vecchia_oracle.c``; parity status in its header).
numpy_families   a second, arithmetically independent numpy/LAPACK restatement
                 (follows the reference's fallback core), used to cross-check the
                 C oracle on the families the reference does not have.
reference_core   loader for ``oracle/_ref/_kernels*.so`` -- the reference's OWN
                 compiled core built by ``oracle/build_ref.sh`` (when present).
"""
