"""TEST INFRASTRUCTURE ONLY -- CPU oracle for the TW / TEW path.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference`` arm) may import this package,
and only as the checker / the timed CPU baseline -- never as the product.

Contents
  tilesparse_oracle.py  restatement of the reference CPU algorithm:
                        naive loop TW/TEW pruning (small sizes), faithful
                        numpy ports of executor.py's _mac_kernel /
                        execute_batched / gemm_tew, and a ctypes binding of
  tw_oracle.c           the same fp64 ascending-k kernel in C (fast parity
                        checks at full BERT sizes).

Pinning: tests/test_oracle_golden.py checks every function here against the
golden vectors in tests/golden/, which tests/golden/make_golden.py generated
by importing the unmodified reference (pkg/src/tilesparse) in the build
container.
"""
