"""CPU oracle for the TokenSwift decode step — TEST INFRASTRUCTURE ONLY.

This package is a numpy (float64) restatement of the reference algorithm
(`/root/reference/pkg/src/swiftdec`, arXiv 2502.18890). Every function cites
the reference file:line it follows. It exists for three callers only:

* ``tests/`` — the parity checker the CUDA path is compared against;
* ``__graft_entry__.smoke()`` — the tiny on-GPU self check;
* ``bench.py`` — the ``cpu_baseline`` leg and ``--impl reference`` arm.

The product package (``paper_2502_18890_b200``) never imports it; the product
path fails loudly when its CUDA library is missing.

Parity pinning: the restatement is checked against golden vectors produced by
running the reference itself in the build container
(``tests/golden/make_golden.py`` -> ``tests/golden/*.json|npz``) and against
the reference's own known-answer tests restated in ``tests/test_oracle_*.py``.
"""

from . import engine, kvcache, model, ngram, rng, sampling, tree  # noqa: F401
