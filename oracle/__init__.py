"""CPU oracle for the SPIR-V codec path -- TEST INFRASTRUCTURE ONLY.

A plain-Python restatement of the reference algorithms (``spirvkit`` 0.1.0,
``/root/reference/pkg/src/spirvkit``) used as the parity checker for the CUDA
path.  Every function cites the reference ``file:line`` it restates.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg may import this package, and only as the checker / baseline -- never as the
thing measured or shipped.  The product package
(``paper_2305_09493_b200``) never imports it; its codec path fails loudly when
the CUDA library is missing.

Parity pinning: ``tests/test_oracle_golden.py`` checks this oracle against the
golden vectors in ``tests/golden/`` (produced by running the reference itself,
``tools/make_golden.py``) and against the known-answer cases of the
reference's own test-suite.
"""

from . import core, disasm, validate  # noqa: F401
