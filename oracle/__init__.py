"""CPU oracle for the exhaustive FCNN-surrogate sweep of arxiv 2306.14011.

TEST INFRASTRUCTURE ONLY.  Nothing on the product path may import, call or
execute anything in this package: only ``tests/``, ``__graft_entry__.smoke()``
and the ``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may.  The
oracle shares no code with ``paper_2306_14011_b200`` (the CUDA path); the only
thing both sides consume is ``workloads/`` (seeded synthetic inputs: space value
lists, weight files produced by ``scripts/make_weights.py`` which calls only this
package).

Everything is plain numpy in IEEE float64.  Citations ``P:n`` are lines of the
paper text, ``S:n`` lines of SPEC.md, both as catalogued in SURVEY.md.

Modules
-------
space   : cardinality, mixed-radix decode/encode, enumeration, sampling, split
cost    : synthetic solver-time surface standing in for the paper's timings
scaler  : StandardScaler and the min-max alternative (G1)
mlp     : FCNN forward / backward / Adam training, R^2
sweep   : t(I) over an index range and the (t, I) top-k

Parity status: every function is pinned by a ``-m "not gpu"`` test in
``tests/test_oracle_*.py`` except where its docstring says "parity unpinned".
"""

from . import space, cost, scaler, mlp, sweep  # noqa: F401
