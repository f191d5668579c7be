"""CPU oracle for the incremental RTEC hot path -- TEST INFRASTRUCTURE ONLY.

This package is a numpy restatement of the reference `streamgnn` algorithms
(`/root/reference/pkg/src/streamgnn/`), used as the *checker* for the B200
engine in `paper_2603_20622_b200`.  Only `tests/`, `__graft_entry__.smoke()`
and `bench.py`'s CPU-baseline / `--impl reference` leg may import it.  The
product path never imports, links or calls anything in here; it fails loudly
when its CUDA extension is missing.

Pinning: every function below cites the reference file:line it restates, and
`tests/test_oracle_golden.py` checks the restatement against golden vectors
produced by the *reference itself* (`tests/golden/make_golden.py` imports
`/root/reference/pkg/src/streamgnn` in the build container and records its
outputs as `.npz` fixtures).  The incremental engine (which the reference does
not ship, Alg. 1/3/4) is pinned through the
reference's own full-recompute oracle (`models.py:461-492`) on the post-batch
graphs: after every batch its state must equal `layer_embeddings` to ~1e-12
in f64.

Modules
- `graph`  : DynamicGraph semantics (graph.py:59-266) over sorted key arrays.
- `models` : make_bundle weight init (models.py:56-384) and the vectorised
             full-neighbourhood layer (models.py:431-492).
- `engine` : frontier (Alg. 4 with the SURVEY §8(a)-F1 rule), state cache and
             Alg. 1 / Alg. 3 incremental layers over the restated operators.
"""
