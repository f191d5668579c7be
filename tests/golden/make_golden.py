"""Generate golden fixtures by running the REFERENCE itself.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden.py

It imports `streamgnn` from /root/reference/pkg/src (read-only) and records
its outputs as small .npz files next to this script.  The fixtures travel with
the repo; nothing at test time reads /root/reference.

Fixtures
- graph_streams.npz : DynamicGraph.from_edges + apply_batch over mixed batches
  (rejects, self-loops), the ApplyResult (applied flags in batch order,
  DegreeDelta rows), final edges()/degrees, plus error cases
  (InvalidVertex / ConfigError ordering, atomicity).
- coalesce.npz      : coalesce_batch on random multi-event sequences.
- models_<name>.npz : make_bundle weights, X, and layer_embeddings (H, A, C)
  on the initial graph and after every batch of a mixed stream
  (graph mutated with the reference's own apply_batch).
"""

from __future__ import annotations

import os
import sys
import zlib

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)
sys.path.insert(0, os.path.abspath(os.path.join(OUT, "..", "..")))

from streamgnn import errors as E  # noqa: E402
from streamgnn import graph as G  # noqa: E402
from streamgnn import models as Mo  # noqa: E402

from paper_2603_20622_b200.workload import chung_lu_edges  # noqa: E402

OPS = {0: G.UpdateOp.INSERT, 1: G.UpdateOp.DELETE}


def to_updates(op, src, dst, ts):
    return [G.EdgeUpdate(OPS[int(o)], int(s), int(d), int(t)) for o, s, d, t in zip(op, src, dst, ts)]


def mixed_batch(rng, g, n, B, p_reject=0.15, p_self=0.05):
    """B distinct-key updates: inserts of absent edges, deletes of live edges,
    plus deliberate rejects (duplicate insert / absent delete) and self-loops."""
    es, ed, _ = g.edges()
    live = set(zip(es.tolist(), ed.tolist()))
    used = set()
    out = []
    while len(out) < B:
        r = rng.random()
        if r < p_reject:
            if rng.random() < 0.5 and live:  # duplicate insert
                k = list(live)[int(rng.integers(len(live)))]
                o = 0
            else:  # absent delete
                k = (int(rng.integers(n)), int(rng.integers(n)))
                if k in live:
                    continue
                o = 1
        elif r < p_reject + p_self:
            v = int(rng.integers(n))
            k = (v, v)
            o = 1 if k in live else 0
        elif rng.random() < 0.5 and live:
            k = list(live)[int(rng.integers(len(live)))]
            o = 1
        else:
            k = (int(rng.integers(n)), int(rng.integers(n)))
            if k in live:
                continue
            o = 0
        if k in used:
            continue
        used.add(k)
        out.append((o, k[0], k[1], 10_000 + len(out)))
    a = np.asarray(out, np.int64)
    return a[:, 0].astype(np.uint8), a[:, 1], a[:, 2], a[:, 3]


def record_result(res, batch_len, upd):
    applied_set = {(u.src, u.dst) for u in res.applied}
    flags = np.array([1 if (u.src, u.dst) in applied_set else 0 for u in upd], np.uint8)
    # also check the reference reports applied/rejected in batch order
    assert [(u.src, u.dst) for u in res.applied] == [(u.src, u.dst) for u in upd if (u.src, u.dst) in applied_set]
    deltas = np.array([[d.vertex, d.old_in, d.new_in, d.old_out, d.new_out] for d in res.deltas], np.int64).reshape(-1, 5)
    return flags, deltas


def graph_streams():
    rng = np.random.default_rng(11)
    out = {}
    cases = [(40, 120, 6, 12), (300, 3000, 5, 64), (3, 0, 2, 3)]
    for ci, (n, m, nb, B) in enumerate(cases):
        if m:
            s, d = chung_lu_edges(n, m, alpha=0.8, seed=ci)
            ts = rng.permutation(m).astype(np.int64)
        else:
            s = d = ts = np.zeros(0, np.int64)
        g = G.DynamicGraph.from_edges(n, list(zip(s.tolist(), d.tolist(), ts.tolist())))
        out[f"c{ci}_n"] = np.int64(n)
        out[f"c{ci}_src"], out[f"c{ci}_dst"], out[f"c{ci}_ts"] = s, d, ts
        out[f"c{ci}_nb"] = np.int64(nb)
        for b in range(nb):
            op, bs, bd, bt = mixed_batch(rng, g, n, B)
            upd = to_updates(op, bs, bd, bt)
            res = g.apply_batch(upd)
            flags, deltas = record_result(res, B, upd)
            p = f"c{ci}_b{b}_"
            out[p + "op"], out[p + "src"], out[p + "dst"], out[p + "ts"] = op, bs, bd, bt
            out[p + "status"], out[p + "deltas"] = flags, deltas
            es, ed, et = g.edges()
            out[p + "esrc"], out[p + "edst"], out[p + "ets"] = es, ed, et
            out[p + "indeg"] = g.in_degrees.copy()
            out[p + "outdeg"] = g.out_degrees.copy()
            # neighbour runs of a few vertices through the public queries
            vs = np.unique(np.concatenate([bs[:4], bd[:4]]))
            out[p + "qv"] = vs
            out[p + "qin"] = np.concatenate([g.in_neighbors(int(v)) for v in vs] + [np.zeros(0, np.int64)])
            out[p + "qin_len"] = np.array([g.in_neighbors(int(v)).size for v in vs], np.int64)
            out[p + "qout"] = np.concatenate([g.out_neighbors(int(v)) for v in vs] + [np.zeros(0, np.int64)])
            out[p + "qout_len"] = np.array([g.out_neighbors(int(v)).size for v in vs], np.int64)
    # error cases: (batch, expected exception name, first-offender semantics)
    n = 10
    g = G.DynamicGraph.from_edges(n, [(0, 1), (1, 2), (2, 3)])
    err = []
    errcases = [
        [(0, 4, 5, 1), (0, 4, 11, 2)],                  # InvalidVertex (dst)
        [(0, 4, 5, 1), (0, 4, 5, 2)],                   # ConfigError duplicate
        [(0, 4, 5, 1), (0, 4, 5, 2), (0, -1, 3, 3)],    # dup before invalid -> ConfigError
        [(0, 4, 5, 1), (0, 12, 3, 2), (0, 4, 5, 3)],    # invalid before dup -> InvalidVertex
        [(1, 0, 1, 1), (0, 10, 0, 2)],                  # src out of range, no mutation
    ]
    for i, rows in enumerate(errcases):
        before = g.edges()
        a = np.asarray(rows, np.int64)
        try:
            g.apply_batch(to_updates(a[:, 0], a[:, 1], a[:, 2], a[:, 3]))
            name = "none"
        except E.InvalidVertex:
            name = "InvalidVertex"
        except E.ConfigError:
            name = "ConfigError"
        after = g.edges()
        assert all(np.array_equal(x, y) for x, y in zip(before, after)), "reference mutated on error"
        out[f"err{i}_batch"] = a
        err.append(name)
    out["err_names"] = np.array(err)
    np.savez_compressed(os.path.join(OUT, "graph_streams.npz"), **out)
    print("graph_streams.npz:", len(out), "arrays; errors", err)


def coalesce_cases():
    rng = np.random.default_rng(5)
    out = {}
    # SURVEY appendix A.2 example
    ex = [(0, 1, 2, 10), (1, 1, 2, 11), (0, 3, 4, 12), (0, 1, 2, 13), (0, 3, 4, 14), (1, 5, 6, 15)]
    cases = [np.asarray(ex, np.int64)]
    for _ in range(20):
        B = int(rng.integers(1, 200))
        k = int(rng.integers(1, 12))
        a = np.stack([rng.integers(0, 2, B), rng.integers(0, k, B), rng.integers(0, k, B),
                      rng.integers(0, 10**9, B)], axis=1).astype(np.int64)
        cases.append(a)
    for i, a in enumerate(cases):
        res = G.coalesce_batch(to_updates(a[:, 0], a[:, 1], a[:, 2], a[:, 3]))
        r = np.array([[0 if u.op is G.UpdateOp.INSERT else 1, u.src, u.dst, u.ts] for u in res], np.int64).reshape(-1, 4)
        out[f"in{i}"], out[f"out{i}"] = a, r
    out["count"] = np.int64(len(cases))
    np.savez_compressed(os.path.join(OUT, "coalesce.npz"), **out)
    print("coalesce.npz:", len(cases), "cases; example ->", out["out0"].tolist())


def head_seed(seed, layer, head, heads):  # mirrors oracle.models.head_seed (multi-head scheme)
    return int(seed) * 1009 + 1 + layer * heads + head


def model_case(name, model, dims, smoothing=True, heads=1, n=100, m=600, nb=6, B=16):
    rng = np.random.default_rng(zlib.crc32(name.encode()))
    s, d = chung_lu_edges(n, m, alpha=0.8, seed=3)
    g = G.DynamicGraph.from_edges(n, list(zip(s.tolist(), d.tolist())))
    X = rng.uniform(-1, 1, (n, dims[0])).astype(np.float32).astype(np.float64)
    out = {"n": np.int64(n), "src": s, "dst": d, "X": X, "dims": np.asarray(dims, np.int64),
           "smoothing": np.int64(smoothing), "heads": np.int64(heads), "nb": np.int64(nb)}
    if heads == 1:
        bundles = [Mo.make_bundle(model, dims, rng_seed=0, degree_smoothing=smoothing)]
        for l, w in enumerate(bundles[0].layers):
            for k, t in w.tensors.items():
                out[f"w{l}_{k}"] = t
            for k, v in w.scalars.items():
                out[f"w{l}_{k}"] = np.float64(v)
    else:
        bundles = None
        hb = {}
        for l in range(len(dims) - 1):
            for h in range(heads):
                bb = Mo.make_bundle("gat", [dims[l], dims[l + 1] // heads],
                                    rng_seed=head_seed(0, l, h, heads))
                hb[(l, h)] = bb
                out[f"w{l}_h{h}_W"] = bb.layers[0].tensors["W"]
                out[f"w{l}_h{h}_a"] = bb.layers[0].tensors["a"]

    def forward(tag):
        H = X
        for l in range(len(dims) - 1):
            if heads == 1:
                Hn, A, C = Mo.layer_embeddings(bundles[0], l, g, H)
            else:
                parts = [Mo.layer_embeddings(hb[(l, h)], 0, g, H) for h in range(heads)]
                Hn = np.concatenate([p[0] for p in parts], axis=1)
                A = np.concatenate([p[1] for p in parts], axis=1)
                C = np.stack([p[2] for p in parts], axis=1)
            out[f"{tag}_H{l + 1}"], out[f"{tag}_A{l}"], out[f"{tag}_C{l}"] = Hn, A, C
            H = Hn

    forward("boot")
    for b in range(nb):
        op, bs, bd, bt = mixed_batch(rng, g, n, B, p_reject=0.1, p_self=0.05)
        upd = to_updates(op, bs, bd, bt)
        g.apply_batch(upd)
        out[f"b{b}_op"], out[f"b{b}_src"], out[f"b{b}_dst"], out[f"b{b}_ts"] = op, bs, bd, bt
        forward(f"b{b}")
    np.savez_compressed(os.path.join(OUT, f"models_{name}.npz"), **out)
    print(f"models_{name}.npz written")


TABLE2 = (("pinsage", [12, 16, 8]), ("monet", [8, 12, 6]), ("commnet", [12, 16, 8]), ("ggcn", [12, 16, 8]),
          ("agnn", [12, 16, 8]))

if __name__ == "__main__":
    if sys.argv[1:] == ["table2"]:  # only the remaining Table II models (models.py:144-348)
        for name, dims in TABLE2:
            model_case(name, name, dims)
        sys.exit(0)
    graph_streams()
    coalesce_cases()
    model_case("gcn", "gcn", [16, 16, 8])
    model_case("gcn_raw", "gcn", [16, 16, 8], smoothing=False)
    model_case("graphsage", "graphsage", [12, 20, 8])
    model_case("gin", "gin", [16, 16, 8])
    model_case("gat", "gat", [16, 16, 8])
    model_case("gat_h4", "gat", [16, 16, 8], heads=4)
    for name, dims in TABLE2:
        model_case(name, name, dims)
