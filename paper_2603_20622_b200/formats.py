"""File formats either side of the hot path.

- NRTF: the reference's binary container for one 2-D float tensor
  (linalg.py:72-117): little-endian header magic "NRTF", u32 version 1, u8
  dtype code (0 float32, 1 float64), u64 rows, u64 cols, then the values
  row-major.
- Weights JSON (operators.py:325-378): {"model", "layers": [{"dims", "W",
  "a", "extra", "scalars"}]}.
- Engine checkpoint / resume (aggregate tensors as NRTF plus a
  JSON sidecar): the edge list, every layer's embeddings and un-normalised
  aggregates (and GAT attention sums), the weights, and the model config, so a
  long stream can restart without a bootstrap.
- Sharded checkpoint: one `rank<r>/` directory per rank
  holding that rank's edge shard, its replica layer inputs, its owned rows of
  the final layer / aggregates / contexts, and the same sidecar plus the world
  size; every rank writes and reads only its own directory (no collective).

Host-side IO only; nothing here is on the timed path.
"""

from __future__ import annotations

import json
import os
import struct

import numpy as np

from . import errors as E
from .models import LayerWeights

_NRTF = struct.Struct("<4sIBQQ")
_NRTF_MAGIC = b"NRTF"
_NRTF_CODES = {0: np.dtype("<f4"), 1: np.dtype("<f8")}


def write_tensor(path: str, array) -> None:
    """NRTF writer (linalg.py:84)."""
    a = np.asarray(array)
    if a.ndim != 2:
        raise E.ConfigError(f"NRTF holds 2-D tensors, got shape {a.shape}")
    codes = {np.dtype(np.float32): 0, np.dtype(np.float64): 1}
    if a.dtype not in codes:
        raise E.ConfigError(f"NRTF supports float32 / float64, got {a.dtype}")
    code = codes[a.dtype]
    with open(path, "wb") as fh:
        fh.write(_NRTF.pack(_NRTF_MAGIC, 1, code, a.shape[0], a.shape[1]))
        fh.write(np.ascontiguousarray(a, _NRTF_CODES[code]).tobytes())


def read_tensor(path: str) -> np.ndarray:
    """NRTF reader (linalg.py:99): validates magic, version, dtype and payload size."""
    with open(path, "rb") as fh:
        head = fh.read(_NRTF.size)
        if len(head) != _NRTF.size:
            raise E.ConfigError(f"{path}: truncated NRTF header")
        magic, version, code, rows, cols = _NRTF.unpack(head)
        if magic != _NRTF_MAGIC:
            raise E.ConfigError(f"{path}: not an NRTF file (magic {magic!r})")
        if version != 1:
            raise E.ConfigError(f"{path}: NRTF version {version} unsupported")
        if code not in _NRTF_CODES:
            raise E.ConfigError(f"{path}: NRTF dtype code {code} unknown")
        dt = _NRTF_CODES[code]
        body = fh.read()
    if len(body) != rows * cols * dt.itemsize:
        raise E.ConfigError(f"{path}: NRTF payload {len(body)} B, header says {rows * cols * dt.itemsize} B")
    return np.frombuffer(body, dtype=dt).reshape(rows, cols).astype(dt.newbyteorder("="))


def save_weights(bundle, path: str) -> None:
    """Weights JSON (operators.py:333) of a bundle (ours or a reference OperatorBundle)."""
    out = []
    for w in bundle.layers:
        t = {k: np.asarray(v) for k, v in w.tensors.items()}
        out.append({"dims": [int(w.in_dim), int(w.out_dim)],
                    "W": t.pop("W").tolist() if "W" in t else None,
                    "a": t.pop("a").tolist() if "a" in t else None,
                    "extra": {k: t[k].tolist() for k in sorted(t)},
                    "scalars": {k: float(v) for k, v in sorted(dict(w.scalars).items())}})
    with open(path, "w", encoding="ascii") as fh:
        json.dump({"model": bundle.model, "layers": out}, fh, indent=1)
        fh.write("\n")


def load_weights(path: str) -> dict:
    """Weights JSON reader (operators.py:350) -> {"model", "layers": [LayerWeights]}."""
    try:
        with open(path, "r", encoding="ascii") as fh:
            data = json.load(fh)
    except (OSError, json.JSONDecodeError) as exc:
        raise E.ConfigError(f"cannot read weights file {path}: {exc}") from exc
    if not isinstance(data, dict) or "model" not in data or "layers" not in data:
        raise E.ConfigError(f"{path}: weights file needs 'model' and 'layers'")
    layers, prev = [], None
    for i, e in enumerate(data["layers"]):
        dims = e.get("dims")
        if not (isinstance(dims, list) and len(dims) == 2):
            raise E.ConfigError(f"{path}: layer {i} has no [in, out] dims")
        d_in, d_out = int(dims[0]), int(dims[1])
        if prev is not None and d_in != prev:
            raise E.ConfigError(f"{path}: layer {i} input {d_in} does not follow output {prev}")
        prev = d_out
        t = {}
        for key in ("W", "a"):
            if e.get(key) is not None:
                t[key] = np.asarray(e[key], np.float64)
        for k, v in (e.get("extra") or {}).items():
            t[k] = np.asarray(v, np.float64)
        layers.append(LayerWeights(d_in, d_out, t, {k: float(v) for k, v in (e.get("scalars") or {}).items()}))
    return {"model": str(data["model"]), "layers": layers}


# ---------------------------------------------------------------- checkpoint / resume
def _edges_table(src, dst, ts) -> np.ndarray:
    """Edge list as an exact float64 NRTF table [src, dst, ts_hi, ts_lo]: ts = ts_hi * 2^32 +
    ts_lo with ts_hi the arithmetic high word and ts_lo in [0, 2^32), both exact in f64, so
    int64 timestamps (the reference keeps them as PMA uint64 payloads) survive any magnitude."""
    ts = np.asarray(ts, np.int64)
    return np.stack([np.asarray(src, np.float64), np.asarray(dst, np.float64),
                     (ts >> 32).astype(np.float64), (ts & 0xFFFFFFFF).astype(np.float64)], 1)


def _edges_from_table(e: np.ndarray):
    """Inverse of _edges_table (also reads the 3-column version-1 layout)."""
    src, dst = e[:, 0].astype(np.int64), e[:, 1].astype(np.int64)
    if e.shape[1] == 3:
        return src, dst, e[:, 2].astype(np.int64)
    return src, dst, (e[:, 2].astype(np.int64) << 32) | e[:, 3].astype(np.int64)


def _graph_knobs(g) -> dict:
    return {"slack": float(g.slack), "min_slack": int(g.min_slack),
            "reserve": None if g.reserve is None else int(g.reserve),
            "segment_slots": int(g.segment_slots), "density_bounds": list(g.density_bounds)}


def _graph_kw(side: dict) -> dict:
    kw = {k: side["graph"][k] for k in ("slack", "min_slack", "reserve", "segment_slots") if "graph" in side}
    if "graph" in side:
        kw["density_bounds"] = tuple(side["graph"]["density_bounds"])
    return kw


def save_checkpoint(engine, directory: str) -> None:
    """Snapshot an RTECEngine between batches: edges (exact float64 NRTF table, see
    _edges_table), per-layer H / S (/ GAT ctx) as float32 NRTF, weights JSON and a JSON
    sidecar (model config and the graph's slack / reserve knobs)."""
    os.makedirs(directory, exist_ok=True)
    src, dst, ts = engine.g.edges()
    write_tensor(os.path.join(directory, "edges.nrtf"), _edges_table(src, dst, ts))
    for l in range(engine.L + 1):
        write_tensor(os.path.join(directory, f"H{l}.nrtf"), engine.H[l].cpu().numpy())
    for l in range(engine.L):
        write_tensor(os.path.join(directory, f"S{l}.nrtf"), engine.S[l].cpu().numpy())
        if engine.ctx[l] is not None:
            write_tensor(os.path.join(directory, f"ctx{l}.nrtf"), engine.ctx[l].cpu().numpy())
    b = engine.b
    save_weights(b, os.path.join(directory, "weights.json"))
    side = {"format": "rtec-b200-checkpoint", "version": 2, "model": b.model, "dims": list(b.dims),
            "heads": int(b.heads), "degree_offset": float(b.degree_offset), "num_vertices": int(engine.n),
            "num_edges": int(len(src)), "graph": _graph_knobs(engine.g)}
    with open(os.path.join(directory, "checkpoint.json"), "w", encoding="ascii") as fh:
        json.dump(side, fh, indent=1)
        fh.write("\n")


def load_checkpoint(directory: str, **engine_kw):
    """Rebuild the graph and the engine state of `save_checkpoint` without a bootstrap."""
    import torch

    from .engine import RTECEngine
    from .graph import DynamicGraph
    from .models import make_bundle

    with open(os.path.join(directory, "checkpoint.json"), "r", encoding="ascii") as fh:
        side = json.load(fh)
    if side.get("format") != "rtec-b200-checkpoint":
        raise E.ConfigError(f"{directory}: not an rtec-b200 checkpoint")
    w = load_weights(os.path.join(directory, "weights.json"))
    bundle = make_bundle(side["model"], side["dims"], weights=w["layers"], heads=side["heads"],
                         degree_smoothing=side["degree_offset"] != 0.0)
    e = _edges_from_table(read_tensor(os.path.join(directory, "edges.nrtf")))
    g = DynamicGraph.from_edges(side["num_vertices"], e, **_graph_kw(side))
    X = read_tensor(os.path.join(directory, "H0.nrtf"))
    eng = RTECEngine(bundle, g, X, bootstrap=False, **engine_kw)
    for l in range(1, eng.L + 1):
        eng.H[l].copy_(torch.from_numpy(read_tensor(os.path.join(directory, f"H{l}.nrtf"))))
    for l in range(eng.L):
        eng.S[l].copy_(torch.from_numpy(read_tensor(os.path.join(directory, f"S{l}.nrtf"))))
        if eng.ctx[l] is not None:
            eng.ctx[l].copy_(torch.from_numpy(read_tensor(os.path.join(directory, f"ctx{l}.nrtf"))))
        if eng.Z[l] is not None:  # GAT projections are a function of H: recompute them
            eng.refresh_projection(l)
    return eng


# ---------------------------------------------------------------- sharded checkpoint
def _rank_dir(directory: str, rank: int) -> str:
    return os.path.join(directory, f"rank{rank:04d}")


def save_sharded_checkpoint(engine, directory: str) -> None:
    """Per-rank snapshot of a ShardedRTECEngine between batches (call on every rank): the
    shard's edges (global ids) and the OWNED rows of every layer; ghost rows are derived
    (their owners refresh them on resume)."""
    r, P = engine.comm.rank, engine.comm.world
    d = _rank_dir(directory, r)
    os.makedirs(d, exist_ok=True)
    src, dst, ts = engine.shard_edges()  # the edges whose destination this rank owns
    write_tensor(os.path.join(d, "edges.nrtf"), _edges_table(src, dst, ts))
    no = engine.n_own
    for l in range(engine.L + 1):
        write_tensor(os.path.join(d, f"H{l}.nrtf"), engine.H[l][:no].cpu().numpy())
    for l in range(engine.L):
        write_tensor(os.path.join(d, f"S{l}.nrtf"), engine.S[l].cpu().numpy())
        if engine.ctx[l] is not None:
            write_tensor(os.path.join(d, f"ctx{l}.nrtf"), engine.ctx[l].cpu().numpy())
    b = engine.b
    save_weights(b, os.path.join(d, "weights.json"))
    side = {"format": "rtec-b200-sharded-checkpoint", "version": 3, "model": b.model, "dims": list(b.dims),
            "heads": int(b.heads), "degree_offset": float(b.degree_offset), "num_vertices": int(engine.n_glob),
            "world_size": int(P), "rank": int(r), "num_edges_shard": int(len(src)), "owned_rows": int(no)}
    with open(os.path.join(d, "checkpoint.json"), "w", encoding="ascii") as fh:
        json.dump(side, fh, indent=1)
        fh.write("\n")


def load_sharded_checkpoint(directory: str, comm, **engine_kw):
    """Rebuild this rank's ShardedRTECEngine from `save_sharded_checkpoint` (collective:
    ghosts are announced to their owners, who refresh their rows and degrees).  The world
    size must match."""
    import torch

    from .models import make_bundle
    from .shard import ShardedRTECEngine

    d = _rank_dir(directory, comm.rank)
    with open(os.path.join(d, "checkpoint.json"), "r", encoding="ascii") as fh:
        side = json.load(fh)
    if side.get("format") != "rtec-b200-sharded-checkpoint" or int(side.get("version", 0)) < 3:
        raise E.ConfigError(f"{d}: not an rtec-b200 sharded checkpoint (version 3)")
    if int(side["world_size"]) != comm.world or int(side["rank"]) != comm.rank:
        raise E.ConfigError(f"{d}: saved by rank {side['rank']} of {side['world_size']}, "
                            f"loading on rank {comm.rank} of {comm.world}")
    w = load_weights(os.path.join(d, "weights.json"))
    bundle = make_bundle(side["model"], side["dims"], weights=w["layers"], heads=side["heads"],
                         degree_smoothing=side["degree_offset"] != 0.0)
    e = _edges_from_table(read_tensor(os.path.join(d, "edges.nrtf")))
    X = read_tensor(os.path.join(d, "H0.nrtf"))
    eng = ShardedRTECEngine(bundle, side["num_vertices"], e, X, comm, bootstrap=False, shard_edges=True,
                            **engine_kw)
    no = eng.n_own
    for l in range(1, eng.L + 1):
        eng.H[l][:no].copy_(torch.from_numpy(read_tensor(os.path.join(d, f"H{l}.nrtf"))))
    for l in range(eng.L):
        eng.S[l].copy_(torch.from_numpy(read_tensor(os.path.join(d, f"S{l}.nrtf"))))
        if eng.ctx[l] is not None:
            eng.ctx[l].copy_(torch.from_numpy(read_tensor(os.path.join(d, f"ctx{l}.nrtf"))))
    if eng.L > 1:
        eng._refresh_ghosts(list(range(1, eng.L)))
    for l in range(eng.L):
        eng.refresh_projection(l)  # GAT Z / el / er of every local row from H^l
    return eng
