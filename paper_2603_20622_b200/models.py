"""Operator bundles for the hot-path models (gcn, graphsage, gin, gat).

Mirrors the reference model zoo (`streamgnn/models.py`) for the four models
on the north-star path: `make_bundle(model, dims, *, dtype, rng_seed,
weights, degree_smoothing)` draws weights with the same RNG sequence as
models.py:56-63 / :88-287 / :364-384, so a given seed produces bit-identical
f64 weights; the engine uploads fp32 copies.  A reference `OperatorBundle`
(duck-typed: `.model`, `.layers[i].tensors`, `.scalars`) can be passed to
`from_reference` instead.  Custom operator callables have no GPU kernels and
raise UnsupportedModel.

Flags follow the reference builders: ctx kinds count/none/sum,
`dest_dependent` (gat), `src_degree_dependent` (gcn), `agg_dims` = dims[:-1]
(aggregate then transform) or dims[1:] for gat (transform then aggregate).
Multi-head GAT (beyond the reference): head h of layer l uses
the weights of a single-head reference GAT bundle of width d_out/heads with
rng_seed = head_seed(seed, l, h, heads); heads are concatenated.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Mapping, Sequence

import numpy as np

from . import errors as E

GCN, GRAPHSAGE, GIN, GAT = "gcn", "graphsage", "gin", "gat"
# GIN with an elementwise-max aggregator (configs[3] "GIN (max/sum agg)"); the
# reference has no max aggregator, so this one is pinned only by the oracle's
# restated full recompute (SURVEY §8(c) "Unpinned by the reference").
GIN_MAX = "gin_max"
MODELS = (GCN, GRAPHSAGE, GIN, GAT, GIN_MAX)
GIN_FAMILY = (GIN, GIN_MAX)
REFERENCE_ONLY = ("pinsage", "monet", "commnet", "ggcn", "agnn")


@dataclass(frozen=True)
class LayerWeights:  # operators.py:42-47
    in_dim: int
    out_dim: int
    tensors: Mapping[str, np.ndarray] = field(default_factory=dict)
    scalars: Mapping[str, float] = field(default_factory=dict)


@dataclass(frozen=True)
class Bundle:
    model: str
    layers: tuple
    dtype: np.dtype
    agg_dims: tuple
    ctx_kind: str
    dest_dependent: bool = False
    src_degree_dependent: bool = False
    degree_offset: float = 1.0
    heads: int = 1

    @property
    def num_layers(self) -> int:
        return len(self.layers)

    @property
    def dims(self) -> tuple:
        return tuple([self.layers[0].in_dim] + [w.out_dim for w in self.layers])

    @property
    def has_nbr_ctx(self) -> bool:
        return self.ctx_kind != "none"

    def empty_context(self) -> float:  # operators.py:99-100
        return 0.0 if self.has_nbr_ctx else 1.0


def _mat(rng, rows, cols, dtype):  # models.py:56-58
    b = 1.0 / math.sqrt(cols)
    return rng.uniform(-b, b, (rows, cols)).astype(dtype)


def _vec(rng, size, fan_in, dtype):  # models.py:61-63
    b = 1.0 / math.sqrt(fan_in)
    return rng.uniform(-b, b, size).astype(dtype)


def head_seed(seed: int, layer: int, head: int, heads: int) -> int:
    return int(seed) * 1009 + 1 + layer * heads + head


def _pairs(dims):  # models.py:66-69
    if len(dims) < 2 or any(d < 1 for d in dims):
        raise E.ConfigError(f"need at least [in, out] positive dims, got {list(dims)}")
    return [(dims[i], dims[i + 1]) for i in range(len(dims) - 1)]


def make_bundle(model: str, dims: Sequence[int], *, dtype=np.float64, rng_seed: int = 0,
                weights: Sequence | None = None, degree_smoothing: bool = True, heads: int = 1) -> Bundle:
    """models.py:364-384 for the hot-path models."""
    name = str(model).lower()
    if name in REFERENCE_ONLY:
        raise E.UnsupportedModel(f"model {model!r} has no B200 kernels (hot path covers {', '.join(MODELS)})")
    if name not in MODELS:
        raise E.UnsupportedModel(f"unknown model {model!r}; known: {', '.join(MODELS)}")
    dims = [int(d) for d in dims]
    pairs = _pairs(dims)
    dt = np.dtype(dtype)
    rng = np.random.default_rng(rng_seed)
    if weights is not None:
        if len(weights) != len(pairs):
            raise E.ConfigError(f"weights have {len(weights)} layers, dims imply {len(pairs)}")
        layers = []
        for w, (i, o) in zip(weights, pairs):
            if (w.in_dim, w.out_dim) != (i, o):
                raise E.ConfigError(f"weights dims ({w.in_dim},{w.out_dim}) != requested ({i},{o})")
            layers.append(LayerWeights(i, o, {k: np.asarray(t, dt) for k, t in w.tensors.items()}, dict(w.scalars)))
    elif name in (GCN, GRAPHSAGE):  # models.py:88-96, :124-128
        layers = [LayerWeights(i, o, {"W": _mat(rng, o, i, dt)}) for i, o in pairs]
    elif name in GIN_FAMILY:  # models.py:178-183 (gin_max: same draws)
        layers = []
        for i, o in pairs:
            W = _mat(rng, o, i, dt)
            layers.append(LayerWeights(i, o, {"W": W, "W2": _mat(rng, o, o, dt)}))
    else:  # GAT models.py:256-260
        layers = []
        for li, (i, o) in enumerate(pairs):
            if heads == 1:
                W = _mat(rng, o, i, dt)
                layers.append(LayerWeights(i, o, {"W": W, "a": _vec(rng, 2 * o, 2 * o, dt)}))
            else:
                if o % heads:
                    raise E.ShapeError(f"width {o} not divisible by {heads} heads")
                hs = [make_bundle(GAT, [i, o // heads], dtype=dt, rng_seed=head_seed(rng_seed, li, h, heads)).layers[0]
                      for h in range(heads)]
                layers.append(LayerWeights(i, o, {"W": np.concatenate([h.tensors["W"] for h in hs], 0),
                                                  "a": np.stack([h.tensors["a"] for h in hs], 0)}))
    if name == GCN:  # models.py:110-121
        return Bundle(name, tuple(layers), dt, tuple(dims[:-1]), "count", src_degree_dependent=True,
                      degree_offset=1.0 if degree_smoothing else 0.0)
    if name == GRAPHSAGE:  # :131-141
        return Bundle(name, tuple(layers), dt, tuple(dims[:-1]), "count")
    if name in GIN_FAMILY:  # :191-200
        return Bundle(name, tuple(layers), dt, tuple(dims[:-1]), "none")
    return Bundle(name, tuple(layers), dt, tuple(dims[1:]), "sum", dest_dependent=True, heads=int(heads))


def from_reference(ref_bundle, heads: int = 1) -> Bundle:
    """Adopt a reference streamgnn OperatorBundle (operators.py:63-181) by value."""
    name = str(getattr(ref_bundle, "model", "")).lower()
    if name not in MODELS:
        raise E.UnsupportedModel(f"model {name!r} has no B200 kernels")
    dims = list(ref_bundle.dims)
    lw = [LayerWeights(w.in_dim, w.out_dim, dict(w.tensors), dict(w.scalars)) for w in ref_bundle.layers]
    smoothing = True
    if name == GCN:
        smoothing = float(ref_bundle.layers[0].scalars.get("degree_offset", 1.0)) != 0.0
    return make_bundle(name, dims, dtype=np.dtype(ref_bundle.dtype), weights=lw, degree_smoothing=smoothing,
                       heads=heads)
