"""Operator bundles for the reference model zoo (Table II).

Mirrors `streamgnn/models.py`: the four north-star models (gcn, graphsage,
gin, gat) and the rest of Table II (pinsage, monet, commnet, ggcn, agnn;
models.py:144-348).  `make_bundle(model, dims, *, dtype, rng_seed,
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
PINSAGE, MONET, COMMNET, GGCN, AGNN = "pinsage", "monet", "commnet", "ggcn", "agnn"
MODELS = (GCN, GRAPHSAGE, GIN, GAT, GIN_MAX, PINSAGE, MONET, COMMNET, GGCN, AGNN)
GIN_FAMILY = (GIN, GIN_MAX)
PROJECTED = (PINSAGE, MONET, GGCN)  # per-source projection cache (rtec_project) besides GAT's
REFERENCE_ONLY = ()


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

    @property
    def projected(self) -> bool:
        """Layers keep a per-vertex projection of H^l (GAT Z/el/er, PinSAGE / MoNet
        payloads, G-GCN gates) that must follow every changed row."""
        return self.model == GAT or self.model in PROJECTED

    def proj_width(self, l: int) -> int:
        d = self.layers[l].in_dim
        return {PINSAGE: d, MONET: 1, GGCN: 2 * d}.get(self.model, 0)

    def update_width(self, l: int) -> int:
        """Columns of the update input: [h_v ; a_v] for PinSAGE / CommNet, the scalar
        aggregate for MoNet, a_v otherwise (rtec_layer_t.d_k)."""
        d = self.layers[l].in_dim
        return {PINSAGE: 2 * d, COMMNET: 2 * d, MONET: 1}.get(self.model, self.agg_dims[l])


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
    elif name == PINSAGE:  # models.py:144-155
        layers = []
        for i, o in pairs:
            W = _mat(rng, o, 2 * i, dt)
            Q = _mat(rng, i, i, dt)
            layers.append(LayerWeights(i, o, {"W": W, "Q": Q, "q": _vec(rng, i, i, dt)}, {"alpha": 1.0}))
    elif name == MONET:  # models.py:203-216
        layers = []
        for i, o in pairs:
            seed_mat = rng.uniform(-1.0, 1.0, (i, i)) / math.sqrt(i)
            kernel = (-(seed_mat @ seed_mat.T) / i).astype(dt)
            W = _mat(rng, o, 1, dt)
            layers.append(LayerWeights(i, o, {"W": W, "Wq": kernel, "mu": rng.uniform(-1.0, 1.0, i).astype(dt)}))
    elif name == COMMNET:  # models.py:235-239
        layers = []
        for i, o in pairs:
            W = _mat(rng, o, i, dt)
            layers.append(LayerWeights(i, o, {"W": W, "W2": _mat(rng, o, i, dt)}))
    elif name == GGCN:  # models.py:290-299
        layers = []
        for i, o in pairs:
            W = _mat(rng, o, i, dt)
            Ws = _mat(rng, i, i, dt)
            layers.append(LayerWeights(i, o, {"W": W, "Wg_src": Ws, "Wg_dst": _mat(rng, i, i, dt)}))
    elif name == AGNN:  # models.py:320-324
        layers = []
        for i, o in pairs:
            W = _mat(rng, o, i, dt)
            layers.append(LayerWeights(i, o, {"W": W}, {"beta": float(rng.uniform(0.5, 1.5))}))
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
    if name in GIN_FAMILY or name == COMMNET:  # :191-200, :240-249
        return Bundle(name, tuple(layers), dt, tuple(dims[:-1]), "none")
    if name == PINSAGE:  # :165-175
        return Bundle(name, tuple(layers), dt, tuple(dims[:-1]), "count")
    if name == MONET:  # :218-227 (scalar aggregate)
        return Bundle(name, tuple(layers), dt, (1,) * len(pairs), "none")
    if name in (GGCN, AGNN):  # :307-317, :337-347
        return Bundle(name, tuple(layers), dt, tuple(dims[:-1]), "none", dest_dependent=True)
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
