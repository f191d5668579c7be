"""Oracle restatement of the reference model zoo -- TEST INFRASTRUCTURE ONLY.

Restates `streamgnn/models.py` for the four hot-path models (gcn, graphsage,
gin, gat) and the rest of Table II (pinsage,
monet, commnet, ggcn, agnn; models.py:144-348):

- `make_bundle` draws weights with the reference's RNG sequence
  (models.py:56-63 `_mat`/`_vec`, builders :88-287, `make_bundle` :364-384),
  so the same seed yields bit-identical f64 weights;
- `layer_full` is a vectorised `layer_embeddings` (models.py:461-477) whose
  per-vertex math is `vertex_aggregate` (models.py:431-458) with the operator
  definitions of each builder.  Context arrays follow the reference: count ->
  in-degree, sum -> attention sum, none -> 1.0; an empty neighbourhood gives a
  zero aggregate and `empty_context()` (operators.py:99-100).

Multi-head GAT (not in the reference): head h of layer l is a
single-head reference GAT layer of width d_out/heads whose weights come from
`make_bundle('gat', [d_in, d_out/heads], rng_seed=head_seed(seed, l, h, heads))`;
heads are concatenated.  heads=1 is exactly the reference bundle.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp

GCN, SAGE, GIN, GAT = "gcn", "graphsage", "gin", "gat"
# GIN with an elementwise-max aggregator: NOT in the reference (no max
# aggregator exists in models.py); restated here as the full recompute
# a_v = max_{u in N_in(v)} h_u (0 for an empty neighbourhood), GIN update.
GIN_MAX = "gin_max"
PINSAGE, MONET, COMMNET, GGCN, AGNN = "pinsage", "monet", "commnet", "ggcn", "agnn"
MODELS = (GCN, SAGE, GIN, GAT, GIN_MAX, PINSAGE, MONET, COMMNET, GGCN, AGNN)
PAYLOAD_MODELS = (PINSAGE, MONET)  # message = a function of h_u alone (per-source payload row)
EDGE_MODELS = (GGCN, AGNN)  # message reads both endpoints (dest-dependent, no context)


def _mat(rng, rows, cols):  # models.py:56-58
    b = 1.0 / math.sqrt(cols)
    return rng.uniform(-b, b, (rows, cols)).astype(np.float64)


def _vec(rng, size, fan_in):  # models.py:61-63
    b = 1.0 / math.sqrt(fan_in)
    return rng.uniform(-b, b, size).astype(np.float64)


def head_seed(seed: int, layer: int, head: int, heads: int) -> int:
    return int(seed) * 1009 + 1 + layer * heads + head


@dataclass
class OracleBundle:
    model: str
    dims: tuple
    layers: list  # per layer: dict of f64 arrays (W, W2, a[heads, 2*dh], Wh[heads, dh, din], ...) + scalars
    degree_offset: float = 1.0
    heads: int = 1
    ctx_kind: str = "none"
    dest_dependent: bool = False
    src_degree_dependent: bool = False
    agg_dims: tuple = field(default_factory=tuple)

    @property
    def num_layers(self) -> int:
        return len(self.dims) - 1

    def empty_context(self) -> float:  # operators.py:99-100
        return 0.0 if self.ctx_kind != "none" else 1.0


def make_bundle(model, dims, *, rng_seed=0, degree_smoothing=True, heads=1) -> OracleBundle:
    model = str(model).lower()
    dims = tuple(int(d) for d in dims)
    if model not in MODELS:
        raise ValueError(f"unknown model {model!r}")
    if len(dims) < 2 or any(d < 1 for d in dims):  # models.py:66-69
        raise ValueError(f"need at least [in, out] positive dims, got {list(dims)}")
    pairs = [(dims[i], dims[i + 1]) for i in range(len(dims) - 1)]
    rng = np.random.default_rng(rng_seed)  # models.py:382
    layers = []
    if model in (GCN, SAGE):  # models.py:88-96, :124-128
        for i, o in pairs:
            layers.append({"W": _mat(rng, o, i)})
    elif model in (GIN, GIN_MAX):  # models.py:178-183 (W then W2, layer by layer)
        for i, o in pairs:
            W = _mat(rng, o, i)
            W2 = _mat(rng, o, o)
            layers.append({"W": W, "W2": W2})
    elif model == PINSAGE:  # models.py:144-155: W [o, 2i], Q [i, i], q [i]; alpha = 1
        for i, o in pairs:
            W = _mat(rng, o, 2 * i)
            Q = _mat(rng, i, i)
            layers.append({"W": W, "Q": Q, "q": _vec(rng, i, i), "alpha": 1.0})
    elif model == MONET:  # models.py:203-216: negative-definite kernel, W [o, 1], mu [i]
        for i, o in pairs:
            seed_mat = rng.uniform(-1.0, 1.0, (i, i)) / math.sqrt(i)
            Wq = -(seed_mat @ seed_mat.T) / i
            W = _mat(rng, o, 1)
            layers.append({"W": W, "Wq": Wq, "mu": rng.uniform(-1.0, 1.0, i)})
    elif model == COMMNET:  # models.py:235-239: W [o, i], W2 [o, i]
        for i, o in pairs:
            W = _mat(rng, o, i)
            layers.append({"W": W, "W2": _mat(rng, o, i)})
    elif model == GGCN:  # models.py:290-299: W [o, i], Wg_src [i, i], Wg_dst [i, i]
        for i, o in pairs:
            W = _mat(rng, o, i)
            Ws = _mat(rng, i, i)
            layers.append({"W": W, "Wg_src": Ws, "Wg_dst": _mat(rng, i, i)})
    elif model == AGNN:  # models.py:320-324: W [o, i], beta ~ U(0.5, 1.5)
        for i, o in pairs:
            W = _mat(rng, o, i)
            layers.append({"W": W, "beta": float(rng.uniform(0.5, 1.5))})
    else:  # GAT models.py:256-260
        if heads == 1:
            for i, o in pairs:
                W = _mat(rng, o, i)
                a = _vec(rng, 2 * o, 2 * o)
                layers.append({"Wh": W[None], "a": a[None]})
        else:
            for li, (i, o) in enumerate(pairs):
                if o % heads:
                    raise ValueError(f"width {o} not divisible by {heads} heads")
                dh = o // heads
                Ws, As = [], []
                for h in range(heads):
                    hb = make_bundle(GAT, [i, dh], rng_seed=head_seed(rng_seed, li, h, heads))
                    Ws.append(hb.layers[0]["Wh"][0])
                    As.append(hb.layers[0]["a"][0])
                layers.append({"Wh": np.stack(Ws), "a": np.stack(As)})
    b = OracleBundle(model=model, dims=dims, layers=layers, heads=heads if model == GAT else 1)
    if model == GCN:  # models.py:110-121
        b.degree_offset = 1.0 if degree_smoothing else 0.0
        b.ctx_kind, b.src_degree_dependent = "count", True
        b.agg_dims = dims[:-1]
    elif model == SAGE:  # :131-141
        b.ctx_kind = "count"
        b.agg_dims = dims[:-1]
    elif model in (GIN, GIN_MAX, COMMNET):  # :191-200, :240-249
        b.ctx_kind = "none"
        b.agg_dims = dims[:-1]
    elif model == PINSAGE:  # :165-175
        b.ctx_kind = "count"
        b.agg_dims = dims[:-1]
    elif model == MONET:  # :218-227 (scalar aggregate)
        b.ctx_kind = "none"
        b.agg_dims = (1,) * (len(dims) - 1)
    elif model in EDGE_MODELS:  # :307-317, :337-347
        b.ctx_kind, b.dest_dependent = "none", True
        b.agg_dims = dims[:-1]
    else:  # GAT :276-287
        b.ctx_kind, b.dest_dependent = "sum", True
        b.agg_dims = dims[1:]
    return b


# ---- per-model operators (vectorised over rows) ----


def leaky(x):  # models.py:272-273 (slope 0.2)
    return np.where(x < 0.0, 0.2 * x, x)


def gat_project(b: OracleBundle, l: int, H):
    """f_nn = W h (models.py:279) and the two logit halves (models.py:269-271).

    Returns z [rows, heads, dh], el (destination half a[:o]·Wh) and er (source
    half a[o:]·Wh), both [rows, heads].
    """
    Wh, a = b.layers[l]["Wh"], b.layers[l]["a"]
    dh = Wh.shape[1]
    z = np.einsum("hoi,ri->rho", Wh, H)
    el = np.einsum("rho,ho->rh", z, a[:, :dh])
    er = np.einsum("rho,ho->rh", z, a[:, dh:])
    return z, el, er


def sigmoid(x):  # linalg.py:46-52 (two-branch form)
    pos = 1.0 / (1.0 + np.exp(-np.maximum(x, 0)))
    ex = np.exp(np.minimum(x, 0))
    return np.where(x >= 0, pos, ex / (1.0 + ex))


def payload(b: OracleBundle, l: int, H):
    """Per-source payload of the source-only models (ms_local * f_nn):
    PinSAGE alpha relu(Q h + q) (models.py:157-159), MoNet exp(0.5 d^T Wq d),
    d = h - mu, as a width-1 row (models.py:211-213)."""
    L = b.layers[l]
    if b.model == PINSAGE:
        return L["alpha"] * np.maximum(H @ L["Q"].T + L["q"], 0.0)
    diff = H - L["mu"]
    return np.exp(0.5 * np.einsum("ri,ri->r", diff, diff @ L["Wq"].T))[:, None]


def edge_message(b: OracleBundle, l: int, Hu, Hv):
    """Dest-dependent payload rows for edges (u, v): G-GCN sigmoid(Wg_src h_u +
    Wg_dst h_v) * h_u (models.py:301-305); A-GNN beta cos(h_u, h_v) h_u, zero
    when either norm is zero (models.py:326-331)."""
    L = b.layers[l]
    if b.model == GGCN:
        return sigmoid(Hu @ L["Wg_src"].T + Hv @ L["Wg_dst"].T) * Hu
    nu = np.linalg.norm(Hu, axis=1)
    nv = np.linalg.norm(Hv, axis=1)
    ok = (nu > 0) & (nv > 0)
    cos = np.where(ok, np.einsum("ri,ri->r", Hu, Hv) / np.where(ok, nu * nv, 1.0), 0.0)
    return (L["beta"] * cos)[:, None] * Hu


def update(b: OracleBundle, l: int, h_v, a_v):
    """apply_update (operators.py:180) for the builders' `update`."""
    L = b.layers[l]
    if b.model in (GCN, SAGE, MONET, GGCN, AGNN):  # models.py:107-108, :137, :225, :315, :345: relu(W a)
        return np.maximum(a_v @ L["W"].T, 0.0)
    if b.model == PINSAGE:  # models.py:161-162: relu(W [h_v ; a_v])
        return np.maximum(np.concatenate([h_v, a_v], 1) @ L["W"].T, 0.0)
    if b.model == COMMNET:  # models.py:247: W h_v + W2 a_v (no activation)
        return h_v @ L["W"].T + a_v @ L["W2"].T
    if b.model in (GIN, GIN_MAX):  # models.py:187-189: W2 relu(W (h_v + a_v))
        return np.maximum((h_v + a_v) @ L["W"].T, 0.0) @ L["W2"].T
    # GAT models.py:282: elu(a) (linalg.py:41-43)
    return np.where(a_v >= 0, a_v, np.expm1(np.minimum(a_v, 0)))


def compose(b: OracleBundle, ctx, x):
    """ms_cbn (operators.py:135-144), row-wise; ctx broadcast per row(/head)."""
    if b.model == GCN:  # models.py:101-102
        return x / np.sqrt(ctx + b.degree_offset)[..., None]
    if b.model in (SAGE, GAT, PINSAGE):  # models.py:135, :280, :169
        return x / ctx[..., None]
    return x


def strip(b: OracleBundle, ctx, x):
    """ms_cbn_inv (operators.py:146-155)."""
    if b.model == GCN:  # models.py:104-105
        return x * np.sqrt(ctx + b.degree_offset)[..., None]
    if b.model in (SAGE, GAT, PINSAGE):
        return x * ctx[..., None]
    return x


def src_coeff(b: OracleBundle, out_deg):
    """ms_local for the degree-only models (models.py:98-99, :133, :193)."""
    if b.model == GCN:
        return 1.0 / np.sqrt(out_deg.astype(np.float64) + b.degree_offset)
    return np.ones(out_deg.shape, np.float64)


def layer_full(b: OracleBundle, l: int, g, H_prev, rows=None):
    """Vectorised layer_embeddings (models.py:461-477) for all or `rows` vertices.

    Returns (H_next, A, C) where A is the composed aggregate a_v and C the
    neighbourhood context, exactly as the reference returns them.
    """
    n = g.n
    indptr, srcs = g.in_csr()
    if rows is None:
        rows = np.arange(n)
    rows = np.asarray(rows, np.int64)
    cnt = indptr[rows + 1] - indptr[rows]
    # edge list of the selected destinations (ascending source inside each row)
    e_row = np.repeat(np.arange(rows.size), cnt)
    starts = np.repeat(indptr[rows], cnt)
    e_src = srcs[starts + (np.arange(e_row.size) - np.repeat(np.cumsum(cnt) - cnt, cnt))]
    heads = b.heads
    if b.model == GAT:
        z, el, er = gat_project(b, l, H_prev)
        dh = z.shape[2]
        logit = el[rows][e_row] + er[e_src]  # [E, heads]
        at = np.exp(leaky(logit))
        C = np.zeros((rows.size, heads))
        np.add.at(C, e_row, at)
        S = np.zeros((rows.size, heads, dh))
        for h in range(heads):
            M = sp.csr_matrix((at[:, h], (e_row, e_src)), shape=(rows.size, n))
            S[:, h, :] = M @ z[:, h, :]
        empty = cnt == 0
        Cs = np.where(empty[:, None], 1.0, C)
        A = (S / Cs[..., None]).reshape(rows.size, heads * dh)
        A[empty] = 0.0
        C[empty] = 0.0
        C = C[:, 0] if heads == 1 else C
    elif b.model == GIN_MAX:
        S = np.full((rows.size, H_prev.shape[1]), -np.inf)
        np.maximum.at(S, e_row, H_prev[e_src])
        empty = cnt == 0
        S[empty] = 0.0
        A = S
        C = np.ones(rows.size)
    elif b.model in EDGE_MODELS:
        msg = edge_message(b, l, H_prev[e_src], H_prev[rows][e_row])
        S = np.zeros((rows.size, H_prev.shape[1]))
        np.add.at(S, e_row, msg)
        A = S
        C = np.ones(rows.size)
        A[cnt == 0] = 0.0
    else:
        if b.model in PAYLOAD_MODELS:
            H_msg = payload(b, l, H_prev)
        else:
            H_msg = H_prev
        with np.errstate(divide="ignore"):  # raw GCN: sources with no out-edges never appear
            c = src_coeff(b, g.out_deg)
        M = sp.csr_matrix((c[e_src], (e_row, e_src)), shape=(rows.size, n))
        S = M @ H_msg
        empty = cnt == 0
        if b.ctx_kind == "count":
            C = cnt.astype(np.float64)
            A = compose(b, np.where(empty, 1.0, C), S)
        else:
            C = np.ones(rows.size)
            A = S
        A[empty] = 0.0
        C[empty] = b.empty_context()
    Hn = update(b, l, H_prev[rows], A)
    return Hn, A, C


def reference_embeddings(b: OracleBundle, g, X):
    """models.py:487-492: final-layer embeddings from scratch."""
    H = np.asarray(X, np.float64)
    for l in range(b.num_layers):
        H = layer_full(b, l, g, H)[0]
    return H
