"""Oracle incremental RTEC engine -- TEST INFRASTRUCTURE ONLY.

The reference ships no engine (SPEC.md:296-509 frontier/state_cache/engines are
absent).  This restates, over the oracle graph/model modules:

- Alg. 4 computation-graph construction with the
  every-layer source-degree rule of SURVEY §8(a)-F1 (SPEC.md:311-319 text is
  unsound for GCN, SPEC.md:352 makes soundness the arbiter):
      Dg = {u : old_out(u) != new_out(u)} if src_degree_dependent else {}
      S(l) = Dg ∪ V_chg(l-1),  V_chg(0) = {}
      E_curr(l) = I ∪ D ∪ {(u, w) in G_post : u in S(l)}   (one entry per edge)
      V_dst(l) = dst(E_curr(l)),  R(l) = V_dst(l) ∩ V_chg(l-1) if dest_dependent
      V_chg(l) = V_dst(l)
- Alg. 1 / SPEC run_incremental for
  v in V_dst(l) \\ R(l): signed messages (-old for edges not inserted, +new
  for edges not deleted), context_update (operators.py:123-133), strip with
  the OLD context (operators.py:146), combine_signed (operators.py:167-178),
  compose with the NEW context (operators.py:135), update (operators.py:180).
  Zero new in-degree -> zero aggregate + empty_context; zero
  old in-degree -> stripped aggregate 0.
- Alg. 3 for GAT: at_sum is the context, old attention
  terms rebuilt from the pre-batch embeddings (state_cache
  design decision "reconstruct from logged old state").
- v in R(l) -> full-neighbourhood recompute on G_post (`vertex_aggregate`,
  models.py:431).

State: per layer H^l (all vertices), composed aggregate A^l and context C^l,
exactly the triple `layer_embeddings` returns (models.py:461-477).  The
DeltaLog is the pre-batch copy of H^l, valid for one batch.
"""

from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from . import models as M
from .graph import OP_DELETE, OP_INSERT, OracleGraph


class OracleEngine:
    def __init__(self, bundle: M.OracleBundle, graph: OracleGraph, X):
        self.b = bundle
        self.g = graph
        self.X = np.asarray(X, np.float64)
        self.bootstrap()

    # SPEC bootstrap == layer_embeddings per layer
    def bootstrap(self):
        self.H = [self.X]
        self.A, self.C = [], []
        for l in range(self.b.num_layers):
            Hn, A, C = M.layer_full(self.b, l, self.g, self.H[l])
            self.H.append(Hn)
            self.A.append(A)
            self.C.append(C)

    def step(self, op, src, dst, ts):
        b, g = self.b, self.g
        n = g.n
        L = b.num_layers
        old_in = g.in_deg.copy()
        old_out = g.out_deg.copy()
        status, deltas = g.apply_batch(op, src, dst, ts)
        op = np.asarray(op, np.int64)
        src = np.asarray(src, np.int64)
        dst = np.asarray(dst, np.int64)
        ap = status.astype(bool)
        Is, Id = src[ap & (op == OP_INSERT)], dst[ap & (op == OP_INSERT)]
        Ds, Dd = src[ap & (op == OP_DELETE)], dst[ap & (op == OP_DELETE)]
        new_in, new_out = g.in_deg, g.out_deg
        nn = np.uint64(max(n, 1))
        e_src = (g.out_keys // nn).astype(np.int64)  # G_post edges
        e_dst = (g.out_keys % nn).astype(np.int64)
        is_ins = np.isin(g.out_keys, Is.astype(np.uint64) * nn + Id.astype(np.uint64))
        Dg = (old_out != new_out) if b.src_degree_dependent else np.zeros(n, bool)
        chg_prev = np.zeros(n, bool)
        frontier = []
        H_old = [self.H[0]]
        for l in range(L):
            S = Dg | chg_prev
            vc = S[e_src] & ~is_ins
            vcs, vcd = e_src[vc], e_dst[vc]
            vdst = np.zeros(n, bool)
            vdst[vcd] = True
            vdst[Id] = True
            vdst[Dd] = True
            R = (vdst & chg_prev) if b.dest_dependent else np.zeros(n, bool)
            if b.model == M.GIN_MAX:  # max has no inverse: the oracle recomputes every affected row
                R = vdst.copy()
            inc = vdst & ~R
            frontier.append(
                dict(vdst=np.flatnonzero(vdst), R=np.flatnonzero(R),
                     n_ecurr=int(vcs.size + Is.size + Ds.size), n_src=int(S.sum()))
            )
            A_new, C_new = self.A[l].copy(), self.C[l].copy()
            h_new, h_old = self.H[l], H_old[l]
            # restrict edge lists to incremental destinations
            m_vc, m_i, m_d = inc[vcd], inc[Id], inc[Dd]
            rows = np.flatnonzero(inc)
            if rows.size:
                self._incremental(l, rows, vcs[m_vc], vcd[m_vc], Is[m_i], Id[m_i], Ds[m_d], Dd[m_d],
                                  h_new, h_old, old_in, old_out, A_new, C_new)
            Rr = np.flatnonzero(R)
            if Rr.size:  # constrained-model recompute (models.py:431 on G_post)
                _, Ar, Cr = M.layer_full(b, l, g, h_new, rows=Rr)
                A_new[Rr] = Ar
                C_new[Rr] = Cr
            self.A[l], self.C[l] = A_new, C_new
            upd = np.flatnonzero(vdst)
            H_old.append(self.H[l + 1].copy())  # DeltaLog
            Hn = self.H[l + 1].copy()
            if upd.size:
                Hn[upd] = M.update(b, l, h_new[upd], A_new[upd])
            self.H[l + 1] = Hn
            chg_prev = vdst
        return dict(status=status, deltas=deltas, frontier=frontier)

    def _incremental(self, l, rows, vcs, vcd, Is, Id, Ds, Dd, h_new, h_old, old_in, old_out, A, C):
        b, g = self.b, self.g
        n = g.n
        pos = np.full(n, -1, np.int64)
        pos[rows] = np.arange(rows.size)
        R = rows.size
        new_in = g.in_deg
        if b.model == M.GAT:
            z_n, el_n, er_n = M.gat_project(b, l, h_new)
            z_o, _, er_o = M.gat_project(b, l, h_old)
            heads, dh = z_n.shape[1], z_n.shape[2]

            def at(d, u, er):  # models.py:265-274
                return np.exp(M.leaky(el_n[d] + er[u]))

            pieces = [  # (sign, src, dst, er, z)
                (+1, vcs, vcd, er_n, z_n), (-1, vcs, vcd, er_o, z_o),
                (+1, Is, Id, er_n, z_n), (-1, Ds, Dd, er_o, z_o),
            ]
            ctx_old = C[rows].reshape(R, heads)
            dctx = np.zeros((R, heads))
            dS = np.zeros((R, heads, dh))
            for s, u, d, er, z in pieces:
                if u.size == 0:
                    continue
                w = at(d, u, er)  # [E, heads]
                np.add.at(dctx, pos[d], s * w)
                for h in range(heads):
                    Mx = sp.csr_matrix((s * w[:, h], (pos[d], u)), shape=(R, n))
                    dS[:, h, :] += Mx @ z[:, h, :]
            A_old = A[rows].reshape(R, heads, dh)
            had = old_in[rows] > 0
            ahat = np.where(had[:, None, None], M.strip(b, ctx_old, A_old), 0.0)  # Alg.3 l.6
            ctx_new = ctx_old + dctx  # Alg.3 l.5
            ahat = ahat + dS  # Alg.3 l.7
            has = new_in[rows] > 0
            safe = np.where(has[:, None], ctx_new, 1.0)
            a_new = np.where(has[:, None, None], M.compose(b, safe, ahat), 0.0)  # Alg.3 l.8
            ctx_new = np.where(has[:, None], ctx_new, 0.0)
            A[rows] = a_new.reshape(R, heads * dh)
            C[rows] = ctx_new[:, 0] if heads == 1 else ctx_new
            return
        if b.model in M.EDGE_MODELS:  # dest-dependent, no context: v ∉ R keeps h_v
            dS = np.zeros((R, h_new.shape[1]))
            for s, u, d, h in ((+1, vcs, vcd, h_new), (-1, vcs, vcd, h_old), (+1, Is, Id, h_new), (-1, Ds, Dd, h_old)):
                if u.size:
                    np.add.at(dS, pos[d], s * M.edge_message(b, l, h[u], h_new[d]))
            had = old_in[rows] > 0
            has = new_in[rows] > 0
            a_new = np.where(had[:, None], A[rows], 0.0) + dS
            A[rows] = np.where(has[:, None], a_new, 0.0)
            C[rows] = 1.0
            return
        if b.model in M.PAYLOAD_MODELS:  # messages are per-source payload rows
            h_new, h_old = M.payload(b, l, h_new), M.payload(b, l, h_old)
        with np.errstate(divide="ignore"):
            c_new = M.src_coeff(b, g.out_deg)
            c_old = M.src_coeff(b, old_out)
        d_a = h_new.shape[1]
        dS = np.zeros((R, d_a))
        dcnt = np.zeros(R)
        for s, u, d, c, h in ((+1, vcs, vcd, c_new, h_new), (-1, vcs, vcd, c_old, h_old),
                              (+1, Is, Id, c_new, h_new), (-1, Ds, Dd, c_old, h_old)):
            if u.size == 0:
                continue
            Mx = sp.csr_matrix((s * c[u], (pos[d], u)), shape=(R, n))
            dS += Mx @ h
        np.add.at(dcnt, pos[Id], 1.0)
        np.add.at(dcnt, pos[Dd], -1.0)
        ctx_old = C[rows]
        had = old_in[rows] > 0
        ahat = np.where(had[:, None], M.strip(b, ctx_old, A[rows]), 0.0)  # Alg.1 l.4
        if b.ctx_kind == "count":
            ctx_new = ctx_old + dcnt  # Alg.1 l.3 (count context)
        else:
            ctx_new = np.ones(R)
        ahat = ahat + dS  # Alg.1 l.5
        has = new_in[rows] > 0
        safe = np.where(has, ctx_new, 1.0)
        a_new = np.where(has[:, None], M.compose(b, safe, ahat), 0.0)  # Alg.1 l.6
        ctx_new = np.where(has, ctx_new, b.empty_context())
        A[rows] = a_new
        C[rows] = ctx_new
