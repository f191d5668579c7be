// layer.cu -- per-layer incremental / full aggregation and the update
// (SURVEY §2.1 K10-K15, K17, K18).
//
// State per layer (rtec_state_t): S = aggregate before ms_cbn (the stripped
// form of Alg. 1 line 4, kept resident so strip/compose never round-trip),
// ctx (GAT attention sums; count contexts are the in-degrees), H_out, and the
// DeltaLog of pre-batch H_out rows of V_dst(l).
//
// Incremental (Alg. 1), v ∈ V_dst(l) \ R(l):
//   ValueChange edge (u,v), u ∈ S(l), (u,v) ∉ I :  + δ_u,  δ_u = c_new(u) h_new(u) - c_old(u) h_old(u)
//   StructInsert (u,v) ∈ I                      :  + c_new(u) h_new(u)
//   StructDelete (u,v) ∈ D                      :  - c_old(u) h_old(u)
//   S_v <- (indeg_new(v) == 0) ? 0 : S_v + Σ ;  a_v = ms_cbn(ctx_new, S_v);  h_v = update(h_v, a_v)
// with c = 1/sqrt(d_out + off) for GCN (models.py:98-99), 1 otherwise.
// GAT (Alg. 3) carries per-edge attention instead of c and
// recomputes R(l) = V_dst(l) ∩ V_chg(l-1) over the full post-batch
// neighbourhood (models.py:431-458).
#include "prims.cuh"
#include "rowops.cuh"
#include "gemm_tc.cuh"
#include "async.cuh"

#include <stdlib.h>

namespace rtec {

constexpr int kLBlk = 256;
constexpr int kUnroll = 4;

__device__ __forceinline__ float src_coeff(int model, int32_t deg, float off) {
  return model == RTEC_MODEL_GCN ? 1.0f / sqrtf(static_cast<float>(deg) + off) : 1.0f;
}

// source coefficient of the fused deltas (update epilogue): 0 for a vertex without
// out-edges, which never contributes (keeps raw-degree GCN finite)
__device__ __forceinline__ float fused_coeff(int model, int32_t deg, float off) {
  return deg > 0 ? src_coeff(model, deg, off) : 0.f;
}

__host__ __device__ __forceinline__ bool is_gin(int model) {
  return model == RTEC_MODEL_GIN || model == RTEC_MODEL_GIN_MAX;
}

// Table II model classes (models.py:144-348)
__host__ __device__ __forceinline__ bool self_concat(int model) {  // update reads [h_v ; a_v]
  return model == RTEC_MODEL_PINSAGE || model == RTEC_MODEL_COMMNET;
}
__host__ __device__ __forceinline__ bool payload_model(int model) {  // message = projected payload of h_u
  return model == RTEC_MODEL_PINSAGE || model == RTEC_MODEL_MONET;
}
__host__ __device__ __forceinline__ bool edge_model(int model) {  // message reads h_u and h_v
  return model == RTEC_MODEL_GGCN || model == RTEC_MODEL_AGNN;
}
__host__ __device__ __forceinline__ int upd_k(const rtec_layer_t& L) { return L.d_k > 0 ? L.d_k : L.d_in; }

__device__ __forceinline__ float leaky02(float x) { return x < 0.f ? 0.2f * x : x; }  // models.py:272-273
__device__ __forceinline__ float elu1(float x) { return x >= 0.f ? x : expm1f(x); }   // linalg.py:41-43

struct LayerArgs {
  rtec_graph_t g;
  rtec_batch_t b;
  rtec_layer_t L;
  rtec_state_t st;
  rtec_frontier_t f;
  const uint32_t* prev_bm_dst;  // V_chg(l-1) (null for l = 0)
  const int32_t* prev_slot;     // vertex -> DeltaLog row of the previous layer
  const float* delta;           // [n_src, d_agg] δ rows (non-GAT)
  int d_agg;
  int tc_nkb;                   // > 0: gemm_in is the tcgen05 A image with tc_nkb K-blocks
  int c0, cw;                   // feature slice [c0, c0 + cw) of the d_agg-wide rows (aggregation)
  int gcol, gk;                 // aggregate columns start at gcol of the gk-wide update input
  const float* self_in;         // H^l (st.H_in is redirected to the payload rows for PinSAGE / MoNet)
  int layer;
  uint64_t* err;
  // light-pass kernel chosen on the device from the layer's scan size Σ indeg(V_dst) and hit
  // density |E_curr| / Σ indeg(V_dst) (frontier counters 5 / 0): 0 always run, 1 run only on
  // large sparse scans (warp-batched pass), 2 otherwise (one destination per warp)
  int pick;
  float pick_thr;
};

// the warp-batched pass pays off only on large, sparse scans (c2-gcn layer 1: 55M scanned
// in-edges, 24 % hits); small layers (c1, c2-sage layer 1) and dense ones favour one
// destination per warp (profiles/r02j_light_pick_ab.md)
constexpr float kBatchMinScan = 8e6f;

__device__ __forceinline__ bool pick_ok(const LayerArgs& a) {
  if (a.pick == 0) return true;
  const float e = static_cast<float>(a.f.counters[0]);
  const float s = static_cast<float>(a.f.counters[5]);
  const bool batched = s >= kBatchMinScan && e < a.pick_thr * s;
  return a.pick == 1 ? batched : !batched;
}

// row of v in S / ctx (and in H_out when out_local): per owned vertex when sharded
__device__ __forceinline__ int64_t srow(const LayerArgs& a, int32_t v) {
  return a.st.row_div > 1 ? static_cast<int64_t>(v / a.st.row_div) : static_cast<int64_t>(v);
}
__device__ __forceinline__ int64_t hrow(const LayerArgs& a, int32_t v) {
  return (a.st.out_local && a.st.row_div > 1) ? static_cast<int64_t>(v / a.st.row_div) : static_cast<int64_t>(v);
}
// row of source u in the δ buffer: its S(l) slot when slot-indexed
__device__ __forceinline__ int64_t drow(const LayerArgs& a, int32_t u) {
  return a.st.delta_slot ? static_cast<int64_t>(a.f.src_slot[u]) : static_cast<int64_t>(u);
}

// ------------------------------------------------------------------ δ rows (K10)
template <int VEC, int K>
__global__ void __launch_bounds__(kLBlk) k_src_delta(LayerArgs a, float* delta) {
  RTEC_PDL_ENTRY();
  using R = RowAcc<VEC, K>;
  // After a fused update (unsharded), S(l) \ V_chg(l-1) = Dg \ V_chg(l-1): walk the batch's
  // DegreeDelta vertices (<= 2B) instead of all of S(l) (c2-gcn layer 2: 124K vs 2.19M)
  const bool dg_walk = a.st.delta_ready && a.prev_bm_dst && !a.st.delta_slot && a.b.dg_bm == nullptr;
  int64_t ns = dg_walk ? *a.b.n_delta : *a.f.n_src;
  int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int d = a.d_agg;
  for (int64_t i = warp; i < ns; i += nw) {
    int32_t u;
    if (dg_walk) {
      u = a.b.d_vertex[i];
      if (!bm_test(a.f.bm_src, u)) continue;
    } else {
      u = a.f.src_list[i];
    }
    // rows of V_chg(l-1) were written by the previous layer's update epilogue
    if (a.st.delta_ready && a.prev_bm_dst && bm_test(a.prev_bm_dst, u)) continue;
    int32_t dn = a.g.out_deg[u], dp = a.g.out_deg_prev[u];
    R acc;
    acc.zero();
    if (dn > 0 && dp > 0) {  // otherwise u has no ValueChange edges
      float cn = src_coeff(a.L.model, dn, a.L.degree_offset);
      float co = src_coeff(a.L.model, dp, a.L.degree_offset);
      float hn[K][VEC], ho[K][VEC];
      R::load(a.st.H_in + static_cast<int64_t>(u) * d, d, hn);
      const float* orow = a.st.H_in + static_cast<int64_t>(u) * d;
      if (a.prev_bm_dst && bm_test(a.prev_bm_dst, u)) orow = a.st.log_in + static_cast<int64_t>(a.prev_slot[u]) * d;
      R::load(orow, d, ho);
      acc.fma(hn, cn);
      acc.fma(ho, -co);
    }
    // indexed by vertex (no slot gather per edge) unless the sharded δ buffer is slot-indexed
    acc.store(delta + (a.st.delta_slot ? i : static_cast<int64_t>(u)) * d, d);
  }
}

// is (u, v) an applied insert?  I/D entries of v are i_src[p, q) ascending
__device__ __forceinline__ bool in_range_has(const int32_t* __restrict__ is, int64_t p, int64_t q, int32_t u) {
  if (p >= q) return false;
  int64_t k = lower_bound_dev(is, p, q, u);
  return k < q && is[k] == u;
}

// ------------------------------------------------------------------ aggregation (K11 incremental, K17 full)
// Edge-balanced: destinations whose scanned in-run is <= kChunk edges are
// handled by one warp each ("light" pass); longer runs ("heavy": hubs, up to
// 392K in-edges at configs[1]) are cut into kChunk-edge chunks, one warp per
// chunk, partial rows written to scratch and reduced in chunk order by the
// last-arriving warp (deterministic; threadfence + per-vertex arrival counter).
constexpr int kChunk = 512;

// chunks of all heavy runs (len > kChunk) within `max_edges` slots: ceil(len / kChunk) <=
// 2 len / kChunk for len > kChunk, so the sum is at most 2 max_edges / kChunk
__host__ __device__ constexpr int64_t heavy_chunk_bound(int64_t max_edges) { return 2 * max_edges / kChunk + 2; }

template <int VEC, int K, bool FULL>
__device__ __forceinline__ void agg_edges(const LayerArgs& a, int64_t beg, int32_t e0, int32_t e1, int64_t p,
                                          int64_t q, RowAcc<VEC, K>& acc) {
  using R = RowAcc<VEC, K>;
  constexpr int UNR = (VEC * K <= 2) ? 8 : kUnroll;  // more rows in flight for thin slices
  const int d = a.d_agg, cw = a.cw;
  const int lane = lane_id();
  const uint64_t pol = l2_evict_first_policy();
  for (int32_t c0 = e0; c0 < e1; c0 += 32) {
    int32_t j = c0 + lane;
    int32_t u = 0;
    bool hit = false;
    float cu = 0.f;
    if (j < e1) {
      u = ld_stream_i32(a.g.in.nbr + beg + j, pol);
      if (FULL) {
        hit = true;
        cu = src_coeff(a.L.model, a.g.out_deg[u], a.L.degree_offset);
      } else {
        hit = bm_test(a.f.bm_src, u) && !in_range_has(a.b.i_src, p, q, u);
      }
    }
    unsigned m = __ballot_sync(0xffffffffu, hit);
    const float* base = (FULL ? a.st.H_in : a.delta) + a.c0;
    // gathered row: the source's own row (H_in, vertex-indexed δ) or its δ slot
    int32_t row = (!FULL && hit && a.st.delta_slot) ? a.f.src_slot[u] : u;
    while (m) {
      int32_t rw[UNR];
      float cs[UNR];
      int cnt = 0;
#pragma unroll
      for (int t = 0; t < UNR; ++t) {
        int src = m ? __ffs(m) - 1 : 0;
        if (m) {
          m &= m - 1;
          cnt = t + 1;
        }
        rw[t] = __shfl_sync(0xffffffffu, row, src);
        cs[t] = __shfl_sync(0xffffffffu, cu, src);
      }
      float r[UNR][K][VEC];
#pragma unroll
      for (int t = 0; t < UNR; ++t)
        if (t < cnt) R::load(base + static_cast<int64_t>(rw[t]) * d, cw, r[t]);
#pragma unroll
      for (int t = 0; t < UNR; ++t) {
        if (t < cnt) {
          if (FULL) acc.fma(r[t], cs[t]);
          else acc.add(r[t]);
        }
      }
    }
  }
}

// structural edges of v (graph.py:202-224 applied set): + c_new h_new for I, - c_old h_old for D
template <int VEC, int K>
__device__ __forceinline__ void agg_struct(const LayerArgs& a, int64_t p, int64_t q, RowAcc<VEC, K>& acc) {
  using R = RowAcc<VEC, K>;
  const int d = a.d_agg, cw = a.cw;
  for (int64_t k = p; k < q; ++k) {
    int32_t u = a.b.i_src[k];
    float r[K][VEC];
    if (a.b.i_op[k] == RTEC_OP_INSERT) {
      R::load(a.st.H_in + static_cast<int64_t>(u) * d + a.c0, cw, r);
      acc.fma(r, src_coeff(a.L.model, a.g.out_deg[u], a.L.degree_offset));
    } else if (a.st.delta_ready && a.prev_bm_dst && bm_test(a.prev_bm_dst, u)) {
      // -c_old h_old(u) = δ_u - c_new h_new(u)  (fused deltas: no DeltaLog)
      R::load(a.delta + drow(a, u) * d + a.c0, cw, r);
      acc.add(r);
      R::load(a.st.H_in + static_cast<int64_t>(u) * d + a.c0, cw, r);
      acc.fma(r, -fused_coeff(a.L.model, a.g.out_deg[u], a.L.degree_offset));
    } else {
      const float* orow = a.st.H_in + static_cast<int64_t>(u) * d;
      if (a.prev_bm_dst && bm_test(a.prev_bm_dst, u)) orow = a.st.log_in + static_cast<int64_t>(a.prev_slot[u]) * d;
      R::load(orow + a.c0, cw, r);
      acc.fma(r, -src_coeff(a.L.model, a.g.out_deg_prev[u], a.L.degree_offset));
    }
  }
}

// S_v update (INC: S += Σ, zero-in-degree rule; FULL: S = Σ), compose, GEMM input row i.
// `pre`: the caller already loaded indeg and the cached row (sv, zero when not to be added).
template <int VEC, int K, bool FULL>
__device__ __forceinline__ void agg_finalize(const LayerArgs& a, int64_t i, int32_t v, int32_t len,
                                             RowAcc<VEC, K>& acc, const RowAcc<VEC, K>* pre = nullptr,
                                             int32_t pre_indeg = 0) {
  using R = RowAcc<VEC, K>;
  const int d = a.d_agg, cw = a.cw;
  float* sp = a.st.S + srow(a, v) * d + a.c0;
  int32_t indeg = FULL ? len : (pre ? pre_indeg : a.g.in_deg[v]);
  if (!FULL) {
    if (indeg == 0) {
      acc.zero();  // empty neighbourhood -> zero aggregate
    } else if (pre) {
      acc.add(pre->v);
    } else if (a.g.in_deg_prev[v] > 0) {
      float sv[K][VEC];
      R::load_stream(sp, cw, sv, l2_evict_first_policy());
      acc.add(sv);
    }
  }
  acc.store_stream(sp, cw, l2_evict_first_policy());
  float scale = 1.f;
  if (indeg > 0) {
    if (a.L.model == RTEC_MODEL_GCN) scale = rsqrtf(static_cast<float>(indeg) + a.L.degree_offset);  // MUFU.RSQ (<= 2 ulp)
    else if (a.L.model == RTEC_MODEL_SAGE || a.L.model == RTEC_MODEL_PINSAGE) scale = 1.0f / static_cast<float>(indeg);
  }
  R out;
  out.zero();
  out.fma(acc.v, scale);
  if (is_gin(a.L.model)) {  // update input h_v + a_v (models.py:187-189)
    float h[K][VEC];
    R::load(a.self_in + static_cast<int64_t>(v) * d + a.c0, cw, h);
    out.add(h);
  } else if (self_concat(a.L.model)) {  // update input [h_v ; a_v] (models.py:161-162, :247)
    R hv;
    R::load(a.self_in + static_cast<int64_t>(v) * d + a.c0, cw, hv.v);
    if (a.tc_nkb > 0) hv.store_tiled(a.st.gemm_in, i, a.c0, cw, a.gk, a.tc_nkb);
    else hv.store(a.st.gemm_in + i * a.gk + a.c0, cw);
  }
  if (a.tc_nkb > 0) out.store_tiled(a.st.gemm_in, i, a.gcol + a.c0, cw, a.gk, a.tc_nkb);
  else out.store_stream(a.st.gemm_in + i * a.gk + a.gcol + a.c0, cw, l2_evict_first_policy());
}

struct AggRows {
  const int32_t* list;  // null -> identity
  const int64_t* n_dev; // null -> n_all
  int64_t n_all;
  __device__ __forceinline__ int64_t count() const { return n_dev ? *n_dev : n_all; }
  __device__ __forceinline__ int32_t at(int64_t i) const { return list ? list[i] : static_cast<int32_t>(i); }
};

struct HeavyPlan {
  int32_t* heavy;   // dst indices i of heavy destinations
  int64_t* n_heavy; // [0] heavy destinations, [1] chunks, [2] packed scan total (then hoff)
  int64_t* hoff;    // [n_heavy + 1] chunk offsets
  int32_t* cmap;    // chunk -> heavy index j
  int32_t* arrive;  // [n_heavy] arrival counters (zeroed per launch)
  float* part;      // [chunks, d] partial rows
  // chunk visit order: chunks sorted (stably) by their relative position c / nch in
  // their destination's in-run, so the warps resident at one time gather from the
  // same band of (ascending) source ids of every hub -- an L2-sized working set.
  // nullptr: destination-major.  Execution order only: partials are still reduced
  // in chunk order (results identical).
  const uint32_t* order;
  uint64_t* okey;   // 8-bit sort keys (c << 8) / nch written by k_chunk_map (256 position bands: one radix pass)
  uint32_t* oval;   // chunk ids
};

// resident CTAs per SM: wide rows need the registers (no spills)
template <int VEC, int K>
struct AggOcc {
  static constexpr int value = (VEC * K <= 8) ? 4 : 2;  // measured: 3 CTAs for VEC*K = 8 (no spills) is slower
};

// acc += rows 0..nch-1 (stride `stride` floats, width w) in row order, 4 rows in flight:
// the last-arriving warp of a hub reduces up to ~10^3 chunk partials
template <int VEC, int K>
__device__ __forceinline__ void sum_partials(const float* part, int64_t stride, int w, int32_t nch,
                                             RowAcc<VEC, K>& acc) {
  int32_t cc = 0;
  for (; cc + 4 <= nch; cc += 4) {
    float r[4][K][VEC];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const int col = lane_id() + 32 * k;
#pragma unroll
        for (int jj = 0; jj < VEC; ++jj)
          r[u][k][jj] = (col * VEC < w) ? __ldcg(part + (cc + u) * stride + col * VEC + jj) : 0.f;
      }
#pragma unroll
    for (int u = 0; u < 4; ++u) acc.add(r[u]);
  }
  for (; cc < nch; ++cc) {
    float r[K][VEC];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int col = lane_id() + 32 * k;
#pragma unroll
      for (int jj = 0; jj < VEC; ++jj) r[k][jj] = (col * VEC < w) ? __ldcg(part + cc * stride + col * VEC + jj) : 0.f;
    }
    acc.add(r);
  }
}

template <int VEC, int K, bool FULL>
__global__ void __launch_bounds__(kLBlk, AggOcc<VEC, K>::value) k_agg_light(LayerArgs a, AggRows rows) {
  RTEC_PDL_ENTRY();
  using R = RowAcc<VEC, K>;
  __shared__ __align__(16) float s_sv[kLBlk / 32][(!FULL && VEC == 4) ? 32 * VEC * K : 4];
  if (!FULL && err_set(a.err)) return;
  if (!FULL && !pick_ok(a)) return;
  const int64_t nr = rows.count();
  const bool scan = FULL || *a.f.n_src > 0;
  int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < nr; i += nw) {
    int32_t v = rows.at(i);
    // independent per-destination loads issued together (the chain below is latency-bound)
    const int32_t len = a.g.in.len[v];
    const int64_t beg = a.g.in.beg[v];
    int2 rg = make_int2(-1, 0);
    int32_t indeg = len, had = 0;
    if (!FULL) {
      rg = reinterpret_cast<const int2*>(a.b.irange)[v];
      indeg = a.g.in_deg[v];
      had = a.g.in_deg_prev[v];
    }
    if (scan && len > kChunk) continue;  // heavy pass
    int64_t p = 0, q = 0;
    if (rg.x >= 0) {
      p = rg.x;
      q = rg.x + rg.y;
    }
    // the cached aggregate row, requested before the edge scan so its latency overlaps it
    // (16-byte rows: staged in shared memory by cp.async, so it holds no registers --
    // and is not spilled -- across the gather loop)
    const bool pre = !FULL && indeg > 0 && had > 0;
    R sv;
    sv.zero();
    if constexpr (VEC == 4) {
      if (pre) R::stage_async(s_sv[threadIdx.x >> 5], a.st.S + srow(a, v) * a.d_agg + a.c0, a.cw, l2_evict_first_policy());
    } else {
      if (pre) R::load_stream(a.st.S + srow(a, v) * a.d_agg + a.c0, a.cw, sv.v, l2_evict_first_policy());
    }
    R acc;
    acc.zero();
    if (scan) agg_edges<VEC, K, FULL>(a, beg, 0, len, p, q, acc);
    if (!FULL) agg_struct<VEC, K>(a, p, q, acc);
    if constexpr (VEC == 4) {
      if (pre) R::from_stage(s_sv[threadIdx.x >> 5], a.cw, sv.v);
    }
    agg_finalize<VEC, K, FULL>(a, i, v, len, acc, FULL ? nullptr : &sv, indeg);
  }
}

// Warp-batched incremental light pass: a warp takes 32 consecutive destinations
// (one per lane for the metadata loads, all issued together), scans the in-runs
// of a run of them as ONE flattened edge sequence (lane e finds its
// destination by a shuffle binary search over the run offsets) and compacts
// the ValueChange hits, in order, into a per-warp shared-memory window with
// per-destination counts; then, destination by destination, gathers its hit
// rows UNR at a time (the cached S row prefetched first), adds the structural
// edges and finalises.  Per destination this replaces the dependent chain
// metadata -> run -> bitmap -> rows of k_agg_light by batched loads, for the
// scan-heavy layers (few hits among many scanned edges).  Summation order per
// destination (run order, then structural edges) matches k_agg_light.
constexpr int kBatchWin = kChunk;  // flattened edges per window: any light run fits one window

template <int VEC, int K, int OCC = 0>
__global__ void __launch_bounds__(kLBlk, OCC > 0 ? OCC : AggOcc<VEC, K>::value) k_agg_batch(LayerArgs a, AggRows rows) {
  RTEC_PDL_ENTRY();
  using R = RowAcc<VEC, K>;
  constexpr int UNR = kUnroll;  // measured: 8 rows in flight spill next to the prefetched S row
  __shared__ int32_t s_u[kLBlk / 32][kBatchWin];
  __shared__ int32_t s_c[kLBlk / 32][32];
  if (err_set(a.err)) return;
  if (!pick_ok(a)) return;
  const int64_t nr = rows.count();
  const bool scan = *a.f.n_src > 0;
  const int lane = lane_id();
  const int wib = threadIdx.x >> 5;
  int32_t* hu = s_u[wib];
  int32_t* hc = s_c[wib];
  const int d = a.d_agg, cw = a.cw;
  const float* base = a.delta + a.c0;
  const int64_t ngroups = (nr + 31) >> 5;
  int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t grp = warp; grp < ngroups; grp += nw) {
    const int64_t i0 = grp << 5;
    const int nd = static_cast<int>(nr - i0 < 32 ? nr - i0 : 32);
    int32_t v = 0, len = 0, indeg = 0, had = 0, p = 0, q = 0;
    int64_t beg = 0;
    bool live = lane < nd;
    if (live) {
      v = rows.at(i0 + lane);
      len = a.g.in.len[v];
      beg = a.g.in.beg[v];
      const int2 rg = reinterpret_cast<const int2*>(a.b.irange)[v];
      indeg = a.g.in_deg[v];
      had = a.g.in_deg_prev[v];
      if (rg.x >= 0) {
        p = rg.x;
        q = rg.x + rg.y;
      }
      if (scan && len > kChunk) live = false;  // heavy pass owns it
    }
    const int32_t slen = (live && scan) ? len : 0;
    int32_t end = slen;  // inclusive scan: end of this lane's run in the flattened sequence
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t t = __shfl_up_sync(0xffffffffu, end, o);
      if (lane >= o) end += t;
    }
    const int32_t off = end - slen;
    const unsigned live_mask = __ballot_sync(0xffffffffu, live);
    int j0 = 0;
    while (j0 < nd) {
      // window [j0, j1): the longest run of destinations whose edges fit kBatchWin
      const int32_t w0 = __shfl_sync(0xffffffffu, off, j0);
      const unsigned fit = __ballot_sync(0xffffffffu, lane >= j0 && lane < nd && end - w0 <= kBatchWin);
      const int j1 = max(j0 + 1, 32 - __clz(fit));  // fit is a prefix of [j0, nd) (ends grow)
      const int32_t w1 = __shfl_sync(0xffffffffu, end, j1 - 1);
      hc[lane] = 0;
      __syncwarp();
      int nh = 0;
      for (int32_t e0 = w0; e0 < w1; e0 += 32) {
        const int32_t e = e0 + lane;
        int lo = j0;  // last destination j in [j0, j1) with off_j <= e
#pragma unroll
        for (int step = 16; step > 0; step >>= 1) {
          const int cand = lo + step;
          const int32_t oc = __shfl_sync(0xffffffffu, off, cand & 31);
          if (cand < j1 && oc <= e) lo = cand;
        }
        const int64_t bj = __shfl_sync(0xffffffffu, beg, lo);
        const int32_t oj = __shfl_sync(0xffffffffu, off, lo);
        const int32_t pj = __shfl_sync(0xffffffffu, p, lo);
        const int32_t qj = __shfl_sync(0xffffffffu, q, lo);
        bool hit = false;
        int32_t u = 0;
        if (e < w1) {
          u = a.g.in.nbr[bj + (e - oj)];
          hit = bm_test(a.f.bm_src, u) && !in_range_has(a.b.i_src, pj, qj, u);
        }
        const unsigned m = __ballot_sync(0xffffffffu, hit);
        if (hit) {
          hu[nh + __popc(m & ((1u << lane) - 1u))] = a.st.delta_slot ? a.f.src_slot[u] : u;
          atomicAdd(hc + lo, 1);
        }
        nh += __popc(m);
      }
      __syncwarp();
      int32_t hs = hc[lane];  // exclusive scan of the per-destination hit counts
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int32_t t = __shfl_up_sync(0xffffffffu, hs, o);
        if (lane >= o) hs += t;
      }
      hs -= hc[lane];
      // destinations of the window in order; the cached S row of the next one is
      // requested before this one's gathers (one DRAM latency hidden per destination)
      const unsigned wm = live_mask & (j1 >= 32 ? 0xffffffffu : ((1u << j1) - 1u)) & ~((1u << j0) - 1u);
      int jn = wm ? __ffs(wm) - 1 : 32;
      R svn;
      svn.zero();
      if (jn < 32) {
        const int32_t vn = __shfl_sync(0xffffffffu, v, jn);
        if (__shfl_sync(0xffffffffu, indeg, jn) > 0 && __shfl_sync(0xffffffffu, had, jn) > 0)
          R::load_stream(a.st.S + srow(a, vn) * d + a.c0, cw, svn.v, l2_evict_first_policy());
      }
      while (jn < 32) {
        const int j = jn;
        R sv = svn;
        const unsigned rest = wm & ~(j >= 31 ? 0xffffffffu : ((2u << j) - 1u));
        jn = rest ? __ffs(rest) - 1 : 32;
        svn.zero();
        if (jn < 32) {
          const int32_t vn = __shfl_sync(0xffffffffu, v, jn);
          if (__shfl_sync(0xffffffffu, indeg, jn) > 0 && __shfl_sync(0xffffffffu, had, jn) > 0)
            R::load_stream(a.st.S + srow(a, vn) * d + a.c0, cw, svn.v, l2_evict_first_policy());
        }
        const int32_t vj = __shfl_sync(0xffffffffu, v, j);
        const int32_t lj = __shfl_sync(0xffffffffu, len, j);
        const int32_t ij = __shfl_sync(0xffffffffu, indeg, j);
        const int32_t pj = __shfl_sync(0xffffffffu, p, j);
        const int32_t qj = __shfl_sync(0xffffffffu, q, j);
        const int32_t h0 = __shfl_sync(0xffffffffu, hs, j);
        const int32_t h1 = h0 + hc[j];
        R acc;
        acc.zero();
        for (int32_t k0 = h0; k0 < h1; k0 += UNR) {
          const int cnt = min(UNR, h1 - k0);
          float r[UNR][K][VEC];
#pragma unroll
          for (int t = 0; t < UNR; ++t)
            if (t < cnt) R::load(base + static_cast<int64_t>(hu[k0 + t]) * d, cw, r[t]);
#pragma unroll
          for (int t = 0; t < UNR; ++t)
            if (t < cnt) acc.add(r[t]);
        }
        agg_struct<VEC, K>(a, pj, qj, acc);
        agg_finalize<VEC, K, false>(a, i0 + j, vj, lj, acc, &sv, ij);
      }
      __syncwarp();
      j0 = j1;
    }
  }
}

template <int VEC, int K, bool FULL>
__global__ void __launch_bounds__(kLBlk, AggOcc<VEC, K>::value) k_agg_heavy(LayerArgs a, AggRows rows, HeavyPlan hp) {
  RTEC_PDL_ENTRY();
  using R = RowAcc<VEC, K>;
  if (!FULL && err_set(a.err)) return;
  const int64_t nh = *hp.n_heavy;
  if (nh == 0) return;
  const int64_t T = hp.hoff[nh];
  const int cw = a.cw;
  int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t tt = warp; tt < T; tt += nw) {
    const int64_t t = hp.order ? static_cast<int64_t>(hp.order[tt]) : tt;
    int32_t j = hp.cmap[t];
    int64_t c0 = hp.hoff[j];
    int32_t nch = static_cast<int32_t>(hp.hoff[j + 1] - c0);
    int32_t c = static_cast<int32_t>(t - c0);
    int64_t i = hp.heavy[j];
    int32_t v = rows.at(i);
    int32_t len = a.g.in.len[v];
    int64_t p = 0, q = 0;
    if (!FULL) {
      int2 rg = reinterpret_cast<const int2*>(a.b.irange)[v];
      if (rg.x >= 0) {
        p = rg.x;
        q = rg.x + rg.y;
      }
    }
    R acc;
    acc.zero();
    int32_t e0 = c * kChunk, e1 = min(len, e0 + kChunk);
    agg_edges<VEC, K, FULL>(a, a.g.in.beg[v], e0, e1, p, q, acc);
    if (!FULL && c == 0) agg_struct<VEC, K>(a, p, q, acc);
    acc.store(hp.part + t * cw, cw);
    __threadfence();
    __syncwarp();  // every lane's partial is fenced before the arrival is published
    int old = 0;
    if (lane_id() == 0) old = atomicAdd(hp.arrive + j, 1);
    old = __shfl_sync(0xffffffffu, old, 0);
    if (old != nch - 1) continue;
    __threadfence();
    acc.zero();
    sum_partials<VEC, K>(hp.part + c0 * cw, cw, cw, nch, acc);  // chunk order: deterministic sum
    agg_finalize<VEC, K, FULL>(a, i, v, len, acc);
  }
}

// heavy-destination planning: list, chunk offsets, chunk -> heavy map
struct HeavyFlagF {
  AggRows rows;
  const int32_t* len;
  const int64_t* n_src;  // null in FULL mode
  __device__ __forceinline__ int64_t operator()(int64_t i) const {
    if (n_src && *n_src == 0) return 0;
    return len[rows.at(i)] > kChunk ? 1 : 0;
  }
};
struct HeavyStore {
  HeavyFlagF f;
  int32_t* heavy;
  __device__ __forceinline__ void operator()(int64_t i, int64_t off, int64_t v) const {
    if (v) heavy[off] = static_cast<int32_t>(i);
  }
};
// one scan for the heavy list and its chunk offsets: (1 << 32 | chunks) per heavy destination
// (heavy count < 2^31, chunks < 2^32: the packed sums never carry between the halves)
struct HeavyPackF {
  HeavyFlagF f;
  __device__ __forceinline__ int64_t operator()(int64_t i) const {
    if (f.n_src && *f.n_src == 0) return 0;
    const int32_t len = f.len[f.rows.at(i)];
    return len > kChunk ? ((int64_t(1) << 32) | ((len + kChunk - 1) / kChunk)) : 0;
  }
};
struct HeavyPackStore {
  AggRows rows;
  int32_t* heavy;
  int64_t* hoff;
  __device__ __forceinline__ void operator()(int64_t i, int64_t off, int64_t v) const {
    if (v) {
      heavy[off >> 32] = static_cast<int32_t>(i);
      hoff[off >> 32] = off & 0xffffffffll;
    }
    if (i == rows.count() - 1) {  // tail: hoff[n_heavy] = total chunks
      const int64_t t = off + v;
      hoff[t >> 32] = t & 0xffffffffll;
    }
  }
};
struct StoreOffTailL {
  int64_t* dst;
  const int64_t* n;
  __device__ __forceinline__ void operator()(int64_t i, int64_t off, int64_t v) const {
    dst[i] = off;
    if (i == *n - 1) dst[i + 1] = off + v;
  }
};

__global__ void k_chunk_map(HeavyPlan hp) {
  RTEC_PDL_ENTRY();
  const int64_t packed = hp.n_heavy[2];  // HeavyPackF total: heavy count << 32 | chunks
  const int64_t nh = packed >> 32;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    hp.n_heavy[0] = nh;
    hp.n_heavy[1] = packed & 0xffffffffll;  // total chunks (sort count)
  }
  int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t j = warp; j < nh; j += nw) {
    int64_t c0 = hp.hoff[j], c1 = hp.hoff[j + 1];
    for (int64_t c = c0 + lane_id(); c < c1; c += 32) {
      hp.cmap[c] = static_cast<int32_t>(j);
      if (hp.okey) {
        hp.okey[c] = static_cast<uint64_t>(((c - c0) << 8) / (c1 - c0));
        hp.oval[c] = static_cast<uint32_t>(c);
      }
    }
    if (lane_id() == 0) hp.arrive[j] = 0;
  }
}

// RTEC_AGG_SLICE env: feature-slice width of the aggregation passes (default 0 = whole rows)
static int agg_slice_width() {
  static int w = -1;
  if (w < 0) {
    const char* e = getenv("RTEC_AGG_SLICE");
    w = e ? atoi(e) : 0;  // measured: slicing costs more per-edge work than it saves in L2 misses
    if (w < 0 || w > 256) w = 256;
    w &= ~1;
  }
  return w;
}

// RTEC_AGG_BATCH env: rows up to this width use the warp-batched light pass (0: never)
static bool agg_batched(int d) {
  static int b = -1;
  if (b < 0) {
    const char* e = getenv("RTEC_AGG_BATCH");
    b = e ? atoi(e) : 128;
  }
  return d <= b;
}

// RTEC_AGG_DENSE env: hit density |E_curr| / Σ indeg(V_dst) below which a large scan of rows
// <= 128 floats uses the warp-batched light pass instead of one destination per warp
static float agg_dense_thr() {
  static float t = -1.f;
  if (t < 0.f) {
    const char* e = getenv("RTEC_AGG_DENSE");
    t = e ? static_cast<float>(atof(e)) : 0.3f;
    if (t < 0.f) t = 0.f;
  }
  return t;
}

// RTEC_AGG_BATCH_OCC env: resident CTAs per SM of the warp-batched pass (0: AggOcc, 6: A/B)
static int agg_batch_occ() {
  static int o = -1;
  if (o < 0) {
    const char* e = getenv("RTEC_AGG_BATCH_OCC");
    o = e ? atoi(e) : 0;
  }
  return o;
}

// RTEC_HEAVY_ORDER env: visit hub chunks in relative-position order (default 1; 0: destination-major)
static bool heavy_order() {
  static int o = -1;
  if (o < 0) {
    const char* e = getenv("RTEC_HEAVY_ORDER");
    o = e ? atoi(e) : 1;
  }
  return o != 0;
}

// heavy-destination plan (list, chunk offsets, chunk -> heavy map); partial rows of `pw` floats
template <bool FULL>
static int plan_heavy(const LayerArgs& a, AggRows rows, int64_t max_rows, int64_t max_edges, int pw, Ws& w,
                      cudaStream_t s, HeavyPlan& hp, bool every_long_run = false) {
  hp.heavy = w.alloc<int32_t>(max_rows + 1);
  hp.n_heavy = w.alloc<int64_t>(max_rows + 2 + 4);  // [0] heavy count, [1] chunks, [2] packed total
  hp.hoff = hp.n_heavy + 4;
  int64_t max_chunks = heavy_chunk_bound(max_edges);
  hp.cmap = w.alloc<int32_t>(max_chunks);
  hp.arrive = w.alloc<int32_t>(max_rows + 1);
  hp.part = w.alloc<float>(max_chunks * static_cast<int64_t>(pw));
  RTEC_WS_CHECK(w);
  RTEC_CUDA(cudaMemsetAsync(hp.n_heavy, 0, sizeof(int64_t) * 5, s));  // counts, packed total, hoff[0]
  HeavyFlagF hf{rows, a.g.in.len, (FULL || every_long_run) ? nullptr : a.f.n_src};
  Count cnt{rows.n_dev, max_rows};
  if (!rows.n_dev) cnt = Count{nullptr, rows.n_all};
  RTEC_TRY(exclusive_scan(HeavyPackF{hf}, cnt, max_rows, HeavyPackStore{rows, hp.heavy, hp.hoff}, hp.n_heavy + 2, w,
                          s));
  if (heavy_order()) {
    hp.okey = w.alloc<uint64_t>(max_chunks);
    hp.oval = w.alloc<uint32_t>(max_chunks);
    RTEC_WS_CHECK(w);
  }
  launch(k_chunk_map, kSMs * 4, kLBlk, 0, s, hp);
  RTEC_LAUNCH_CHECK("k_chunk_map");
  if (hp.okey) {
    uint64_t* kout = w.alloc<uint64_t>(max_chunks);
    uint32_t* order = w.alloc<uint32_t>(max_chunks);
    RTEC_WS_CHECK(w);
    RTEC_TRY(sort_pairs(hp.okey, hp.oval, kout, order, Count{hp.n_heavy + 1, max_chunks}, max_chunks, 8, w, s));
    hp.order = order;
  }
  return RTEC_OK;
}

// plan + light + heavy launches for one aggregation
template <bool FULL>
static int launch_aggregation(LayerArgs& a, AggRows rows, int64_t max_rows, int64_t max_edges, Ws& w,
                              cudaStream_t s) {
  const int d = a.d_agg;
  HeavyPlan hp{};
  RTEC_TRY(plan_heavy<FULL>(a, rows, max_rows, max_edges, d, w, s, hp));
  const int grid = kSMs * 8;
  // Feature slicing: one pass per `sw`-column slice keeps the gathered rows'
  // working set (|S| x sw x 4 B) small enough for the hot sources to stay in
  // L2 (126 MB); the plan above is shared by all passes.
  const int sw = agg_slice_width();
  bool ok = true;
  for (int c0 = 0; c0 < d && ok; c0 += (sw > 0 ? sw : d)) {
    a.c0 = c0;
    a.cw = sw > 0 ? (d - c0 < sw ? d - c0 : sw) : d;
    if (c0 > 0) RTEC_CUDA(cudaMemsetAsync(hp.arrive, 0, sizeof(int32_t) * (max_rows + 1), s));
    const bool sliced = a.cw <= 64;
    // The hub chunks (heavy) touch other destinations than the light pass: run them on a
    // side stream so each pass fills the other's tail (a fork / join the CUDA graph keeps).
    // Not while profiling (per-kernel events need the passes apart).
    cudaStream_t hs = g_prof_on ? s : side_stream();
    if (hs != s) {
      RTEC_CUDA(cudaEventRecord(side_fork(), s));
      RTEC_CUDA(cudaStreamWaitEvent(hs, side_fork(), 0));
    }
    {
      RTEC_PROF(FULL ? "k_agg_full_heavy" : "k_agg_inc_heavy", hs);
      ok = (sliced ? RTEC_SLICE_DISPATCH(a.cw, (launch(k_agg_heavy<VEC, K, FULL>, grid, kLBlk, 0, hs, a, rows, hp)))
                   : RTEC_ROW_DISPATCH(a.cw, (launch(k_agg_heavy<VEC, K, FULL>, grid, kLBlk, 0, hs, a, rows, hp))));
    }
    {
      RTEC_PROF(FULL ? "k_agg_full_light" : "k_agg_inc", s);
      if (!FULL && !sliced && agg_batched(a.cw)) {
        // both light-pass kernels are enqueued; each runs only in its hit-density regime
        LayerArgs ab = a, al = a;
        ab.pick = 1;
        al.pick = 2;
        ab.pick_thr = al.pick_thr = agg_dense_thr();
        if (agg_batch_occ() == 6)
          ok = ok && RTEC_ROW_DISPATCH(a.cw, (launch(k_agg_batch<VEC, K, 6>, grid, kLBlk, 0, s, ab, rows)));
        else
          ok = ok && RTEC_ROW_DISPATCH(a.cw, (launch(k_agg_batch<VEC, K>, grid, kLBlk, 0, s, ab, rows)));
        ok = ok && RTEC_ROW_DISPATCH(a.cw, (launch(k_agg_light<VEC, K, false>, grid, kLBlk, 0, s, al, rows)));
      } else
        ok = ok && (sliced ? RTEC_SLICE_DISPATCH(a.cw, (launch(k_agg_light<VEC, K, FULL>, grid, kLBlk, 0, s, a, rows)))
                           : RTEC_ROW_DISPATCH(a.cw, (launch(k_agg_light<VEC, K, FULL>, grid, kLBlk, 0, s, a, rows))));
    }
    if (hs != s) {
      RTEC_CUDA(cudaEventRecord(side_join(), hs));
      RTEC_CUDA(cudaStreamWaitEvent(s, side_join(), 0));
    }
  }
  if (!ok) {
    set_error("row width %d unsupported", d);
    return RTEC_SHAPE_ERROR;
  }
  RTEC_LAUNCH_CHECK("aggregation");
  return RTEC_OK;
}

// ------------------------------------------------------------------ dest-dependent sums (G-GCN, A-GNN)
// m(u, v) reads both endpoints (models.py:301-305, :326-331), so a destination
// whose own h_v changed (R(l) = V_dst(l) ∩ V_chg(l-1)) is summed
// over its whole post-batch in-run; every other destination keeps h_v and adds
//   ValueChange (u,v), u ∈ S(l), not inserted :  m(u_new, v) - m(u_old, v)
//   insert (u,v) :  + m(u_new, v)        delete (u,v) :  - m(u_old, v)
// to its cached sum.  Old rows of V_chg(l-1) sources come from the previous
// layer's DeltaLog (h) and the projection log (G-GCN gates), both by prev_slot.
template <int VEC, int K>
struct DstRow {
  float hv[K][VEC];  // h_v
  float pv[K][VEC];  // G-GCN: Wg_dst h_v
  float nv;          // A-GNN: |h_v|
};

__device__ __forceinline__ float sigmoid_ref(float x) {  // linalg.py:46-52 two-branch form
  if (x >= 0.f) return 1.f / (1.f + expf(-x));
  const float e = expf(x);
  return e / (1.f + e);
}

template <int VEC, int K>
__device__ __forceinline__ void dd_load_dst(const LayerArgs& a, int32_t v, DstRow<VEC, K>& D) {
  using R = RowAcc<VEC, K>;
  const int d = a.d_agg;
  R::load(a.st.H_in + static_cast<int64_t>(v) * d, d, D.hv);
  D.nv = 0.f;
  if (a.L.model == RTEC_MODEL_GGCN) {
    R::load(a.st.Z + static_cast<int64_t>(v) * 2 * d + d, d, D.pv);
  } else {
    float s2 = 0.f;
#pragma unroll
    for (int k = 0; k < K; ++k)
#pragma unroll
      for (int j = 0; j < VEC; ++j) s2 = fmaf(D.hv[k][j], D.hv[k][j], s2);
    D.nv = sqrtf(warp_sum(s2));
  }
}

// acc += sign * m(u, v) for the source row hu (and its gate projection ps)
template <int VEC, int K>
__device__ __forceinline__ void dd_msg(const LayerArgs& a, const DstRow<VEC, K>& D, const float (&hu)[K][VEC],
                                       const float (&ps)[K][VEC], float sign, RowAcc<VEC, K>& acc) {
  if (a.L.model == RTEC_MODEL_GGCN) {
#pragma unroll
    for (int k = 0; k < K; ++k)
#pragma unroll
      for (int j = 0; j < VEC; ++j) acc.v[k][j] = fmaf(sign * sigmoid_ref(ps[k][j] + D.pv[k][j]), hu[k][j], acc.v[k][j]);
  } else {
    float dot = 0.f, n2 = 0.f;
#pragma unroll
    for (int k = 0; k < K; ++k)
#pragma unroll
      for (int j = 0; j < VEC; ++j) {
        dot = fmaf(hu[k][j], D.hv[k][j], dot);
        n2 = fmaf(hu[k][j], hu[k][j], n2);
      }
    dot = warp_sum(dot);
    const float nu = sqrtf(warp_sum(n2));
    const float c = (nu > 0.f && D.nv > 0.f) ? a.L.scalar * dot / (nu * D.nv) : 0.f;  // models.py:327-331
    acc.fma(hu, sign * c);
  }
}

// new (or old) rows of source u: h and, for G-GCN, the source gate projection
template <int VEC, int K>
__device__ __forceinline__ void dd_src(const LayerArgs& a, int32_t u, bool old, float (&h)[K][VEC],
                                       float (&ps)[K][VEC]) {
  using R = RowAcc<VEC, K>;
  const int d = a.d_agg;
  const bool logged = old && a.prev_bm_dst && bm_test(a.prev_bm_dst, u);
  const int64_t slot = logged ? static_cast<int64_t>(a.prev_slot[u]) : 0;
  R::load(logged ? a.st.log_in + slot * d : a.st.H_in + static_cast<int64_t>(u) * d, d, h);
  if (a.L.model == RTEC_MODEL_GGCN)
    R::load(logged ? a.st.Z_log + slot * 2 * d : a.st.Z + static_cast<int64_t>(u) * 2 * d, d, ps);
}

// in-run edges [e0, e1) of v: every edge when `full`, else the ValueChange ones (new - old)
template <int VEC, int K>
__device__ __forceinline__ void dd_edges(const LayerArgs& a, const DstRow<VEC, K>& D, int64_t beg, int32_t e0,
                                         int32_t e1, int64_t p, int64_t q, bool full, RowAcc<VEC, K>& acc) {
  for (int32_t c0 = e0; c0 < e1; c0 += 32) {
    const int32_t j = c0 + lane_id();
    int32_t u = 0;
    bool hit = false;
    if (j < e1) {
      u = a.g.in.nbr[beg + j];
      hit = full || (bm_test(a.f.bm_src, u) && !in_range_has(a.b.i_src, p, q, u) && a.prev_bm_dst &&
                     bm_test(a.prev_bm_dst, u));  // S(l) sources whose row changed (Dg is empty here)
    }
    unsigned m = __ballot_sync(0xffffffffu, hit);
    while (m) {
      const int src = __ffs(m) - 1;
      m &= m - 1;
      const int32_t uu = __shfl_sync(0xffffffffu, u, src);
      float h[K][VEC], ps[K][VEC];
      dd_src<VEC, K>(a, uu, false, h, ps);
      dd_msg<VEC, K>(a, D, h, ps, 1.f, acc);
      if (!full) {
        dd_src<VEC, K>(a, uu, true, h, ps);
        dd_msg<VEC, K>(a, D, h, ps, -1.f, acc);
      }
    }
  }
}

template <int VEC, int K>
__device__ __forceinline__ void dd_struct(const LayerArgs& a, const DstRow<VEC, K>& D, int64_t p, int64_t q,
                                          RowAcc<VEC, K>& acc) {
  for (int64_t k = p; k < q; ++k) {
    const int32_t u = a.b.i_src[k];
    const bool ins = a.b.i_op[k] == RTEC_OP_INSERT;
    float h[K][VEC], ps[K][VEC];
    dd_src<VEC, K>(a, u, !ins, h, ps);
    dd_msg<VEC, K>(a, D, h, ps, ins ? 1.f : -1.f, acc);
  }
}

// per-destination setup shared by the light / heavy kernels
struct DdRow {
  int64_t beg, p, q;
  int32_t len, indeg, had;
  bool full;
};
template <bool FULL>
__device__ __forceinline__ DdRow dd_row(const LayerArgs& a, int32_t v) {
  DdRow r{a.g.in.beg[v], 0, 0, a.g.in.len[v], 0, 0, true};
  r.indeg = r.len;
  if (!FULL) {
    const int2 rg = reinterpret_cast<const int2*>(a.b.irange)[v];
    if (rg.x >= 0) {
      r.p = rg.x;
      r.q = rg.x + rg.y;
    }
    r.indeg = a.g.in_deg[v];
    r.had = a.g.in_deg_prev[v];
    r.full = a.prev_bm_dst && bm_test(a.prev_bm_dst, v);  // v ∈ R(l)
  }
  return r;
}

// S_v: the new sum (R(l) / FULL) or the cached sum plus the signed changes
template <int VEC, int K, bool FULL>
__device__ __forceinline__ void dd_finalize(const LayerArgs& a, int64_t i, int32_t v, const DdRow& r,
                                            RowAcc<VEC, K>& acc) {
  using R = RowAcc<VEC, K>;
  if (FULL) {
    agg_finalize<VEC, K, true>(a, i, v, r.len, acc);
    return;
  }
  R pre;
  pre.zero();
  if (!r.full && r.indeg > 0 && r.had > 0) R::load(a.st.S + srow(a, v) * a.d_agg, a.d_agg, pre.v);
  agg_finalize<VEC, K, false>(a, i, v, r.len, acc, &pre, r.indeg);
}

template <int VEC, int K, bool FULL>
__global__ void __launch_bounds__(kLBlk) k_dd_light(LayerArgs a, AggRows rows) {
  RTEC_PDL_ENTRY();
  using R = RowAcc<VEC, K>;
  if (!FULL && err_set(a.err)) return;
  const int64_t nr = rows.count();
  const bool scan = FULL || *a.f.n_src > 0;
  int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < nr; i += nw) {
    const int32_t v = rows.at(i);
    const DdRow r = dd_row<FULL>(a, v);
    if (scan && r.len > kChunk) continue;  // heavy pass
    DstRow<VEC, K> D;
    dd_load_dst<VEC, K>(a, v, D);
    R acc;
    acc.zero();
    if (scan) dd_edges<VEC, K>(a, D, r.beg, 0, r.len, r.p, r.q, r.full, acc);
    if (!FULL && !r.full) dd_struct<VEC, K>(a, D, r.p, r.q, acc);
    dd_finalize<VEC, K, FULL>(a, i, v, r, acc);
  }
}

template <int VEC, int K, bool FULL>
__global__ void __launch_bounds__(kLBlk) k_dd_heavy(LayerArgs a, AggRows rows, HeavyPlan hp) {
  RTEC_PDL_ENTRY();
  using R = RowAcc<VEC, K>;
  if (!FULL && err_set(a.err)) return;
  const int64_t nh = *hp.n_heavy;
  if (nh == 0) return;
  const int64_t T = hp.hoff[nh];
  const int d = a.d_agg;
  int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t tt = warp; tt < T; tt += nw) {
    const int64_t t = hp.order ? static_cast<int64_t>(hp.order[tt]) : tt;
    const int32_t j = hp.cmap[t];
    const int64_t c0 = hp.hoff[j];
    const int32_t nch = static_cast<int32_t>(hp.hoff[j + 1] - c0);
    const int32_t c = static_cast<int32_t>(t - c0);
    const int64_t i = hp.heavy[j];
    const int32_t v = rows.at(i);
    const DdRow r = dd_row<FULL>(a, v);
    DstRow<VEC, K> D;
    dd_load_dst<VEC, K>(a, v, D);
    R acc;
    acc.zero();
    const int32_t e0 = c * kChunk, e1 = min(r.len, e0 + kChunk);
    dd_edges<VEC, K>(a, D, r.beg, e0, e1, r.p, r.q, r.full, acc);
    if (!FULL && !r.full && c == 0) dd_struct<VEC, K>(a, D, r.p, r.q, acc);
    acc.store(hp.part + t * d, d);
    __threadfence();
    __syncwarp();  // every lane's partial is fenced before the arrival is published
    int old = 0;
    if (lane_id() == 0) old = atomicAdd(hp.arrive + j, 1);
    old = __shfl_sync(0xffffffffu, old, 0);
    if (old != nch - 1) continue;
    __threadfence();
    acc.zero();
    sum_partials<VEC, K>(hp.part + c0 * d, d, d, nch, acc);  // chunk order: deterministic
    dd_finalize<VEC, K, FULL>(a, i, v, r, acc);
  }
}

template <bool FULL>
static int launch_dd(LayerArgs& a, AggRows rows, int64_t max_rows, int64_t max_edges, Ws& w, cudaStream_t s) {
  const int d = a.d_agg;
  a.c0 = 0;
  a.cw = d;
  HeavyPlan hp{};
  RTEC_TRY(plan_heavy<FULL>(a, rows, max_rows, max_edges, d, w, s, hp));
  const int grid = kSMs * 8;
  bool ok;
  {
    RTEC_PROF(FULL ? "k_dd_full_heavy" : "k_dd_inc_heavy", s);
    ok = RTEC_ROW_DISPATCH(d, (launch(k_dd_heavy<VEC, K, FULL>, grid, kLBlk, 0, s, a, rows, hp)));
  }
  {
    RTEC_PROF(FULL ? "k_dd_full_light" : "k_dd_inc", s);
    ok = ok && RTEC_ROW_DISPATCH(d, (launch(k_dd_light<VEC, K, FULL>, grid, kLBlk, 0, s, a, rows)));
  }
  if (!ok) {
    set_error("row width %d unsupported", d);
    return RTEC_SHAPE_ERROR;
  }
  RTEC_LAUNCH_CHECK("k_dd");
  return RTEC_OK;
}

// ------------------------------------------------------------------ GIN-max (K16)
// a_v = max_{u in N_in(v)} h_u elementwise (0 for an empty neighbourhood); the
// cached S row is the max itself.  Incremental (retract-and-recompute): new
// values of inserted / value-changed sources can only raise the max, so
// S' = max(S, new rows) -- unless a retracted value (old row of a deleted or
// value-changed source) attained the cached max in some column and did not
// stay at least as large, in which case that destination is re-maxed over its
// whole post-batch in-run.  Max is exact, so S' is bit-identical to a full
// recompute in the same precision.
template <int VEC, int K>
__device__ __forceinline__ void max_row(const float (&r)[K][VEC], RowAcc<VEC, K>& acc) {
#pragma unroll
  for (int k = 0; k < K; ++k)
#pragma unroll
    for (int j = 0; j < VEC; ++j) acc.v[k][j] = fmaxf(acc.v[k][j], r[k][j]);
}

template <int VEC, int K>
__device__ __forceinline__ void max_neg_inf(RowAcc<VEC, K>& acc) {
#pragma unroll
  for (int k = 0; k < K; ++k)
#pragma unroll
    for (int j = 0; j < VEC; ++j) acc.v[k][j] = -INFINITY;
}

// acc = max(acc, chunk partial rows 0..nch-1), 4 rows in flight
template <int VEC, int K>
__device__ __forceinline__ void max_partials(const float* part, int d, int32_t nch, RowAcc<VEC, K>& acc) {
  for (int32_t cc = 0; cc < nch; cc += 4) {
    float r[4][K][VEC];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const int col = lane_id() + 32 * k;
#pragma unroll
        for (int jj = 0; jj < VEC; ++jj)
          r[u][k][jj] = (cc + u < nch && col * VEC < d) ? __ldcg(part + (cc + u) * d + col * VEC + jj) : -INFINITY;
      }
#pragma unroll
    for (int u = 0; u < 4; ++u) max_row<VEC, K>(r[u], acc);
  }
}

// max over the current rows of in-run positions [e0, e1), 4 rows in flight
template <int VEC, int K>
__device__ __forceinline__ void max_run(const LayerArgs& a, int64_t beg, int32_t e0, int32_t e1,
                                        RowAcc<VEC, K>& acc) {
  using R = RowAcc<VEC, K>;
  const int d = a.d_agg;
  const int lane = lane_id();
  for (int32_t c0 = e0; c0 < e1; c0 += 32) {
    int32_t j = c0 + lane;
    int32_t u = j < e1 ? a.g.in.nbr[beg + j] : 0;
    int cnt = min(32, e1 - c0);
    for (int t = 0; t < cnt; t += 4) {
      float r[4][K][VEC];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        int32_t uu = __shfl_sync(0xffffffffu, u, min(t + q, cnt - 1));
        R::load(a.st.H_in + static_cast<int64_t>(uu) * d, d, r[q]);
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) max_row<VEC, K>(r[q], acc);  // repeats of the last row are harmless
    }
  }
}

// incremental candidates of in-run positions [e0, e1) (+ structural edges when
// p < q): new rows of value-changed / inserted sources raise the max; returns
// whether a retracted old value attained the cached max sv in some column
template <int VEC, int K>
__device__ __forceinline__ bool max_incremental(const LayerArgs& a, int64_t beg, int32_t e0, int32_t e1, int64_t p,
                                                int64_t q, bool with_struct, const float (&sv)[K][VEC],
                                                RowAcc<VEC, K>& acc) {
  using R = RowAcc<VEC, K>;
  const int d = a.d_agg;
  const int lane = lane_id();
  bool retract = false;
  if (*a.f.n_src > 0) {
    for (int32_t c0 = e0; c0 < e1; c0 += 32) {
      int32_t j = c0 + lane;
      int32_t u = 0;
      bool hit = false;
      if (j < e1) {
        u = a.g.in.nbr[beg + j];
        hit = bm_test(a.f.bm_src, u) && !in_range_has(a.b.i_src, p, q, u);
      }
      unsigned m = __ballot_sync(0xffffffffu, hit);
      while (m) {
        int32_t uu[2];
        int cnt = 0;
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          int src = m ? __ffs(m) - 1 : 0;
          if (m) {
            m &= m - 1;
            cnt = t + 1;
          }
          uu[t] = __shfl_sync(0xffffffffu, u, src);
        }
        float hn[2][K][VEC], ho[2][K][VEC];
#pragma unroll
        for (int t = 0; t < 2; ++t)
          if (t < cnt) {
            R::load(a.st.H_in + static_cast<int64_t>(uu[t]) * d, d, hn[t]);
            const float* orow = a.st.H_in + static_cast<int64_t>(uu[t]) * d;
            if (a.prev_bm_dst && bm_test(a.prev_bm_dst, uu[t]))
              orow = a.st.log_in + static_cast<int64_t>(a.prev_slot[uu[t]]) * d;
            R::load(orow, d, ho[t]);
          }
#pragma unroll
        for (int t = 0; t < 2; ++t)
          if (t < cnt) {
            max_row<VEC, K>(hn[t], acc);
#pragma unroll
            for (int k = 0; k < K; ++k)
#pragma unroll
              for (int jj = 0; jj < VEC; ++jj)
                retract |= R::has(k, d) && ho[t][k][jj] >= sv[k][jj] && hn[t][k][jj] < ho[t][k][jj];
          }
      }
    }
  }
  if (with_struct) {
    for (int64_t kk = p; kk < q; ++kk) {
      int32_t u = a.b.i_src[kk];
      float r[K][VEC];
      if (a.b.i_op[kk] == RTEC_OP_INSERT) {
        R::load(a.st.H_in + static_cast<int64_t>(u) * d, d, r);
        max_row<VEC, K>(r, acc);
      } else {
        const float* orow = a.st.H_in + static_cast<int64_t>(u) * d;
        if (a.prev_bm_dst && bm_test(a.prev_bm_dst, u)) orow = a.st.log_in + static_cast<int64_t>(a.prev_slot[u]) * d;
        R::load(orow, d, r);
#pragma unroll
        for (int k = 0; k < K; ++k)
#pragma unroll
          for (int jj = 0; jj < VEC; ++jj) retract |= R::has(k, d) && r[k][jj] >= sv[k][jj];
      }
    }
  }
  return __any_sync(0xffffffffu, retract);
}

// S = a_v, GEMM input h_v + a_v (models.py:187-189); empty neighbourhood -> 0
template <int VEC, int K>
__device__ __forceinline__ void max_finalize(const LayerArgs& a, int64_t i, int32_t v, int32_t len,
                                             RowAcc<VEC, K>& acc) {
  using R = RowAcc<VEC, K>;
  const int d = a.d_agg;
  if (len == 0) acc.zero();
  acc.store(a.st.S + srow(a, v) * d, d);
  R out;
  out.zero();
  out.add(acc.v);
  float h[K][VEC];
  R::load(a.st.H_in + static_cast<int64_t>(v) * d, d, h);
  out.add(h);
  if (a.tc_nkb > 0) out.store_tiled(a.st.gemm_in, i, 0, d, d, a.tc_nkb);
  else out.store(a.st.gemm_in + i * d, d);
}

__device__ __forceinline__ int2 irange_of(const LayerArgs& a, int32_t v) {
  int2 rg = reinterpret_cast<const int2*>(a.b.irange)[v];
  return rg.x >= 0 ? make_int2(rg.x, rg.x + rg.y) : make_int2(0, 0);
}

// When most sources changed (|S(l)| > n/8), nearly every cached max is retracted
// in some column; re-maxing every affected destination directly (1 row gather per
// in-edge) then beats the incremental pass (2 per changed edge) plus rescans.
template <bool FULL>
__device__ __forceinline__ bool max_direct(const LayerArgs& a) {
  return !FULL && (*a.f.n_src) * 8 > a.g.n;
}

// destinations with <= kChunk scanned edges: one warp each, re-max in place on retract
template <int VEC, int K, bool FULL>
__global__ void __launch_bounds__(kLBlk) k_max_light(LayerArgs a, AggRows rows) {
  RTEC_PDL_ENTRY();
  using R = RowAcc<VEC, K>;
  if (!FULL && err_set(a.err)) return;
  const int d = a.d_agg;
  const int64_t nr = rows.count();
  const bool direct = max_direct<FULL>(a);
  int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < nr; i += nw) {
    int32_t v = rows.at(i);
    int64_t beg = a.g.in.beg[v];
    int32_t len = a.g.in.len[v];
    if (len > kChunk) continue;  // heavy pass
    R acc;
    max_neg_inf<VEC, K>(acc);
    bool rescan = FULL || direct;
    if (!rescan && len > 0) {
      int2 pq = irange_of(a, v);
      const bool had = a.g.in_deg_prev[v] > 0;
      float sv[K][VEC];
      R::load_rw(a.st.S + srow(a, v) * d, d, sv);
      bool retract = max_incremental<VEC, K>(a, beg, 0, len, pq.x, pq.y, true, sv, acc);
      rescan = had && retract;
      if (!rescan && had) max_row<VEC, K>(sv, acc);
    }
    if (rescan) {
      max_neg_inf<VEC, K>(acc);
      max_run<VEC, K>(a, beg, 0, len, acc);
    }
    max_finalize<VEC, K>(a, i, v, len, acc);
  }
}

// Rescan queue of heavy destinations whose cached max was retracted
struct MaxRescan {
  int64_t* n;       // [1] queued destinations
  int64_t* total;   // [1] queued chunks
  int32_t* dest;    // [max_rows] heavy index j of each queued destination
  int64_t* off;     // [max_rows] first chunk of each queued destination
  int32_t* cmap;    // [max_chunks] chunk -> queue entry
  int32_t* arrive;  // [max_rows]
  int32_t* flag;    // [max_rows] per heavy destination: retract seen by some chunk
  float* part;      // [max_chunks, d]
};

// heavy destinations, pass 1: chunked incremental candidates (FULL: chunked max);
// the last chunk to arrive finalizes, or queues the destination for a rescan
template <int VEC, int K, bool FULL>
__global__ void __launch_bounds__(kLBlk) k_max_heavy(LayerArgs a, AggRows rows, HeavyPlan hp, MaxRescan rq) {
  RTEC_PDL_ENTRY();
  using R = RowAcc<VEC, K>;
  if (!FULL && err_set(a.err)) return;
  const int64_t nh = *hp.n_heavy;
  if (nh == 0) return;
  const int64_t T = hp.hoff[nh];
  const int d = a.d_agg;
  const bool direct = max_direct<FULL>(a);
  int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t tt = warp; tt < T; tt += nw) {
    const int64_t t = hp.order ? static_cast<int64_t>(hp.order[tt]) : tt;
    int32_t j = hp.cmap[t];
    int64_t c0 = hp.hoff[j];
    int32_t nch = static_cast<int32_t>(hp.hoff[j + 1] - c0);
    int32_t c = static_cast<int32_t>(t - c0);
    int64_t i = hp.heavy[j];
    int32_t v = rows.at(i);
    int64_t beg = a.g.in.beg[v];
    int32_t len = a.g.in.len[v];
    int32_t e0 = c * kChunk, e1 = min(len, e0 + kChunk);
    R acc;
    max_neg_inf<VEC, K>(acc);
    float sv[K][VEC];
    bool had = false;
    if (FULL || direct) {
      max_run<VEC, K>(a, beg, e0, e1, acc);
    } else {
      int2 pq = irange_of(a, v);
      had = a.g.in_deg_prev[v] > 0;
      R::load_rw(a.st.S + srow(a, v) * d, d, sv);
      bool retract = max_incremental<VEC, K>(a, beg, e0, e1, pq.x, pq.y, c == 0, sv, acc);
      if (retract && had && lane_id() == 0) atomicOr(rq.flag + j, 1);
    }
    acc.store(hp.part + t * d, d);
    __threadfence();
    __syncwarp();  // every lane's partial is fenced before the arrival is published
    int old = 0;
    if (lane_id() == 0) old = atomicAdd(hp.arrive + j, 1);
    old = __shfl_sync(0xffffffffu, old, 0);
    if (old != nch - 1) continue;
    __threadfence();
    if (!FULL && *reinterpret_cast<volatile int32_t*>(rq.flag + j)) {
      // queue a chunked re-max over the whole post-batch in-run (pass 2)
      int64_t e = 0, base = 0;
      if (lane_id() == 0) {
        e = atomicAdd(reinterpret_cast<unsigned long long*>(rq.n), 1ull);
        base = atomicAdd(reinterpret_cast<unsigned long long*>(rq.total), static_cast<unsigned long long>(nch));
        rq.dest[e] = j;
        rq.off[e] = base;
        rq.arrive[e] = 0;
      }
      e = __shfl_sync(0xffffffffu, e, 0);
      base = __shfl_sync(0xffffffffu, base, 0);
      for (int32_t cc = lane_id(); cc < nch; cc += 32) rq.cmap[base + cc] = static_cast<int32_t>(e);
      continue;
    }
    max_neg_inf<VEC, K>(acc);
    max_partials<VEC, K>(hp.part + c0 * d, d, nch, acc);
    if (!FULL && had) max_row<VEC, K>(sv, acc);
    max_finalize<VEC, K>(a, i, v, len, acc);
  }
}

// heavy destinations, pass 2: chunked re-max of the queued destinations
template <int VEC, int K>
__global__ void __launch_bounds__(kLBlk) k_max_rescan(LayerArgs a, AggRows rows, HeavyPlan hp, MaxRescan rq) {
  RTEC_PDL_ENTRY();
  using R = RowAcc<VEC, K>;
  if (err_set(a.err)) return;
  const int64_t T = *rq.total;
  const int d = a.d_agg;
  int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t t = warp; t < T; t += nw) {
    int32_t e = rq.cmap[t];
    int32_t j = rq.dest[e];
    int64_t c0 = rq.off[e];
    int32_t nch = static_cast<int32_t>(hp.hoff[j + 1] - hp.hoff[j]);
    int32_t c = static_cast<int32_t>(t - c0);
    int64_t i = hp.heavy[j];
    int32_t v = rows.at(i);
    int64_t beg = a.g.in.beg[v];
    int32_t len = a.g.in.len[v];
    R acc;
    max_neg_inf<VEC, K>(acc);
    max_run<VEC, K>(a, beg, c * kChunk, min(len, (c + 1) * kChunk), acc);
    acc.store(rq.part + t * d, d);
    __threadfence();
    __syncwarp();  // every lane's partial is fenced before the arrival is published
    int old = 0;
    if (lane_id() == 0) old = atomicAdd(rq.arrive + e, 1);
    old = __shfl_sync(0xffffffffu, old, 0);
    if (old != nch - 1) continue;
    __threadfence();
    max_neg_inf<VEC, K>(acc);
    max_partials<VEC, K>(rq.part + c0 * d, d, nch, acc);
    max_finalize<VEC, K>(a, i, v, len, acc);
  }
}

template <bool FULL>
static int launch_max(LayerArgs& a, AggRows rows, int64_t max_rows, int64_t max_edges, Ws& w, cudaStream_t s) {
  const int d = a.d_agg;
  const int grid = kSMs * 8;
  HeavyPlan hp{};
  RTEC_TRY(plan_heavy<FULL>(a, rows, max_rows, max_edges, d, w, s, hp, true));
  MaxRescan rq{};
  int64_t max_chunks = heavy_chunk_bound(max_edges);
  rq.n = w.alloc<int64_t>(2);
  rq.total = rq.n + 1;
  rq.dest = w.alloc<int32_t>(max_rows + 1);
  rq.off = w.alloc<int64_t>(max_rows + 1);
  rq.cmap = w.alloc<int32_t>(max_chunks);
  rq.arrive = w.alloc<int32_t>(max_rows + 1);
  rq.flag = w.alloc<int32_t>(max_rows + 1);
  rq.part = FULL ? nullptr : w.alloc<float>(max_chunks * static_cast<int64_t>(d));
  RTEC_WS_CHECK(w);
  RTEC_CUDA(cudaMemsetAsync(rq.n, 0, sizeof(int64_t) * 2, s));
  RTEC_CUDA(cudaMemsetAsync(rq.flag, 0, sizeof(int32_t) * (max_rows + 1), s));
  RTEC_PROF(FULL ? "k_max_full" : "k_max_inc", s);
  bool ok = RTEC_ROW_DISPATCH(d, (launch(k_max_light<VEC, K, FULL>, grid, kLBlk, 0, s, a, rows),
                                  launch(k_max_heavy<VEC, K, FULL>, grid, kLBlk, 0, s, a, rows, hp, rq)));
  if (ok && !FULL) ok = RTEC_ROW_DISPATCH(d, (launch(k_max_rescan<VEC, K>, grid, kLBlk, 0, s, a, rows, hp, rq)));
  if (!ok) {
    set_error("row width %d unsupported", d);
    return RTEC_SHAPE_ERROR;
  }
  RTEC_LAUNCH_CHECK("k_max");
  return RTEC_OK;
}

// ------------------------------------------------------------------ GAT (K13-K15)
// Alg. 3 for v in V_dst(l) \ R(l): per ValueChange edge
// + a_new Z_new(u) - a_old Z_old(u) with a = exp(leaky_0.2(el_v + er_u)) per head
// (dst half first, models.py:266-271), per structural edge +/- a Z; the
// attention sums are the context.  v in R(l) (and every vertex at bootstrap):
// full edge softmax over the post-batch in-run (models.py:431-458).  Gathers
// run 2-4 rows deep per warp like the sum aggregation; destinations with more
// than kChunk scanned edges are split into chunks reduced in chunk order.
constexpr int kHMax = 8;

template <int VEC>
__device__ __forceinline__ int chunk_head(int k, int dh) {
  return ((lane_id() + 32 * k) * VEC) / dh;
}

struct GatEdgeState {
  float elh[kHMax];  // el_v per head (destination half of the logit)
};


// contributions of in-run positions [e0, e1) of v: all edges (recompute) or the
// ValueChange edges (sources in S(l), edge not inserted) -> acc, cacc
template <int VEC, int K, int UNR = 1>
__device__ __forceinline__ void gat_edges(const LayerArgs& a, const GatEdgeState& es, int64_t beg, int32_t e0,
                                          int32_t e1, int64_t p, int64_t q, bool all, RowAcc<VEC, K>& acc,
                                          float (&cacc)[K]) {
  using R = RowAcc<VEC, K>;
  const int d = a.L.d_out, H = a.L.heads, dh = d / H;
  const int lane = lane_id();
  // The attention of a 32-edge window is evaluated once per edge, lane j for edge j,
  // all heads (same inputs and expf as before), into a per-warp shared-memory table;
  // the gather loop then reads the head of its own columns from it (one LDS per chunk
  // instead of an er load + expf per lane per edge, no per-head register arrays).
  __shared__ float s_att[kLBlk / 32][2][32][kHMax + 1];
  float(*an)[kHMax + 1] = s_att[threadIdx.x >> 5][0];
  float(*ao)[kHMax + 1] = s_att[threadIdx.x >> 5][1];
  int hk[K];
#pragma unroll
  for (int k = 0; k < K; ++k) hk[k] = R::has(k, d) ? chunk_head<VEC>(k, dh) : 0;
  // the next window's source ids are requested before this window's gathers
  int32_t u_nx = e0 + lane < e1 ? a.g.in.nbr[beg + e0 + lane] : 0;
  for (int32_t c0 = e0; c0 < e1; c0 += 32) {
    const int32_t j = c0 + lane;
    int32_t u = u_nx, sl = 0;
    if (j + 32 < e1) u_nx = a.g.in.nbr[beg + j + 32];
    bool hit = false;
    if (j < e1) {
      hit = all || (bm_test(a.f.bm_src, u) && !in_range_has(a.b.i_src, p, q, u));
    }
    if (hit && !all) sl = a.prev_slot[u];
    unsigned m = __ballot_sync(0xffffffffu, hit);
    if (!m) continue;
    if (hit) {
#pragma unroll
      for (int h = 0; h < kHMax; ++h)
        if (h < H) {
          an[lane][h] = expf(leaky02(es.elh[h] + __ldg(a.st.er + static_cast<int64_t>(u) * H + h)));
          if (!all) ao[lane][h] = expf(leaky02(es.elh[h] + __ldg(a.st.er_log + static_cast<int64_t>(sl) * H + h)));
        }
    }
    __syncwarp();
    if constexpr (UNR == 2) {
      // two edges' (Z, Z_log) row pairs in flight per warp -- or, for a recompute (no
      // DeltaLog rows), four edges' Z rows in the same registers; accumulated in edge
      // order (same sums)
      const int32_t v2 = all ? u : sl;  // the second pair: log slots or two more sources
      const float* zb = all ? a.st.Z : a.st.Z_log;
      while (m) {
        const int s0 = __ffs(m) - 1;
        m &= m - 1;
        const int s1 = m ? __ffs(m) - 1 : -1;
        if (m) m &= m - 1;
        int s2 = -1, s3 = -1;
        if (all) {
          s2 = m ? __ffs(m) - 1 : -1;
          if (m) m &= m - 1;
          s3 = m ? __ffs(m) - 1 : -1;
          if (m) m &= m - 1;
        }
        const int s1c = s1 >= 0 ? s1 : s0;
        const int t0 = all ? (s2 >= 0 ? s2 : s0) : s0;
        const int t1 = all ? (s3 >= 0 ? s3 : s0) : s1c;
        const int32_t u0 = __shfl_sync(0xffffffffu, u, s0), u1 = __shfl_sync(0xffffffffu, u, s1c);
        const int32_t x0 = __shfl_sync(0xffffffffu, v2, t0), x1 = __shfl_sync(0xffffffffu, v2, t1);
        const bool b0 = all ? s2 >= 0 : true, b1 = all ? s3 >= 0 : s1 >= 0;
        float zn0[K][VEC], zo0[K][VEC], zn1[K][VEC], zo1[K][VEC];
        R::load(a.st.Z + static_cast<int64_t>(u0) * d, d, zn0);
        if (b0) R::load(zb + static_cast<int64_t>(x0) * d, d, zo0);
        if (s1 >= 0) R::load(a.st.Z + static_cast<int64_t>(u1) * d, d, zn1);
        if (b1) R::load(zb + static_cast<int64_t>(x1) * d, d, zo1);
        if (all) {
#pragma unroll
          for (int k = 0; k < K; ++k) {
            const float w0 = an[s0][hk[k]];
            cacc[k] += w0;
#pragma unroll
            for (int jj = 0; jj < VEC; ++jj) acc.v[k][jj] += w0 * zn0[k][jj];
            if (s1 >= 0) {
              const float w1 = an[s1][hk[k]];
              cacc[k] += w1;
#pragma unroll
              for (int jj = 0; jj < VEC; ++jj) acc.v[k][jj] += w1 * zn1[k][jj];
            }
            if (b0) {
              const float w2 = an[t0][hk[k]];
              cacc[k] += w2;
#pragma unroll
              for (int jj = 0; jj < VEC; ++jj) acc.v[k][jj] += w2 * zo0[k][jj];
            }
            if (b1) {
              const float w3 = an[t1][hk[k]];
              cacc[k] += w3;
#pragma unroll
              for (int jj = 0; jj < VEC; ++jj) acc.v[k][jj] += w3 * zo1[k][jj];
            }
          }
          continue;
        }
#pragma unroll
        for (int k = 0; k < K; ++k) {
          const float wn = an[s0][hk[k]];
          const float wo = ao[s0][hk[k]];
          cacc[k] += wn - wo;
#pragma unroll
          for (int jj = 0; jj < VEC; ++jj) acc.v[k][jj] += fmaf(-wo, zo0[k][jj], wn * zn0[k][jj]);
        }
        if (s1 >= 0) {
#pragma unroll
          for (int k = 0; k < K; ++k) {
            const float wn = an[s1][hk[k]];
            const float wo = ao[s1][hk[k]];
            cacc[k] += wn - wo;
#pragma unroll
            for (int jj = 0; jj < VEC; ++jj) acc.v[k][jj] += fmaf(-wo, zo1[k][jj], wn * zn1[k][jj]);
          }
        }
      }
    } else {
      while (m) {
        const int src = __ffs(m) - 1;
        m &= m - 1;
        const int32_t uu = __shfl_sync(0xffffffffu, u, src);
        const int32_t ss = __shfl_sync(0xffffffffu, sl, src);
        float zn[K][VEC], zo[K][VEC];
        R::load(a.st.Z + static_cast<int64_t>(uu) * d, d, zn);
        if (!all) R::load(a.st.Z_log + static_cast<int64_t>(ss) * d, d, zo);
#pragma unroll
        for (int k = 0; k < K; ++k) {
          const float wn = an[src][hk[k]];
          const float wo = all ? 0.f : ao[src][hk[k]];
          cacc[k] += all ? wn : wn - wo;
#pragma unroll
          for (int jj = 0; jj < VEC; ++jj) {
            float x = wn * zn[k][jj];
            if (!all) x = fmaf(-wo, zo[k][jj], x);
            acc.v[k][jj] += x;
          }
        }
      }
    }
    __syncwarp();
  }
}

// structural edges of v (applied inserts / deletes), Alg. 3 with signed attention
template <int VEC, int K>
__device__ __forceinline__ void gat_struct(const LayerArgs& a, const GatEdgeState& es, int64_t p, int64_t q,
                                           RowAcc<VEC, K>& acc, float (&cacc)[K]) {
  using R = RowAcc<VEC, K>;
  const int d = a.L.d_out, H = a.L.heads, dh = d / H;
  for (int64_t kk = p; kk < q; ++kk) {
    int32_t u = a.b.i_src[kk];
    bool ins = a.b.i_op[kk] == RTEC_OP_INSERT;
    const float* zrow = a.st.Z + static_cast<int64_t>(u) * d;
    const float* errow = a.st.er + static_cast<int64_t>(u) * H;
    if (!ins && a.prev_bm_dst && bm_test(a.prev_bm_dst, u)) {
      int32_t sl = a.prev_slot[u];
      zrow = a.st.Z_log + static_cast<int64_t>(sl) * d;
      errow = a.st.er_log + static_cast<int64_t>(sl) * H;
    }
    float z[K][VEC];
    R::load(zrow, d, z);
    float sgn = ins ? 1.f : -1.f;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      float at = 0.f;
      if (R::has(k, d)) {
        const int h = chunk_head<VEC>(k, dh);
        float elv = 0.f;
#pragma unroll
        for (int hh = 0; hh < kHMax; ++hh)  // static index: keeps es.elh in registers
          if (hh == h) elv = es.elh[hh];
        at = expf(leaky02(elv + errow[h]));
      }
      cacc[k] += sgn * at;
#pragma unroll
      for (int jj = 0; jj < VEC; ++jj) acc.v[k][jj] = fmaf(sgn * at, z[k][jj], acc.v[k][jj]);
    }
  }
}

template <int VEC, int K>
__device__ __forceinline__ void gat_state(const LayerArgs& a, int32_t v, GatEdgeState& es) {
  const int H = a.L.heads;
#pragma unroll
  for (int h = 0; h < kHMax; ++h) {
    es.elh[h] = h < H ? __ldg(a.st.el + static_cast<int64_t>(v) * H + h) : 0.f;
  }
}

// S / ctx update, zero-in-degree rule, DeltaLog, h = elu(S / ctx) (models.py:280-282)
template <int VEC, int K, bool FULL>
__device__ __forceinline__ void gat_finalize(const LayerArgs& a, int64_t i, int32_t v, int32_t len, bool recompute,
                                             RowAcc<VEC, K>& acc, float (&cacc)[K]) {
  using R = RowAcc<VEC, K>;
  const int d = a.L.d_out, H = a.L.heads, dh = d / H;
  const int lane = lane_id();
  if (!recompute && a.g.in_deg_prev[v] > 0 && a.g.in_deg[v] > 0) {
    float sv[K][VEC];
    R::load_rw(a.st.S + srow(a, v) * d, d, sv);
    acc.add(sv);
#pragma unroll
    for (int k = 0; k < K; ++k)
      if (R::has(k, d)) cacc[k] += a.st.ctx[srow(a, v) * H + chunk_head<VEC>(k, dh)];
  }
  int32_t indeg = recompute ? len : a.g.in_deg[v];
  if (indeg == 0) {
    acc.zero();
#pragma unroll
    for (int k = 0; k < K; ++k) cacc[k] = 0.f;
  }
  acc.store(a.st.S + srow(a, v) * d, d);
#pragma unroll
  for (int k = 0; k < K; ++k) {  // ctx per head: written by the lane holding the head's first chunk
    int c = lane + 32 * k;
    if (c * VEC < d && (c * VEC) % dh == 0)
      for (int hh = 0; hh < (VEC > dh ? VEC / dh : 1); ++hh) a.st.ctx[srow(a, v) * H + (c * VEC) / dh + hh] = cacc[k];
  }
  float* hrow = a.st.H_out + ::rtec::hrow(a, v) * d;
  if (!FULL && a.st.log_out) {
    float old[K][VEC];
    R::load_rw(hrow, d, old);
    R o;
    o.zero();
    o.add(old);
    o.store(a.st.log_out + i * d, d);
  }
  R o;
  bool finite = true;
#pragma unroll
  for (int k = 0; k < K; ++k)
#pragma unroll
    for (int jj = 0; jj < VEC; ++jj) {
      const float x = indeg > 0 ? acc.v[k][jj] / cacc[k] : 0.f;
      finite = finite && (isfinite(x) || !R::has(k, d));  // chunks beyond d hold 0 / 0
      o.v[k][jj] = elu1(x);
    }
  o.store(hrow, d);
  // an attention weight or sum that overflowed fp32 (exp of a logit above ~88.7; the f64
  // reference's math.exp overflows above ~709.8) or a non-finite aggregate: NumericError
  // at the destination (linalg.py:55-60 exp overflow, :22-29 non-finite result)
  if (__any_sync(0xffffffffu, !finite) && lane_id() == 0) report_error(a.err, RTEC_NUMERIC_ERROR, v);
}

// Occupancy / rows in flight: template OCC (CTAs / SM) and UNR (edges gathered per warp
// step); with one row pair in flight 6 CTAs / SM won (c3-gat p50 3 CTAs 16.4 ms, 4 CTAs
// 14.7, 5 CTAs 14.55, 6 CTAs 14.1), two pairs at 4 CTAs win over that (launch_gat_passes)
template <int VEC, int K, bool FULL, int UNR = 1, int OCC = 6>
__global__ void __launch_bounds__(kLBlk, OCC) k_gat_light(LayerArgs a, AggRows rows) {
  RTEC_PDL_ENTRY();
  using R = RowAcc<VEC, K>;
  if (!FULL && err_set(a.err)) return;
  const int64_t nr = rows.count();
  const bool scan = FULL || *a.f.n_src > 0;
  int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < nr; i += nw) {
    int32_t v = rows.at(i);
    int32_t len = a.g.in.len[v];
    if (scan && len > kChunk) continue;  // heavy pass
    const bool recompute = FULL || (a.prev_bm_dst && bm_test(a.prev_bm_dst, v));
    int64_t p = 0, q = 0;
    if (!FULL) {
      int2 rg = reinterpret_cast<const int2*>(a.b.irange)[v];
      if (rg.x >= 0) {
        p = rg.x;
        q = rg.x + rg.y;
      }
    }
    GatEdgeState es;
    gat_state<VEC, K>(a, v, es);
    R acc;
    acc.zero();
    float cacc[K];
#pragma unroll
    for (int k = 0; k < K; ++k) cacc[k] = 0.f;
    if (scan) gat_edges<VEC, K, UNR>(a, es, a.g.in.beg[v], 0, len, p, q, recompute, acc, cacc);
    if (!recompute) gat_struct<VEC, K>(a, es, p, q, acc, cacc);
    gat_finalize<VEC, K, FULL>(a, i, v, len, recompute, acc, cacc);
  }
}

template <int VEC, int K, bool FULL, int UNR = 1, int OCC = 6>
__global__ void __launch_bounds__(kLBlk, OCC) k_gat_heavy(LayerArgs a, AggRows rows, HeavyPlan hp) {
  RTEC_PDL_ENTRY();
  using R = RowAcc<VEC, K>;
  if (!FULL && err_set(a.err)) return;
  const int64_t nh = *hp.n_heavy;
  if (nh == 0) return;
  const int64_t T = hp.hoff[nh];
  const int d = a.L.d_out, H = a.L.heads, dh = d / H;
  const int pw = (d + H + 3) & ~3;  // partial row: d floats + H attention sums, 16-byte aligned
  int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t tt = warp; tt < T; tt += nw) {
    const int64_t t = hp.order ? static_cast<int64_t>(hp.order[tt]) : tt;
    int32_t j = hp.cmap[t];
    int64_t c0 = hp.hoff[j];
    int32_t nch = static_cast<int32_t>(hp.hoff[j + 1] - c0);
    int32_t c = static_cast<int32_t>(t - c0);
    int64_t i = hp.heavy[j];
    int32_t v = rows.at(i);
    int32_t len = a.g.in.len[v];
    const bool recompute = FULL || (a.prev_bm_dst && bm_test(a.prev_bm_dst, v));
    int64_t p = 0, q = 0;
    if (!FULL) {
      int2 rg = reinterpret_cast<const int2*>(a.b.irange)[v];
      if (rg.x >= 0) {
        p = rg.x;
        q = rg.x + rg.y;
      }
    }
    GatEdgeState es;
    gat_state<VEC, K>(a, v, es);
    R acc;
    acc.zero();
    float cacc[K];
#pragma unroll
    for (int k = 0; k < K; ++k) cacc[k] = 0.f;
    int32_t e0 = c * kChunk, e1 = min(len, e0 + kChunk);
    gat_edges<VEC, K, UNR>(a, es, a.g.in.beg[v], e0, e1, p, q, recompute, acc, cacc);
    if (!recompute && c == 0) gat_struct<VEC, K>(a, es, p, q, acc, cacc);
    float* part = hp.part + t * pw;
    acc.store(part, d);
#pragma unroll
    for (int k = 0; k < K; ++k) {
      int cc = lane_id() + 32 * k;
      if (cc * VEC < d && (cc * VEC) % dh == 0)
        for (int hh = 0; hh < (VEC > dh ? VEC / dh : 1); ++hh) part[d + (cc * VEC) / dh + hh] = cacc[k];
    }
    __threadfence();
    __syncwarp();  // every lane's partial is fenced before the arrival is published
    int old = 0;
    if (lane_id() == 0) old = atomicAdd(hp.arrive + j, 1);
    old = __shfl_sync(0xffffffffu, old, 0);
    if (old != nch - 1) continue;
    __threadfence();
    acc.zero();
#pragma unroll
    for (int k = 0; k < K; ++k) cacc[k] = 0.f;
    sum_partials<VEC, K>(hp.part + c0 * pw, pw, d, nch, acc);  // chunk order: deterministic sum
#pragma unroll 4
    for (int32_t cc = 0; cc < nch; ++cc) {
      const float* src = hp.part + (c0 + cc) * pw + d;
#pragma unroll
      for (int k = 0; k < K; ++k)
        if (R::has(k, d)) cacc[k] += __ldcg(src + chunk_head<VEC>(k, dh));
    }
    gat_finalize<VEC, K, FULL>(a, i, v, len, recompute, acc, cacc);
  }
}

// Gathers of the VEC = 4 passes: two edges' (Z, Z_log) row pairs in flight per warp at
// 4 CTAs / SM (64 registers) -- measured c3-gat GAT stage 6.2 -> 5.5 ms against one pair at
// 6 CTAs / SM; three or four pairs at 2-3 CTAs / SM and two pairs at 5-6 (spills) lose
// (profiles/r02v_gat_unroll_ab.md).  RTEC_GAT_UNR=1: one pair at 6 CTAs / SM (A/B).
static bool gat_unr1() {
  static int u = -1;
  if (u < 0) {
    const char* e = getenv("RTEC_GAT_UNR");
    u = e ? (atoi(e) == 1) : 0;
  }
  return u != 0;
}

template <int VEC, int K, bool FULL>
static int launch_gat_passes(const LayerArgs& a, AggRows rows, const HeavyPlan& hp, int grid, cudaStream_t s,
                             cudaStream_t hs) {
  if (gat_unr1()) {
    launch(k_gat_heavy<VEC, K, FULL, 1, 6>, grid, kLBlk, 0, hs, a, rows, hp);
    launch(k_gat_light<VEC, K, FULL, 1, 6>, grid, kLBlk, 0, s, a, rows);
  } else {
    launch(k_gat_heavy<VEC, K, FULL, 2, 4>, grid, kLBlk, 0, hs, a, rows, hp);
    launch(k_gat_light<VEC, K, FULL, 2, 4>, grid, kLBlk, 0, s, a, rows);
  }
  return RTEC_OK;
}

template <bool FULL>
static int launch_gat(LayerArgs& a, AggRows rows, int64_t max_rows, int64_t max_edges, Ws& w, cudaStream_t s) {
  const int d = a.L.d_out;
  if (a.L.heads > kHMax) {
    set_error("GAT supports up to %d heads (got %d)", kHMax, a.L.heads);
    return RTEC_SHAPE_ERROR;
  }
  a.d_agg = d;
  HeavyPlan hp{};
  RTEC_TRY(plan_heavy<FULL>(a, rows, max_rows, max_edges, (d + a.L.heads + 3) & ~3, w, s, hp));
  const int grid = kSMs * 8;
  const int dh = d / a.L.heads;
  bool ok;
  RTEC_PROF(FULL ? "k_gat_full" : "k_gat_layer", s);
  if (d % 4 == 0 && dh % 4 == 0) {
    // hub chunks on the side stream, as in launch_aggregation: the two passes write
    // disjoint destinations and fill each other's tails (not while profiling)
    cudaStream_t hs = g_prof_on ? s : side_stream();
    if (hs != s) {
      RTEC_CUDA(cudaEventRecord(side_fork(), s));
      RTEC_CUDA(cudaStreamWaitEvent(hs, side_fork(), 0));
    }
    int grc = RTEC_OK;
    ok = RTEC_ROW_DISPATCH(d, (grc = launch_gat_passes<VEC, K, FULL>(a, rows, hp, grid, s, hs)));
    if (grc != RTEC_OK) return grc;
    if (hs != s) {
      RTEC_CUDA(cudaEventRecord(side_join(), hs));
      RTEC_CUDA(cudaStreamWaitEvent(s, side_join(), 0));
    }
  } else {
    int kk = (d + 31) / 32;
    ok = true;
    if (kk <= 1) {
      launch(k_gat_light<1, 1, FULL>, grid, kLBlk, 0, s, a, rows);
      launch(k_gat_heavy<1, 1, FULL>, grid, kLBlk, 0, s, a, rows, hp);
    } else if (kk <= 4) {
      launch(k_gat_light<1, 4, FULL>, grid, kLBlk, 0, s, a, rows);
      launch(k_gat_heavy<1, 4, FULL>, grid, kLBlk, 0, s, a, rows, hp);
    } else if (kk <= 8) {
      launch(k_gat_light<1, 8, FULL>, grid, kLBlk, 0, s, a, rows);
      launch(k_gat_heavy<1, 8, FULL>, grid, kLBlk, 0, s, a, rows, hp);
    } else {
      ok = false;
    }
  }
  if (!ok) {
    set_error("row width %d unsupported", d);
    return RTEC_SHAPE_ERROR;
  }
  RTEC_LAUNCH_CHECK("k_gat");
  return RTEC_OK;
}

// el / er for projected rows: el = a[:dh]·z_h, er = a[dh:]·z_h per head
__global__ void k_gat_logits(const float* __restrict__ Z, const int32_t* rows, const int64_t* n_rows, int64_t n_all,
                             int d, int H, const float* __restrict__ att, float* el, float* er, float* er_log,
                             const uint64_t* err) {
  RTEC_PDL_ENTRY();
  if (err && err_set(err)) return;
  int dh = d / H;
  int64_t nr = rows ? *n_rows : n_all;
  int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  int lane = lane_id();
  for (int64_t i = warp; i < nr; i += nw) {
    int32_t v = rows ? rows[i] : static_cast<int32_t>(i);
    for (int h = 0; h < H; ++h) {
      float sl = 0.f, sr = 0.f;
      for (int j = lane; j < dh; j += 32) {
        float z = Z[static_cast<int64_t>(v) * d + h * dh + j];
        sl = fmaf(att[h * 2 * dh + j], z, sl);
        sr = fmaf(att[h * 2 * dh + dh + j], z, sr);
      }
      sl = warp_sum(sl);
      sr = warp_sum(sr);
      if (lane == 0) {
        if (er_log) er_log[i * H + h] = er[static_cast<int64_t>(v) * H + h];
        el[static_cast<int64_t>(v) * H + h] = sl;
        er[static_cast<int64_t>(v) * H + h] = sr;
      }
    }
  }
}

// ------------------------------------------------------------------ update GEMM (K12), SIMT fp32
// Y[i] = act(X[i] · W^T); X rows optionally gathered, Y rows optionally
// scattered with DeltaLog capture of the overwritten rows.
struct GemmArgs {
  const float* X; int64_t ldx; const int32_t* x_rows;
  const float* W; int d_in; int d_out;
  const int64_t* n_rows; int64_t max_rows;
  int act;
  float* Y; int64_t ldy; const int32_t* y_rows;
  float* log;
  const uint64_t* err;  // skip when the batch failed validation / reservation
  int ydiv;             // > 1: Y row of y_rows[i] is y_rows[i] / ydiv (sharded final layer)
  const float* bias;    // Y = scale * act(X W^T + bias) (PinSAGE payload, models.py:159)
  float scale;
  int has_scale;
  uint64_t* nerr;       // non-finite output -> NumericError at the row's vertex (linalg.py:22-29)
};

constexpr int kGM = 64, kGN = 64, kGK = 16;

__global__ void __launch_bounds__(256) k_gemm_simt(GemmArgs g) {
  RTEC_PDL_ENTRY();
  __shared__ float As[kGK][kGM + 4];
  __shared__ float Bs[kGK][kGN + 4];
  if (g.err && err_set(g.err)) return;
  const int64_t nr = g.n_rows ? *g.n_rows : g.max_rows;
  const int64_t row0 = static_cast<int64_t>(blockIdx.x) * kGM;
  if (row0 >= nr) return;
  const int col0 = blockIdx.y * kGN;
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < g.d_in; k0 += kGK) {
    // load A tile: 64 rows x 16 k -> 1024 values, 4 per thread
    for (int e = threadIdx.x; e < kGM * kGK; e += 256) {
      int r = e / kGK, kk = e % kGK;
      int64_t gr = row0 + r;
      float val = 0.f;
      if (gr < nr && k0 + kk < g.d_in) {
        int64_t src = g.x_rows ? g.x_rows[gr] : gr;
        val = g.X[src * g.ldx + k0 + kk];
      }
      As[kk][r] = val;
    }
    for (int e = threadIdx.x; e < kGN * kGK; e += 256) {
      int c = e / kGK, kk = e % kGK;
      float val = 0.f;
      if (col0 + c < g.d_out && k0 + kk < g.d_in) val = g.W[static_cast<int64_t>(col0 + c) * g.d_in + k0 + kk];
      Bs[kk][c] = val;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < kGK; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) a[r] = As[kk][ty * 4 + r];
#pragma unroll
      for (int c = 0; c < 4; ++c) b[c] = Bs[kk][tx * 4 + c];
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[r][c] = fmaf(a[r], b[c], acc[r][c]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    int64_t gr = row0 + ty * 4 + r;
    if (gr >= nr) continue;
    int64_t dst = (g.y_rows ? g.y_rows[gr] : gr) / (g.ydiv > 1 ? g.ydiv : 1);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      int col = col0 + tx * 4 + c;
      if (col >= g.d_out) continue;
      float y = acc[r][c];
      if (g.bias) y += g.bias[col];
      if (g.nerr && !isfinite(y)) report_error(g.nerr, RTEC_NUMERIC_ERROR, g.y_rows ? g.y_rows[gr] : gr);
      if (g.act == 1) y = fmaxf(y, 0.f);
      if (g.has_scale) y *= g.scale;
      float* yp = g.Y + dst * g.ldy + col;
      if (g.log) g.log[gr * g.d_out + col] = *yp;
      *yp = y;
    }
  }
}



int gemm_launch(const GemmArgs& g, cudaStream_t s) {
  if (g.max_rows <= 0) return RTEC_OK;
  dim3 grid(static_cast<unsigned>((g.max_rows + kGM - 1) / kGM), static_cast<unsigned>((g.d_out + kGN - 1) / kGN));
  RTEC_PROF("k_gemm_update", s);
  launch(k_gemm_simt, grid, 256, 0, s, g);
  RTEC_LAUNCH_CHECK("k_gemm_simt");
  return RTEC_OK;
}

// ------------------------------------------------------------------ MoNet payload (models.py:211-213)
// P[v] = exp(0.5 (h_v - mu)^T Wq (h_v - mu)); Wq symmetrised on the host so the
// lane-strided reads of row k are coalesced.  One warp per row, d <= 256.
constexpr int kQuadM = 8;
__global__ void __launch_bounds__(256) k_quadform(const float* __restrict__ H, const int32_t* rows,
                                                  const int64_t* n_rows, int64_t n_all, int d,
                                                  const float* __restrict__ Wq, const float* __restrict__ mu,
                                                  float* P, float* P_log, const uint64_t* err) {
  RTEC_PDL_ENTRY();
  if (err && err_set(err)) return;
  const int64_t nr = rows ? *n_rows : n_all;
  int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int lane = lane_id();
  for (int64_t i = warp; i < nr; i += nw) {
    const int32_t v = rows ? rows[i] : static_cast<int32_t>(i);
    float df[kQuadM], t[kQuadM];
#pragma unroll
    for (int m = 0; m < kQuadM; ++m) {
      const int k = lane + 32 * m;
      df[m] = k < d ? H[static_cast<int64_t>(v) * d + k] - mu[k] : 0.f;
      t[m] = 0.f;
    }
#pragma unroll
    for (int m = 0; m < kQuadM; ++m) {
      if (32 * m >= d) break;
      for (int kk = 0; kk < 32 && 32 * m + kk < d; ++kk) {
        const float dk = __shfl_sync(0xffffffffu, df[m], kk);
        const float* wr = Wq + static_cast<int64_t>(32 * m + kk) * d;
#pragma unroll
        for (int mm = 0; mm < kQuadM; ++mm) {
          const int j = lane + 32 * mm;
          if (j < d) t[mm] = fmaf(__ldg(wr + j), dk, t[mm]);
        }
      }
    }
    float q = 0.f;
#pragma unroll
    for (int m = 0; m < kQuadM; ++m) q = fmaf(df[m], t[m], q);
    q = warp_sum(q);
    if (lane == 0) {
      if (P_log) P_log[i] = P[v];
      P[v] = expf(0.5f * q);
    }
  }
}

// ------------------------------------------------------------------ query (K18)
__global__ void k_query(const float* __restrict__ H, int64_t d, const int32_t* __restrict__ ids, int64_t k, int32_t n,
                        float* out, uint64_t* err) {
  RTEC_PDL_ENTRY();
  int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < k; i += nw) {
    int32_t v = ids[i];
    if (v < 0 || v >= n) {
      if (lane_id() == 0) report_error(err, RTEC_INVALID_VERTEX, i);
      continue;
    }
    for (int64_t j = lane_id(); j < d; j += 32) out[i * d + j] = H[static_cast<int64_t>(v) * d + j];
  }
}

}  // namespace rtec

using namespace rtec;

// update (and GIN's chained MLP) on rows of gemm_in: tcgen05 3xTF32 when the
// layer carries prepared weights, SIMT fp32 otherwise
static int run_update(const rtec_graph_t* g, const rtec_layer_t* L, rtec_state_t* st, const int64_t* n_rows,
                      int64_t max_rows, const int32_t* y_rows, float* log, const uint64_t* err, cudaStream_t s,
                      uint64_t* nerr);

static int layer_dims_ok(const rtec_layer_t* L) {
  if (L->model < 0 || L->model > RTEC_MODEL_AGNN) {
    set_error("unsupported model id %d", L->model);
    return RTEC_UNSUPPORTED_MODEL;
  }
  if (L->d_in <= 0 || L->d_out <= 0 || L->heads <= 0 || (L->d_out % L->heads) != 0) {
    set_error("bad layer dims d_in=%d d_out=%d heads=%d", L->d_in, L->d_out, L->heads);
    return RTEC_SHAPE_ERROR;
  }
  return RTEC_OK;
}

// err: skip when set (the batch failed); nerr: where non-finite outputs are reported
static int run_update(const rtec_graph_t* g, const rtec_layer_t* L, rtec_state_t* st, const int64_t* n_rows,
                      int64_t max_rows, const int32_t* y_rows, float* log, const uint64_t* err, cudaStream_t s,
                      uint64_t* nerr) {
  const int ydiv = (st->out_local && st->row_div > 1) ? st->row_div : 1;
  auto fuse = [&](TcArgs& t) {  // the next layer's source deltas from this update's epilogue
    if (!st->delta_next || !y_rows || (L->d_out & 3)) return;
    t.delta_next = st->delta_next;
    t.deg_new = g->out_deg;
    t.deg_old = g->out_deg_prev;
    t.coeff_gcn = L->model == RTEC_MODEL_GCN;
    t.deg_off = L->degree_offset;
    t.log = nullptr;
  };
  const int dk = upd_k(*L);
  const int act = L->model == RTEC_MODEL_COMMNET ? 0 : 1;  // CommNet: W h_v + W2 a_v (models.py:247)
  if (L->Wt_hi) {
    const int nkb = tc_nkb_of(dk);
    if (is_gin(L->model)) {  // W2 relu(W (h + a)) (models.py:187-189), hidden kept in tile layout
      const int nkb2 = tc_nkb_of(L->d_out);
      TcArgs t1{st->gemm_in, L->Wt_hi, L->Wt_lo, nkb, tc_npad_of(L->d_out), L->d_out, n_rows, max_rows, 1,
                nullptr, 0, nullptr, nullptr, st->gemm_mid, nkb2, err};
      t1.nerr = nerr;
      RTEC_TRY(gemm_tc_launch(t1, s));
      TcArgs t2{st->gemm_mid, L->W2t_hi, L->W2t_lo, nkb2, tc_npad_of(L->d_out), L->d_out, n_rows, max_rows, 0,
                st->H_out, L->d_out, y_rows, log, nullptr, 0, err};
      t2.ydiv = ydiv;
      t2.nerr = nerr;
      fuse(t2);
      return gemm_tc_launch(t2, s);
    }
    TcArgs t{st->gemm_in, L->Wt_hi, L->Wt_lo, nkb, tc_npad_of(L->d_out), L->d_out, n_rows, max_rows, act,
             st->H_out, L->d_out, y_rows, log, nullptr, 0, err};
    t.ydiv = ydiv;
    t.nerr = nerr;
    fuse(t);
    return gemm_tc_launch(t, s);
  }
  if (is_gin(L->model)) {
    GemmArgs g1{st->gemm_in, L->d_in, nullptr, L->W, L->d_in, L->d_out, n_rows, max_rows, 1,
                st->gemm_mid, L->d_out, nullptr, nullptr, err};
    g1.nerr = nerr;
    RTEC_TRY(gemm_launch(g1, s));
    GemmArgs g2{st->gemm_mid, L->d_out, nullptr, L->W2, L->d_out, L->d_out, n_rows, max_rows, 0,
                st->H_out, L->d_out, y_rows, log, err, ydiv};
    g2.nerr = nerr;
    return gemm_launch(g2, s);
  }
  GemmArgs g1{st->gemm_in, dk, nullptr, L->W, dk, L->d_out, n_rows, max_rows, act,
              st->H_out, L->d_out, y_rows, log, err, ydiv};
  g1.nerr = nerr;
  return gemm_launch(g1, s);
}

// LayerArgs common to the incremental and full layer passes
static void layer_args_init(LayerArgs& a, const rtec_layer_t* L, const rtec_state_t* st) {
  a.self_in = st->H_in;
  a.gk = upd_k(*L);
  a.gcol = self_concat(L->model) ? L->d_in : 0;
  a.d_agg = L->model == RTEC_MODEL_MONET ? 1 : L->d_in;
  if (payload_model(L->model)) {  // messages are the projected payload rows (and their log)
    a.st.H_in = st->Z;
    a.st.log_in = st->Z_log;
  }
  a.tc_nkb = L->Wt_hi ? tc_nkb_of(a.gk) : 0;
}

extern "C" {

int rtec_update_gemm(const float* X, int64_t ldx, const float* W, int32_t d_in, int32_t d_out, const int64_t* n_rows,
                     int64_t max_rows, int32_t act, float* Y, int64_t ldy, const int32_t* scatter_rows,
                     float* scatter_dst, float* log_dst, rtec_stream_t stream) {
  GemmArgs g{X, ldx, nullptr, W, d_in, d_out, n_rows, max_rows, act,
             scatter_rows ? scatter_dst : Y, ldy, scatter_rows, log_dst, nullptr};
  return gemm_launch(g, reinterpret_cast<cudaStream_t>(stream));
}

int rtec_layer_incremental(const rtec_graph_t* g, const rtec_batch_t* b, const rtec_layer_t* L, rtec_state_t* st,
                           const rtec_frontier_t* prev, const rtec_frontier_t* f, uint64_t* err, void* ws,
                           size_t ws_bytes, rtec_stream_t stream) {
  RTEC_TRY(layer_dims_ok(L));
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  int64_t n = g->n;
  Ws w(ws, ws_bytes);
  LayerArgs a{};
  a.g = *g;
  a.b = *b;
  a.L = *L;
  a.st = *st;
  a.f = *f;
  // V_chg(l-1) and its DeltaLog rows: all ranks' changed vertices when sharded
  a.prev_bm_dst = prev ? (prev->bm_chg ? prev->bm_chg : prev->bm_dst) : nullptr;
  a.prev_slot = prev ? (prev->chg_slot ? prev->chg_slot : prev->dst_slot) : nullptr;
  a.err = err;
  const int grid = kSMs * 8;
  if (L->model == RTEC_MODEL_GAT)
    return launch_gat<false>(a, AggRows{f->dst_list, f->n_dst, n}, n, g->in.slots, w, s);
  layer_args_init(a, L, st);
  if (L->model == RTEC_MODEL_GIN_MAX) {
    RTEC_TRY(launch_max<false>(a, AggRows{f->dst_list, f->n_dst, n}, n, g->in.slots, w, s));
    return run_update(g, L, st, f->n_dst, n, f->dst_list, st->log_out, err, s, err);
  }
  if (edge_model(L->model)) {
    RTEC_TRY(launch_dd<false>(a, AggRows{f->dst_list, f->n_dst, n}, n, g->in.slots, w, s));
    return run_update(g, L, st, f->n_dst, n, f->dst_list, st->log_out, err, s, err);
  }
  float* delta = st->delta ? st->delta : w.alloc<float>(n * static_cast<int64_t>(a.d_agg));
  RTEC_WS_CHECK(w);
  a.delta = delta;
  bool ok;
  {
    RTEC_PROF("k_src_delta", s);
    ok = RTEC_ROW_DISPATCH(a.d_agg, (launch(k_src_delta<VEC, K>, grid, kLBlk, 0, s, a, delta)));
  }
  if (!ok) {
    set_error("row width %d unsupported", a.d_agg);
    return RTEC_SHAPE_ERROR;
  }
  {
    RTEC_PROF("aggregation", s);  // the whole stage (plan + light / heavy, or compaction + slice passes)
    RTEC_TRY(launch_aggregation<false>(a, AggRows{f->dst_list, f->n_dst, n}, n, g->in.slots, w, s));
  }
  // update on V_dst(l) rows with DeltaLog capture (operators.py:180)
  return run_update(g, L, st, f->n_dst, n, f->dst_list, st->log_out, err, s, err);
}


int rtec_layer_full(const rtec_graph_t* g, const rtec_layer_t* L, rtec_state_t* st, const int32_t* rows,
                    const int64_t* n_rows, int64_t max_rows, uint64_t* err, void* ws, size_t ws_bytes,
                    rtec_stream_t stream) {
  RTEC_TRY(layer_dims_ok(L));
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  int64_t n = g->n;
  LayerArgs a{};
  a.g = *g;
  a.L = *L;
  a.st = *st;
  a.err = err;
  if (L->model == RTEC_MODEL_GAT) {
    Ws w(ws, ws_bytes);
    if (rows)  // listed rows (UER): the caller keeps Z / el / er current for the changed sources
      return launch_gat<true>(a, AggRows{rows, n_rows, n}, max_rows, g->in.slots, w, s);
    // Z = W H (all rows; tcgen05 when the layer carries operand images), logits, then the
    // full softmax aggregation
    RTEC_TRY(rtec_gat_project(L, st->H_in, nullptr, nullptr, n, st->Z, st->el, st->er, nullptr, nullptr, err,
                              st->gemm_in, stream));
    return launch_gat<true>(a, AggRows{nullptr, nullptr, n}, n, g->in.slots, w, s);
  }
  if (!rows) RTEC_TRY(rtec_project(L, st->H_in, nullptr, nullptr, n, st->Z, nullptr, nullptr, stream));
  layer_args_init(a, L, st);
  int64_t mr = rows ? max_rows : n;
  if (L->model == RTEC_MODEL_GIN_MAX) {
    Ws w(ws, ws_bytes);
    RTEC_TRY(launch_max<true>(a, AggRows{rows, rows ? n_rows : nullptr, n}, mr, g->in.slots, w, s));
    return run_update(g, L, st, rows ? n_rows : nullptr, mr, rows, nullptr, nullptr, s, err);
  }
  {
    Ws w(ws, ws_bytes);
    if (edge_model(L->model))
      RTEC_TRY(launch_dd<true>(a, AggRows{rows, rows ? n_rows : nullptr, n}, mr, g->in.slots, w, s));
    else
      RTEC_TRY(launch_aggregation<true>(a, AggRows{rows, rows ? n_rows : nullptr, n}, mr, g->in.slots, w, s));
  }
  return run_update(g, L, st, rows ? n_rows : nullptr, mr, rows, nullptr, nullptr, s, err);
}

int rtec_gat_project(const rtec_layer_t* L, const float* H, const int32_t* rows, const int64_t* n_rows,
                     int64_t n_or_max_rows, float* Z, float* el, float* er, float* Z_log, float* er_log,
                     const uint64_t* err, float* a_img, rtec_stream_t stream) {
  RTEC_TRY(layer_dims_ok(L));
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int64_t* nr = rows ? n_rows : nullptr;
  uint64_t* nerr = const_cast<uint64_t*>(err);
  if (L->Wt_hi && a_img) {
    // K13 on tcgen05: the rows are gathered into the SW128 A image, then the 3xTF32
    // GEMM scatters Z[rows] (old rows into Z_log) -- f_nn = W h_u (models.py:279)
    const int nkb = tc_nkb_of(L->d_in);
    const uint64_t* skip = rows ? err : nullptr;  // a failed batch skips; bootstrap always runs
    RTEC_TRY(gemm_tc_pack_rows(H, L->d_in, L->d_in, rows, nr, n_or_max_rows, a_img, nkb, skip, s));
    TcArgs t{a_img, L->Wt_hi, L->Wt_lo, nkb, tc_npad_of(L->d_out), L->d_out, nr, n_or_max_rows, 0,
             Z, L->d_out, rows, Z_log, nullptr, 0, skip};
    t.nerr = nerr;
    RTEC_TRY(gemm_tc_launch(t, s));
  } else {
    GemmArgs gz{H, L->d_in, rows, L->W, L->d_in, L->d_out, nr, n_or_max_rows, 0,
                Z, L->d_out, rows, Z_log, rows ? err : nullptr};
    gz.nerr = nerr;
    RTEC_TRY(gemm_launch(gz, s));
  }
  RTEC_PROF("k_gat_logits", s);
  launch(k_gat_logits, kSMs * 8, kLBlk, 0, s, Z, rows, n_rows, n_or_max_rows, L->d_out, L->heads, L->att, el, er, er_log,
                                          rows ? err : nullptr);
  RTEC_LAUNCH_CHECK("k_gat_logits");
  return RTEC_OK;
}

int rtec_project(const rtec_layer_t* L, const float* H, const int32_t* rows, const int64_t* n_rows,
                 int64_t n_or_max_rows, float* P, float* P_log, const uint64_t* err, rtec_stream_t stream) {
  RTEC_TRY(layer_dims_ok(L));
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (n_or_max_rows <= 0) return RTEC_OK;
  const int d = L->d_in;
  const int64_t* nr = rows ? n_rows : nullptr;
  switch (L->model) {
    case RTEC_MODEL_PINSAGE: {  // alpha relu(Q h + q)
      GemmArgs g{H, d, rows, L->Wp, d, d, nr, n_or_max_rows, 1, P, d, rows, P_log, err};
      g.bias = L->bp;
      g.scale = L->scalar;
      g.has_scale = 1;
      return gemm_launch(g, s);
    }
    case RTEC_MODEL_GGCN: {  // [Wg_src h ; Wg_dst h]
      GemmArgs g{H, d, rows, L->Wp, d, 2 * d, nr, n_or_max_rows, 0, P, 2 * d, rows, P_log, err};
      return gemm_launch(g, s);
    }
    case RTEC_MODEL_MONET: {
      if (d > 32 * kQuadM) {
        set_error("MoNet input width %d > %d", d, 32 * kQuadM);
        return RTEC_SHAPE_ERROR;
      }
      RTEC_PROF("k_quadform", s);
      launch(k_quadform, kSMs * 8, 256, 0, s, H, rows, nr, n_or_max_rows, d, L->Wp, L->bp, P, P_log, err);
      RTEC_LAUNCH_CHECK("k_quadform");
      return RTEC_OK;
    }
    default:
      return RTEC_OK;
  }
}

int rtec_query(const float* H, int64_t d, const int32_t* ids, int64_t k, float* out, int32_t n, uint64_t* err,
               rtec_stream_t stream) {
  if (k <= 0) return RTEC_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  launch(k_query, grid_for(k * 32, 256), 256, 0, s, H, d, ids, k, n, out, err);
  RTEC_LAUNCH_CHECK("k_query");
  return RTEC_OK;
}

}  // extern "C"
