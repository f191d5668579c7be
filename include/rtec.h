/*
 * rtec.h -- C ABI of librtec.so, the B200 (sm_100a) incremental RTEC engine.
 *
 * The reference (`streamgnn`, pure Python) exposes no FFI; this header is the
 * drop-in boundary for its hot path.  Each entry point names
 * the reference interface it replaces (file:line, relative to
 * /root/reference/pkg/src/streamgnn/).
 *
 * Conventions
 *  - All array pointers are DEVICE pointers unless the name ends in `_host`.
 *  - Every call is asynchronous on the given stream, returns an rtec_status
 *    for argument errors detected on the host, and reports data-dependent
 *    errors (InvalidVertex, ConfigError, ...) through a device status word
 *    (`err`: uint64 packed as position << 32 | code, all-ones = ok; the
 *    smallest position wins) that the caller reads after the batch.
 *  - The library allocates nothing persistent.  Persistent state lives in
 *    caller-owned device buffers described by the POD structs below; scratch
 *    space comes from the caller's workspace (`ws`, `ws_bytes`), sized with
 *    rtec_workspace_bytes().
 *  - Vertex ids are int32 (n < 2^31), edge slots int64.
 *  - One host thread / stream per graph; not re-entrant per graph
 *    (pma.py:22).
 */
#ifndef RTEC_H_
#define RTEC_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* rtec_stream_t; /* == cudaStream_t */

/* status codes: 1:1 with errors.py:6-35 exception classes */
enum {
  RTEC_OK = 0,
  RTEC_INVALID_VERTEX = 1,   /* errors.InvalidVertex   */
  RTEC_CONFIG_ERROR = 2,     /* errors.ConfigError     */
  RTEC_SHAPE_ERROR = 3,      /* errors.ShapeError      */
  RTEC_NUMERIC_ERROR = 4,    /* errors.NumericError    */
  RTEC_SINGULAR_CONTEXT = 5, /* errors.SingularContext */
  RTEC_STALE_STATE = 6,      /* errors.StaleState      */
  RTEC_UNSUPPORTED_MODEL = 7,/* errors.UnsupportedModel*/
  RTEC_CUDA_ERROR = 100
};

/* update ops (graph.py:28-30) */
enum { RTEC_OP_INSERT = 0, RTEC_OP_DELETE = 1 };

/* models (models.py:42-52); the hot-path four, plus GIN with an elementwise
 * max aggregator (configs[3]; no reference counterpart -- retract-and-recompute
 * per destination) */
enum { RTEC_MODEL_GCN = 0, RTEC_MODEL_SAGE = 1, RTEC_MODEL_GIN = 2, RTEC_MODEL_GAT = 3, RTEC_MODEL_GIN_MAX = 4,
       /* the rest of Table II (models.py:144-348):
        *   PINSAGE  payload alpha relu(Q h_u + q), mean, update relu(W [h_v ; a_v])
        *   MONET    scalar payload exp(0.5 (h_u-mu)^T Wq (h_u-mu)), sum, update relu(W a)
        *   COMMNET  sum of h_u, update W h_v + W2 a_v
        *   GGCN     dest-dependent sigmoid(Wg_src h_u + Wg_dst h_v) * h_u, sum, relu(W a)
        *   AGNN     dest-dependent beta cos(h_u, h_v) h_u, sum, relu(W a) */
       RTEC_MODEL_PINSAGE = 5, RTEC_MODEL_MONET = 6, RTEC_MODEL_COMMNET = 7, RTEC_MODEL_GGCN = 8,
       RTEC_MODEL_AGNN = 9 };

/* One direction of the adjacency: gapped per-vertex runs.  Run of v is
 * nbr[beg[v] .. beg[v]+len[v]) ascending, with cap[v] >= len[v] slots reserved.
 * Runs that outgrow their capacity are relocated to the arena tail (*top).
 * Replaces one PackedMemoryArray (pma.py:37-326) of composite keys. */
typedef struct {
  int64_t slots;     /* capacity of nbr[] / ts[] */
  int64_t* beg;      /* [n] */
  int32_t* len;      /* [n] */
  int32_t* cap;      /* [n] */
  int32_t* nbr;      /* [slots] */
  int64_t* ts;       /* [slots] timestamps (out direction) or NULL */
  int64_t* top;      /* [1] arena bump pointer */
} rtec_adj_t;

/* DynamicGraph (graph.py:59-235): out + in adjacency, degrees. */
typedef struct {
  int64_t n;
  rtec_adj_t out;    /* src -> dst runs, with ts (graph.py:73-76 `_out`) */
  rtec_adj_t in;     /* dst -> src runs (graph.py `_in`) */
  int32_t* out_deg;  /* [n] current degrees */
  int32_t* in_deg;   /* [n] */
  int32_t* out_deg_prev; /* [n] degrees before the current batch (== current between batches) */
  int32_t* in_deg_prev;  /* [n] */
  int64_t* num_edges;    /* [1] */
  float slack;           /* relocated / rebuilt runs get cap = len + max(min_slack, ceil(len*slack)) */
  int32_t min_slack;
  /* Vertex sharding: this graph is the shard of rank
   * part_rank out of part_count and holds exactly the edges whose dst it owns
   * (owner(v) = v mod part_count).  part_count <= 1: unsharded.  apply
   * validates the whole batch but probes / mutates only owned-dst updates. */
  int32_t part_rank;
  int32_t part_count;
} rtec_graph_t;

/* Internal status: the arena (or the in-place merge scratch) cannot hold this
 * batch; nothing was mutated.  The host compacts / grows and re-applies. */
#define RTEC_ARENA_FULL 8

/* Per-batch derived data (capacity `cap` updates).  Written by
 * rtec_batch_apply, read by the frontier / layer kernels of the same batch. */
typedef struct {
  int64_t cap;
  uint64_t* err;       /* [1] packed (position << 32 | code); ~0 = ok */
  uint8_t* status;     /* [cap] per update in batch order: 1 applied, 0 rejected */
  /* applied updates sorted by (src, dst) -- out-key order */
  int32_t* a_src; int32_t* a_dst; uint8_t* a_op; int64_t* a_ts;
  int64_t* n_applied;  /* [1] */
  /* applied updates sorted by (dst, src) -- in-key order */
  int32_t* i_src; int32_t* i_dst; uint8_t* i_op;
  /* DegreeDelta rows (graph.py:41-48), ascending vertex */
  int32_t* d_vertex; int32_t* d_old_in; int32_t* d_new_in; int32_t* d_old_out; int32_t* d_new_out;
  int64_t* n_delta;    /* [1] */
  /* [2n] per-vertex (first, count) of its entries in the in-key list i_*;
   * (-1, 0) for vertices without applied updates.  Caller initialises it once
   * to (-1, 0); rtec_batch_apply sets it, rtec_batch_commit resets it. */
  int32_t* irange;
  /* Sharded runs: bitmap of vertices whose GLOBAL out-degree changed in this
   * batch (rtec_shard_degrees); the frontier seeds Dg from it instead of the
   * shard-local DegreeDelta.  NULL when unsharded. */
  const uint32_t* dg_bm;
  /* [4] or NULL: run-merge volume of the last apply, in elements -- out-runs: old
   * suffix + update items read, in-place new suffix staged; in-runs: the same two.
   * The bench turns them into the apply chain's algorithmic bytes. */
  int64_t* apply_ctr;
} rtec_batch_t;

/* Per-layer frontier (Alg. 4).  Bitmaps
 * are n bits (uint32 words).  Lists ascending. */
typedef struct {
  uint32_t* bm_src;    /* [words] S(l) = Dg ∪ V_chg(l-1) */
  uint32_t* bm_dst;    /* [words] V_dst(l) */
  int32_t* src_list;  int64_t* n_src;   /* S(l) */
  int32_t* dst_list;  int64_t* n_dst;   /* V_dst(l) */
  int32_t* src_slot;   /* [n] vertex -> index in src_list (valid where bm_src bit set) */
  int32_t* dst_slot;   /* [n] vertex -> index in dst_list (valid where bm_dst bit set) */
  int64_t* counters;   /* [8] |E_curr|, |V_dst|, |S|, |R|, Σ outdeg(new S), Σ indeg(V_dst), Σ indeg(R), reserved */
  /* Sharded runs: V_chg(l) over ALL ranks (union of every shard's V_dst(l),
   * assembled by rtec_shard_unpack_changed) and vertex -> row of the exchanged
   * DeltaLog.  The next layer reads S(l+1) = S(l) ∪ bm_chg and old rows through
   * chg_slot.  NULL: bm_dst / dst_slot (unsharded). */
  uint32_t* bm_chg;
  int32_t* chg_slot;
} rtec_frontier_t;

/* Layer descriptor (operators.py:42-47 LayerWeights + bundle flags).
 * Weights are fp32 copies of make_bundle's f64 weights (models.py:364). */
typedef struct {
  int32_t model;       /* RTEC_MODEL_* */
  int32_t d_in;        /* input width  */
  int32_t d_out;       /* output width */
  int32_t heads;       /* GAT heads (1 for others) */
  float degree_offset; /* GCN: 1 if degree_smoothing else 0 (models.py:89) */
  int32_t pad;
  const float* W;      /* [d_out, d_in] row-major (GAT: heads stacked [heads*dh, d_in]) */
  const float* W2;     /* GIN second matrix [d_out, d_out] (models.py:181) */
  const float* att;    /* GAT attention [heads, 2*dh] (dst half first, models.py:266-271) */
  /* tcgen05 3xTF32 operand images of W / W2 from rtec_gemm_prepare_weights
   * (NULL -> SIMT fp32 update).  With them set, state.gemm_in / gemm_mid hold
   * the SW128 tile image: ceil(rows/128)*128 x ceil(d/32)*32 floats. */
  const float* Wt_hi; const float* Wt_lo;
  const float* W2t_hi; const float* W2t_lo;
  /* per-source projection of the payload / gate models (rtec_project):
   *   PINSAGE Q [d_in, d_in] + bias q;  MONET symmetrised Wq [d_in, d_in] + mean mu;
   *   GGCN [Wg_src ; Wg_dst] [2 d_in, d_in] (no bias).  NULL for the other models. */
  const float* Wp;
  const float* bp;
  float scalar;        /* PINSAGE alpha (models.py:151), AGNN beta (models.py:322) */
  int32_t d_k;         /* update GEMM input width: 2 d_in for PINSAGE / COMMNET ([h_v ; a_v]), 1 for
                          MONET, d_in otherwise (0 = d_in).  W is [d_out, d_k]; COMMNET W = [W | W2]. */
} rtec_layer_t;

/* Per-layer cached state (SPEC.md:355-419 state_cache; stored un-normalised):
 *   S   [n, d_agg]  aggregate before ms_cbn (= ms_cbn_inv(ctx, a))
 *   ctx [n, heads]  GAT attention sums (count contexts are the in-degrees)
 *   H_out [n, d_out] layer output; H_in = previous layer's output (or X)
 *   log_out [n_dst cap, d_out] DeltaLog: pre-batch H_out rows of V_dst(l),
 *            indexed by frontier.dst_slot
 *   GAT caches for the layer: Z [n, d_out] = W h, el/er [n, heads].
 *   PINSAGE / MONET / GGCN: Z = the rtec_project payload rows, Z_log their
 *   pre-batch values for V_chg(l-1) (indexed by the previous dst_slot). */
typedef struct {
  const float* H_in;   float* H_out;
  float* S;            float* ctx;
  float* log_out;      /* DeltaLog rows of this layer's output */
  const float* log_in; /* previous layer's DeltaLog (NULL for layer 0); rows indexed by
                          the previous frontier's dst_slot, membership = its bm_dst */
  float* Z; float* el; float* er;           /* GAT caches (Z: projected payloads of the Table II models) */
  float* Z_log; float* er_log;              /* GAT DeltaLog of Z/er rows of V_chg(l-1) */
  float* gemm_in;      /* [n_dst cap, max(d_agg,d_in)] scratch: composed rows fed to the update GEMM */
  float* gemm_mid;     /* [n_dst cap, d_out] GIN hidden */
  /* Source deltas of the sum aggregators (GCN / SAGE / GIN), vertex-indexed:
   *   delta       [n, d_in]  δ_u = c_new(u) h_new(u) - c_old(u) h_old(u) of this layer's
   *               sources S(l) (NULL: computed into the workspace);
   *   delta_ready  rows of V_chg(l-1) were written by the previous layer's update, so only
   *               the other sources (Dg) are computed here, and a deleted edge of a changed
   *               source contributes -c_old h_old = δ - c_new h_new (no DeltaLog needed);
   *   delta_next  [n, d_out] set (tcgen05 update, d_out % 4 == 0): this layer's update
   *               writes δ_v of every updated row for the next layer instead of log_out. */
  float* delta;
  float* delta_next;
  int32_t delta_ready;
  /* Sharded state: rows of S / ctx (and of H_out when out_local) are
   * stored per owned vertex at v / row_div (owner(v) = v mod row_div); delta_slot: δ rows
   * indexed by the source's slot in S(l) (frontier src_slot) instead of by vertex, so the
   * δ buffer holds |S(l)| rows.  0 / 0 / 0: unsharded, vertex-indexed. */
  int32_t row_div;
  int32_t out_local;
  int32_t delta_slot;
} rtec_state_t;

/* ---- workspace ---- */
/* per-batch calls (apply / frontier / layers); m_slots bounds the in-place merge scratch */
size_t rtec_workspace_bytes(int64_t n, int64_t max_batch, int64_t m_slots, int32_t max_dim);
/* the same without the [n, max_dim] δ region (callers that pass state.delta) */
size_t rtec_workspace_bytes_ext(int64_t n, int64_t max_batch, int64_t m_slots, int32_t max_dim);
/* bulk build / compaction of m edges */
size_t rtec_build_workspace_bytes(int64_t n, int64_t m);

/* ---- graph store (graph.py) ---- */
/* from_edges (graph.py:81-121): builds both adjacencies with slack capacity
 * (cap = len + max(min_slack, ceil(len*slack))).  err <- InvalidVertex /
 * ConfigError("duplicate edges in bulk load"). */
int rtec_graph_build(rtec_graph_t* g, const int32_t* src, const int32_t* dst, const int64_t* ts,
                     int64_t m, float slack, int32_t min_slack, uint64_t* err,
                     void* ws, size_t ws_bytes, rtec_stream_t stream);
/* Degree histogram of a bulk edge list; err <- InvalidVertex (graph.py:101-102). */
int rtec_graph_count(const int32_t* src, const int32_t* dst, int64_t m, int64_t n, int32_t* out_deg,
                     int32_t* in_deg, uint64_t* err, rtec_stream_t stream);
/* Required slots for a build/compaction of `m` edges at the given slack, given
 * per-vertex run lengths `len` (device) -- written to *slots_dev. */
int rtec_graph_slots_needed(const int32_t* len, int64_t n, float slack, int32_t min_slack,
                            int64_t* slots_dev, void* ws, size_t ws_bytes, rtec_stream_t stream);
/* Compaction: copy every run of `src` into `dst` (fresh arrays) with fresh
 * slack.  Replaces PMA rebalancing (pma.py:304-326). */
int rtec_adj_compact(int64_t n, const rtec_adj_t* src, rtec_adj_t* dst, float slack, int32_t min_slack,
                     void* ws, size_t ws_bytes, rtec_stream_t stream);
/* edges() (graph.py:166-170): all runs of `a` flattened in (vertex, nbr) order;
 * out_ts may be NULL. Caller sizes outputs with num_edges. */
int rtec_adj_export(int64_t n, const rtec_adj_t* a, int32_t* out_v, int32_t* out_nbr, int64_t* out_ts,
                    void* ws, size_t ws_bytes, rtec_stream_t stream);

/* coalesce_batch (graph.py:241-260): net effect per (src, dst), survivors in
 * first-appearance order; *n_out written on device. */
int rtec_batch_coalesce(const int32_t* src, const int32_t* dst, const uint8_t* op, const int64_t* ts,
                        int64_t B, int32_t* out_src, int32_t* out_dst, uint8_t* out_op, int64_t* out_ts,
                        int64_t* n_out, void* ws, size_t ws_bytes, rtec_stream_t stream);

/* apply_batch (graph.py:184-231): validate (range -> InvalidVertex, repeated
 * edge -> ConfigError; first offender in batch order wins; nothing mutated on
 * error), probe, reject duplicate inserts / absent deletes, update degrees,
 * merge both adjacencies, emit DegreeDelta rows. */
int rtec_batch_apply(rtec_graph_t* g, rtec_batch_t* b, const int32_t* src, const int32_t* dst,
                     const uint8_t* op, const int64_t* ts, int64_t B,
                     void* ws, size_t ws_bytes, rtec_stream_t stream);
/* apply_batch in two phases (phase 1: validate + probe + plan, no mutation;
 * phase 2: mutate; 3: both == rtec_batch_apply).  Sharded runs combine the
 * ranks' status words between the phases so an error (or a full arena) on
 * any rank leaves every shard untouched.  Both phases must see the same
 * arguments and workspace. */
int rtec_batch_apply_phase(rtec_graph_t* g, rtec_batch_t* b, const int32_t* src, const int32_t* dst,
                           const uint8_t* op, const int64_t* ts, int64_t B, int32_t phase,
                           void* ws, size_t ws_bytes, rtec_stream_t stream);
/* Close the batch: degree snapshots catch up (out_deg_prev = out_deg ...). */
int rtec_batch_commit(rtec_graph_t* g, const rtec_batch_t* b, rtec_stream_t stream);

/* ---- frontier (Alg. 4 / SPEC frontier.build SPEC.md:311-319, F1 rule) ---- */
/* Layer `l` (0-based).  prev == NULL for l = 0.  src_degree_dependent seeds
 * S with Dg (degree-changed sources) at every layer. */
int rtec_frontier_layer(const rtec_graph_t* g, const rtec_batch_t* b, int32_t l,
                        int32_t src_degree_dependent, const rtec_frontier_t* prev, rtec_frontier_t* f,
                        void* ws, size_t ws_bytes, rtec_stream_t stream);

/* ---- layers ---- */
/* Alg. 1 / Alg. 3 for V_dst(l) \ R(l),
 * full-neighbourhood recompute (models.py:431) for R(l), then the update
 * (operators.py:180) on the affected rows with DeltaLog capture. */
int rtec_layer_incremental(const rtec_graph_t* g, const rtec_batch_t* b, const rtec_layer_t* L,
                           rtec_state_t* st, const rtec_frontier_t* prev, const rtec_frontier_t* f,
                           uint64_t* err, void* ws, size_t ws_bytes, rtec_stream_t stream);
/* layer_embeddings (models.py:461-477) for all vertices (rows == NULL) or the
 * listed rows: bootstrap, refresh, dense fallback and the UER baseline (SPEC.md:455:
 * affected rows over their full in-neighbourhoods).  GAT with rows expects Z / el / er
 * of the changed sources to be current (rtec_gat_project). */
int rtec_layer_full(const rtec_graph_t* g, const rtec_layer_t* L, rtec_state_t* st,
                    const int32_t* rows, const int64_t* n_rows, int64_t max_rows, uint64_t* err,
                    void* ws, size_t ws_bytes, rtec_stream_t stream);
/* GAT f_nn / logit halves for rows (models.py:265-279): Z = W h, el, er.  With the
 * layer's tcgen05 operand images (L->Wt_hi) and an A-image scratch `a_img` of
 * ceil(rows/128)*128 x ceil(d_in/32)*32 floats, the rows are packed and Z runs on
 * tcgen05 (3xTF32); a_img == NULL -> SIMT fp32.  A non-finite Z row -> NumericError
 * (position = vertex) in *err. */
int rtec_gat_project(const rtec_layer_t* L, const float* H, const int32_t* rows, const int64_t* n_rows,
                     int64_t n_or_max_rows, float* Z, float* el, float* er,
                     float* Z_log, float* er_log, const uint64_t* err, float* a_img, rtec_stream_t stream);

/* Per-source projections of the payload / gate models for all vertices
 * (rows == NULL) or the listed rows (V_chg(l-1) before layer l):
 *   PINSAGE P = alpha relu(Q h + q)             [n, d_in]   (models.py:157-159)
 *   MONET   P = exp(0.5 (h-mu)^T Wq (h-mu))     [n, 1]      (models.py:211-213)
 *   GGCN    P = [Wg_src h ; Wg_dst h]           [n, 2 d_in] (models.py:301-305)
 * P_log (optional) receives the overwritten rows, indexed like the rows list
 * (the old payloads the incremental retraction reads).  Other models: no-op. */
int rtec_project(const rtec_layer_t* L, const float* H, const int32_t* rows, const int64_t* n_rows,
                 int64_t n_or_max_rows, float* P, float* P_log, const uint64_t* err, rtec_stream_t stream);

/* Dense update GEMM on gathered rows (operators.py:180; linalg.py:22):
 * Y[i] = act(X[i] · W^T) (act: 0 none, 1 relu).  Rows i < *n_rows. */
int rtec_update_gemm(const float* X, int64_t ldx, const float* W, int32_t d_in, int32_t d_out,
                     const int64_t* n_rows, int64_t max_rows, int32_t act, float* Y, int64_t ldy,
                     const int32_t* scatter_rows, float* scatter_dst, float* log_dst,
                     rtec_stream_t stream);

/* Split + swizzle W[d_out, d_in] for the tcgen05 update GEMM: Bhi/Blo each
 * ceil(d_in/32) * round_up(d_out,16) * 32 floats.  d_out <= 256. */
int rtec_gemm_prepare_weights(const float* W, int32_t d_in, int32_t d_out, float* Bhi, float* Blo,
                              rtec_stream_t stream);

/* ---- vertex sharding (one process per GPU) ----
 * Rank p of P holds the edges whose dst it owns (owner(v) = v mod P) over LOCAL
 * ids: [0, n_own) its owned vertices (local i <-> global p + P i), [n_own, n_loc)
 * ghosts (sources with an out-edge into the shard).  The graph, frontier and
 * layer calls above run unchanged on the local graph; the calls below keep the
 * ghost rows coherent.  Replaces the paper's CPU-offloaded embedding store
 * with destination-owned rows in HBM. */
#define RTEC_SHARD_MAX_WORLD 32
#define RTEC_SHARD_MAX_MATS 8
typedef struct {
  int32_t rank, world;
  int64_t n;          /* global vertex count */
  int64_t n_own;      /* owned vertices */
  int64_t cap;        /* local id capacity (every per-vertex array of the shard) */
  int32_t* g2l;       /* [n] global -> local id, -1: not on this rank */
  int32_t* l2g;       /* [cap] local -> global id */
  int64_t* n_loc;     /* [1] local ids in use (device) */
  uint32_t* peers;    /* [n_own] bit q: rank q holds a ghost row of this owned vertex */
  int32_t* gout;      /* [cap] global out-degree of every local vertex */
  int32_t* gout_prev; /* [cap] its pre-batch value */
} rtec_shard_t;

/* Validation of a global batch without a graph (graph.py:192-198): range ->
 * InvalidVertex, repeated (src, dst) -> ConfigError; first offender in batch
 * order.  *err is reset first.  Identical on every rank. */
int rtec_batch_validate(const int32_t* src, const int32_t* dst, int64_t B, int64_t n, uint64_t* err,
                        void* ws, size_t ws_bytes, rtec_stream_t stream);
/* Ghost admission for the inserts of a validated global batch (no-op when *err is
 * set).  Receiver: every not-yet-local source of an insert into an owned
 * destination gets the next local id (ascending global id; adm_list = their local
 * ids, *n_adm; sh->n_loc advanced; bm_adm: an all-zero [n]-bit scratch, left
 * zero).  Owner: every (owned source u, rank q) pair whose peers bit was clear is
 * set and listed (send_u = local id of u, send_q, *n_send, peer_count[q]). */
int rtec_shard_admit(const rtec_shard_t* sh, const int32_t* src, const int32_t* dst, const uint8_t* op,
                     int64_t B, uint64_t* err, uint32_t* bm_adm, int32_t* adm_list, int64_t* n_adm,
                     int32_t* send_u, int32_t* send_q, int64_t* n_send, int64_t* peer_count,
                     void* ws, size_t ws_bytes, rtec_stream_t stream);
/* The shard's part of a global batch in batch order, in local ids: updates whose
 * dst this rank owns (l* arrays), lpos = their global position, *n_local. */
int rtec_shard_localize(const rtec_shard_t* sh, const int32_t* src, const int32_t* dst, const uint8_t* op,
                        const int64_t* ts, int64_t B, const uint64_t* err, int32_t* lsrc, int32_t* ldst,
                        uint8_t* lop, int64_t* lts, int32_t* lpos, int64_t* n_local, void* ws, size_t ws_bytes,
                        rtec_stream_t stream);
/* Rows each peer receives from a list of owned local ids (list NULL: 0..max_list-1):
 * peer_count[q] = #{i : peers[list[i]] has bit q}. */
int rtec_shard_count_peers(const rtec_shard_t* sh, const int32_t* list, const int64_t* n_list, int64_t max_list,
                           int64_t* peer_count, rtec_stream_t stream);
/* Pack rows for an all-to-all: segment q starts at peer_off[q] (HOST array of
 * world+1 offsets); each item writes its global id, optionally its global
 * out-degree, and the concatenation of rows mats[j][v] (dims[j] floats; HOST
 * arrays of nmat <= RTEC_SHARD_MAX_MATS device pointers / widths).  Items: list mode
 * (every q in peers[v] of the listed owned v) or pair mode (pair_u / pair_q).
 * cursor: [world] int64 scratch.  Order inside a segment is unspecified. */
int rtec_shard_pack(const rtec_shard_t* sh, int32_t nmat, const float* const* mats, const int32_t* dims,
                    const int64_t* peer_off, const int32_t* list, const int64_t* n_list, int64_t max_list,
                    const int32_t* pair_u, const int32_t* pair_q, int64_t n_pairs, int64_t* cursor,
                    int32_t* out_ids, int32_t* out_deg, float* out_rows, rtec_stream_t stream);
/* k received (global id, rows) items into the ghost rows of mats[] (+ gout / gout_prev
 * from degs when given); out_local[i] = local id (optional). */
int rtec_shard_unpack_rows(const rtec_shard_t* sh, int32_t nmat, float* const* mats, const int32_t* dims,
                           const int32_t* ids, const int32_t* degs, const float* rows, int64_t k,
                           int32_t* out_local, rtec_stream_t stream);
/* V_chg(l) of the shard after layer l, over one or more exchange rounds (clear != 0 on
 * the first: bm_chg zeroed).  The k received changed rows of a round overwrite their
 * ghost rows of H at positions pos_base + [0, k); the owned changed rows own_list[j]
 * (given on the last round) follow; bm_chg, chg_slot[v] = pos, chg_list[pos] = v,
 * *n_chg = total (last round).  Exactly one of
 *   glog:  glog[pos] = the overwritten pre-batch row (owned: own_log[own_slot[v]]) --
 *          the exchanged DeltaLog the next layer retracts with;
 *   delta: delta[v] = c_new h_new - c_old h_old for received rows (c: GCN
 *          1/sqrt(deg + deg_off) if coeff_gcn else 1, 0 for deg 0; global out-degrees),
 *          the source deltas the update epilogue writes for owned rows.
 * The next layer's frontier / retractions read them (rtec_frontier_t.bm_chg / chg_slot). */
int rtec_shard_unpack_changed(const rtec_shard_t* sh, int32_t d, const int32_t* ids, const float* rows, int64_t k,
                              int64_t pos_base, int32_t clear, float* H, const int32_t* own_list,
                              const int64_t* n_own, int64_t max_own, const float* own_log, const int32_t* own_slot,
                              float* glog, float* delta, int32_t coeff_gcn, float deg_off, uint32_t* bm_chg,
                              int32_t* chg_slot, int32_t* chg_list, int64_t* n_chg, rtec_stream_t stream);
/* Global degrees from the globally applied set of a batch (gstatus = per-update
 * status MAX-all-reduced over ranks): sh->gout of local sources, dg_bm (local ids
 * whose global out-degree changed: the F1 Dg seed), bm_touch ([n_own] bits) and the
 * DegreeDelta rows of the OWNED vertices (graph.py:225-230; global ids, ascending;
 * in-degrees from the local graph, exact for owned vertices). */
int rtec_shard_degrees(const rtec_shard_t* sh, const int32_t* src, const int32_t* dst, const uint8_t* op,
                       const uint8_t* gstatus, int64_t B, const int32_t* in_deg, const int32_t* in_deg_prev,
                       uint32_t* bm_touch, uint32_t* dg_bm, int32_t* d_vertex, int32_t* d_old_in,
                       int32_t* d_new_in, int32_t* d_old_out, int32_t* d_new_out, int64_t* n_delta,
                       void* ws, size_t ws_bytes, rtec_stream_t stream);
/* Close the batch: gout_prev catches up, dg_bm / bm_touch cleared. */
int rtec_shard_commit(const rtec_shard_t* sh, const int32_t* src, const int32_t* dst, const uint8_t* gstatus,
                      int64_t B, uint32_t* dg_bm, uint32_t* bm_touch, rtec_stream_t stream);

/* ---- NS baseline (SPEC.md:464 run_ns) ---- */
/* Seeded sampling without replacement of min(len, fanout) in-neighbours (ascending) of
 * every listed row into `sampled` (beg/len set for the rows, nbr filled, *top = total);
 * bm_next <- rows ∪ sampled neighbours (the rows the hop below must provide).
 * fanout in [1, 32]; deterministic in (seed, hop). */
int rtec_ns_sample(const rtec_adj_t* in, const int32_t* rows, const int64_t* n_rows, int64_t max_rows,
                   int32_t fanout, uint64_t seed, int32_t hop, rtec_adj_t* sampled, uint32_t* bm_next,
                   int64_t n, void* ws, size_t ws_bytes, rtec_stream_t stream);
/* ODEC: bm |= rows ∪ in-neighbours(rows) -- one level of the queries'
 * L-hop in-subgraph */
int rtec_in_expand(const rtec_adj_t* in, const int32_t* rows, const int64_t* n_rows, int64_t max_rows, uint32_t* bm,
                   rtec_stream_t stream);
/* ascending id list of the set bits of an n-bit bitmap; *count on device */
int rtec_bitmap_to_list(const uint32_t* bm, int64_t n, int32_t* list, int64_t* count, void* ws, size_t ws_bytes,
                        rtec_stream_t stream);

/* materialize / query final-layer rows (SPEC materialize_h SPEC.md:379). */
int rtec_query(const float* H, int64_t d, const int32_t* ids, int64_t k, float* out, int32_t n,
               uint64_t* err, rtec_stream_t stream);

/* ---- diagnostics ---- */
void rtec_prof_enable(int on);  /* bracket kernels with CUDA events (bench / profiling only) */
size_t rtec_prof_report(char* buf, size_t len, int reset); /* "name count total_ms" lines */
void rtec_struct_sizes(int64_t* out7); /* sizeof adj, graph, batch, frontier, layer, state, shard */
const char* rtec_last_error(void);
int64_t rtec_graph_kernel_nodes(void* graph); /* kernel nodes of a captured cudaGraph_t (launch census) */
const char* rtec_version(void);
int rtec_device_sm_count(void);

#ifdef __cplusplus
}
#endif
#endif /* RTEC_H_ */
