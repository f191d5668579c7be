// frontier.cu -- per-layer affected subgraph (§8(a)-F1).
//
// Alg. 4 with the every-layer source-degree rule:
//   S(l)     = Dg ∪ V_chg(l-1)              (Dg = out-degree-changed sources, GCN only)
//   E_curr(l)= I ∪ D ∪ {(u,w) ∈ G_post : u ∈ S(l)}
//   V_dst(l) = dst(E_curr(l)),  V_chg(l) = V_dst(l)
// V_dst is monotone in l, so layer l only expands the NEW sources
// S(l) \ S(l-1) into a copy of V_dst(l-1).  Sets are n-bit bitmaps; lists are
// ascending id arrays produced by a popcount scan over the bitmap words.
// Expansion is edge-balanced: a prefix over the new sources' out-run lengths
// maps every edge to a thread, and bits are set with warp-aggregated atomicOr.
#include "prims.cuh"

namespace rtec {

constexpr int kFBlk = 256;

// Dg bits and dst(I ∪ D) bits
__global__ void k_seed_layer0(const rtec_batch_t b, int32_t src_degree_dependent, uint32_t* bm_src,
                              uint32_t* bm_dst) {
  RTEC_PDL_ENTRY();
  if (err_set(b.err)) return;
  int64_t nd = *b.n_delta, na = *b.n_applied;
  int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  // loop bound uniform across the warp for the ballot-based helper
  int64_t lim = nd > na ? nd : na;
  for (int64_t i0 = tid - lane_id(); i0 < lim; i0 += stride) {
    int64_t i = i0 + lane_id();
    bool dg = src_degree_dependent && i < nd && b.d_old_out[i] != b.d_new_out[i];
    bm_set_warp(bm_src, dg ? b.d_vertex[i] : 0, dg);
    bool ad = i < na;
    bm_set_warp(bm_dst, ad ? b.a_dst[i] : 0, ad);
  }
}

__global__ void k_union_words(const uint32_t* __restrict__ a, const uint32_t* __restrict__ b, uint32_t* out,
                              int64_t words) {
  RTEC_PDL_ENTRY();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < words; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = a[i] | b[i];
}

// popcount of (a & ~b) per word (b may be null)
struct WordPop {
  const uint32_t* a;
  const uint32_t* b;
  __device__ __forceinline__ uint32_t word(int64_t i) const { return a[i] & (b ? ~b[i] : 0xffffffffu); }
  __device__ __forceinline__ int64_t operator()(int64_t i) const { return __popc(word(i)); }
};

// bitmap -> ascending list: per-word offsets from a popcount scan, then one
// thread per word writes its bits (many CTAs; the scan's out-functor stays cheap)
__global__ void __launch_bounds__(kFBlk) k_word_list(WordPop f, const int64_t* __restrict__ woff, int64_t words,
                                                     int32_t* list, int32_t* slot) {
  RTEC_PDL_ENTRY();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < words; i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t w = f.word(i);
    int64_t off = woff[i];
    while (w) {
      int bit = __ffs(w) - 1;
      w &= w - 1;
      int32_t v = static_cast<int32_t>(i * 32 + bit);
      list[off] = v;
      if (slot) slot[v] = static_cast<int32_t>(off);
      ++off;
    }
  }
}

static int bitmap_to_list(WordPop f, int64_t words, int32_t* list, int32_t* slot, int64_t* count, int64_t* woff,
                          Ws& w, cudaStream_t s) {
  RTEC_TRY(exclusive_scan(f, Count{nullptr, words}, words, StorePrefix{woff}, count, w, s));
  launch(k_word_list, grid_for(words, kFBlk), kFBlk, 0, s, f, woff, words, list, slot);
  RTEC_LAUNCH_CHECK("k_word_list");
  return RTEC_OK;
}

struct OutLenOf {
  const int32_t* list;
  const int32_t* len;
  __device__ __forceinline__ int64_t operator()(int64_t i) const { return len[list[i]]; }
};
struct StoreOffTailF {
  int64_t* dst;
  const int64_t* n;
  __device__ __forceinline__ void operator()(int64_t i, int64_t off, int64_t v) const {
    dst[i] = off;
    if (i == *n - 1) dst[i + 1] = off + v;
  }
};

// Direction-optimising switch (Beamer et al.): push when the new sources' out-edges
// are a small part of the graph, pull (bottom-up over in-runs, early exit) otherwise.
__device__ __forceinline__ bool pull_mode(const int64_t* n_new, const int64_t* off, const int64_t* num_edges) {
  int64_t N = *n_new;
  return N > 0 && off[N] * 16 > *num_edges;
}

// edge-balanced expansion of the new sources' out-runs into bm_dst (push)
__global__ void __launch_bounds__(kFBlk) k_expand(const int32_t* __restrict__ nlist, const int64_t* n_new,
                                                  const int64_t* __restrict__ off, rtec_adj_t out,
                                                  uint32_t* bm_dst, const int64_t* num_edges) {
  RTEC_PDL_ENTRY();
  int64_t N = *n_new;
  if (N == 0 || pull_mode(n_new, off, num_edges)) return;
  int64_t E = off[N];
  int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e0 = tid - lane_id(); e0 < E; e0 += stride) {
    int64_t e = e0 + lane_id();
    bool act = e < E;
    int32_t w = 0;
    if (act) {
      // owner: last i with off[i] <= e
      int64_t lo = 0, hi = N;
      while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if (off[mid] <= e) lo = mid + 1;
        else hi = mid;
      }
      int64_t i = lo - 1;
      int32_t u = nlist[i];
      w = out.nbr[out.beg[u] + (e - off[i])];
    }
    bm_set_warp(bm_dst, w, act);
  }
}

// bottom-up: thread per vertex, 32 consecutive vertices = one bitmap word owned by one warp
__global__ void __launch_bounds__(kFBlk) k_pull(const uint32_t* __restrict__ bm_src, const uint32_t* __restrict__ prev_src,
                                                const int64_t* n_new, const int64_t* __restrict__ off,
                                                const int64_t* num_edges, rtec_adj_t in, int64_t n, uint32_t* bm_dst) {
  RTEC_PDL_ENTRY();
  if (!pull_mode(n_new, off, num_edges)) return;
  int64_t words = (n + 31) / 32;
  int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t v0 = tid - lane_id(); v0 < words * 32; v0 += stride) {
    int64_t v = v0 + lane_id();
    int64_t w = v0 >> 5;
    uint32_t have = bm_dst[w];
    bool hit = (have >> lane_id()) & 1u;
    if (!hit && v < n) {
      int64_t b = in.beg[v];
      int32_t L = in.len[v];
      for (int32_t j = 0; j < L; ++j) {
        int32_t u = in.nbr[b + j];
        uint32_t word = __ldg(bm_src + (u >> 5)) & (prev_src ? ~__ldg(prev_src + (u >> 5)) : 0xffffffffu);
        if ((word >> (u & 31)) & 1u) {
          hit = true;
          break;
        }
      }
    }
    unsigned bal = __ballot_sync(0xffffffffu, hit);
    if (lane_id() == 0) bm_dst[w] = have | bal;
  }
}

// |E_curr(l)| = Σ_{u∈S} outdeg_post(u) + |{e ∈ I : src ∉ S}| + |D|; plus list sizes
__global__ void k_counters(const int32_t* __restrict__ slist, const int64_t* n_src, const int64_t* n_dst,
                           const int32_t* __restrict__ out_len, const int32_t* __restrict__ in_len,
                           const int32_t* __restrict__ dlist, const rtec_batch_t b, const uint32_t* bm_src,
                           int64_t* counters) {
  RTEC_PDL_ENTRY();
  int64_t ns = *n_src, nd = *n_dst, na = err_set(b.err) ? 0 : *b.n_applied;
  int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t e = 0, sin = 0;
  for (int64_t i = tid; i < ns; i += stride) e += out_len[slist[i]];
  for (int64_t i = tid; i < na; i += stride) {
    if (b.a_op[i] == RTEC_OP_DELETE) e += 1;
    else if (!bm_test(bm_src, b.a_src[i])) e += 1;
  }
  for (int64_t i = tid; i < nd; i += stride) sin += in_len[dlist[i]];
  e = warp_sum(e);
  sin = warp_sum(sin);
  if (lane_id() == 0) {
    atomicAdd(reinterpret_cast<unsigned long long*>(counters + 0), static_cast<unsigned long long>(e));
    atomicAdd(reinterpret_cast<unsigned long long*>(counters + 5), static_cast<unsigned long long>(sin));
  }
  if (tid == 0) {
    counters[1] = nd;
    counters[2] = ns;
  }
}

size_t frontier_ws_bytes(int64_t n) {
  int64_t words = (n + 31) / 32;
  return sizeof(int32_t) * (n + 1) + sizeof(int64_t) * (n + 2) + sizeof(int64_t) * (words + 1) + 256 * 5 +
         sizeof(int64_t) * (scan_blocks_for(n > words ? n : words) + 2) * 4 + 8192;
}

}  // namespace rtec

using namespace rtec;

extern "C" int rtec_frontier_layer(const rtec_graph_t* g, const rtec_batch_t* b, int32_t l,
                                   int32_t src_degree_dependent, const rtec_frontier_t* prev, rtec_frontier_t* f,
                                   void* ws, size_t ws_bytes, rtec_stream_t stream) {
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  int64_t n = g->n;
  int64_t words = (n + 31) / 32;
  if (l > 0 && prev == nullptr) {
    set_error("frontier layer %d needs the previous layer's frontier", l);
    return RTEC_CONFIG_ERROR;
  }
  RTEC_PROF("frontier_layer", s);
  Ws w(ws, ws_bytes);
  int32_t* nlist = w.alloc<int32_t>(n + 1);
  int64_t* n_new = w.alloc<int64_t>(4 + n + 2);  // n_new[4], then noff[n + 2]
  int64_t* noff = n_new + 4;
  int64_t* woff = w.alloc<int64_t>(words + 1);
  RTEC_WS_CHECK(w);
  // counters, n_new + noff[0] and (layer 0) both bitmaps cleared by one fill kernel
  Fill4 clr{};
  clr.s[0] = FillSpan{f->counters, static_cast<int64_t>(sizeof(int64_t)) * 8, 0u};
  clr.s[1] = FillSpan{n_new, static_cast<int64_t>(sizeof(int64_t)) * 5, 0u};
  clr.n = 2;
  if (l == 0) {
    clr.s[2] = FillSpan{f->bm_src, static_cast<int64_t>(sizeof(uint32_t)) * words, 0u};
    clr.s[3] = FillSpan{f->bm_dst, static_cast<int64_t>(sizeof(uint32_t)) * words, 0u};
    clr.n = 4;
  }
  RTEC_TRY(fill_spans(clr, s));
  const uint32_t* prev_src = nullptr;
  if (l == 0) {
    // sharded: Dg is the global out-degree change set, not the shard's DegreeDelta
    launch(k_seed_layer0, grid_for(b->cap * 2, kFBlk), kFBlk, 0, s, *b, b->dg_bm ? 0 : src_degree_dependent, f->bm_src,
                                                                 f->bm_dst);
    if (b->dg_bm && src_degree_dependent)
      launch(k_union_words, grid_for(words, kFBlk), kFBlk, 0, s, f->bm_src, b->dg_bm, f->bm_src, words);
  } else {
    // S(l) = S(l-1) ∪ V_chg(l-1); V_dst(l) starts as V_dst(l-1) (this shard's part when sharded)
    const uint32_t* chg = prev->bm_chg ? prev->bm_chg : prev->bm_dst;
    launch(k_union_words, grid_for(words, kFBlk), kFBlk, 0, s, prev->bm_src, chg, f->bm_src, words);
    RTEC_CUDA(cudaMemcpyAsync(f->bm_dst, prev->bm_dst, sizeof(uint32_t) * words, cudaMemcpyDeviceToDevice, s));
    prev_src = prev->bm_src;
  }
  // new sources N = S(l) \ S(l-1)
  WordPop np{f->bm_src, prev_src};
  RTEC_TRY(bitmap_to_list(np, words, nlist, nullptr, n_new, woff, w, s));
  RTEC_TRY(exclusive_scan(OutLenOf{nlist, g->out.len}, Count{n_new, n}, n, StoreOffTailF{noff, n_new}, nullptr, w, s));
  {
    RTEC_PROF("k_expand", s);
    launch(k_expand, kSMs * 8, kFBlk, 0, s, nlist, n_new, noff, g->out, f->bm_dst, g->num_edges);
    launch(k_pull, kSMs * 8, kFBlk, 0, s, f->bm_src, prev_src, n_new, noff, g->num_edges, g->in, n, f->bm_dst);
  }
  RTEC_LAUNCH_CHECK("k_expand");
  // lists + slots
  WordPop sp{f->bm_src, nullptr};
  RTEC_TRY(bitmap_to_list(sp, words, f->src_list, f->src_slot, f->n_src, woff, w, s));
  WordPop dp{f->bm_dst, nullptr};
  RTEC_TRY(bitmap_to_list(dp, words, f->dst_list, f->dst_slot, f->n_dst, woff, w, s));
  launch(k_counters, kSMs * 2, kFBlk, 0, s, f->src_list, f->n_src, f->n_dst, g->out.len, g->in.len, f->dst_list, *b,
                                        f->bm_src, f->counters);
  RTEC_LAUNCH_CHECK("k_counters");
  return RTEC_OK;
}

// ------------------------------------------------------------------ NS baseline (SPEC.md:464 run_ns)
// Seeded neighbour sampling without replacement: row v keeps min(len, fanout) of its
// in-neighbours, chosen by Floyd's algorithm over a counter-hash RNG (seed, hop, v, j),
// written in ascending order; every kept neighbour and v itself are marked in bm_next
// (the rows whose embeddings the hop below must provide).
namespace rtec {

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

struct SampleCount {
  const int32_t* rows;
  const int32_t* len;
  int32_t fanout;
  __device__ __forceinline__ int64_t operator()(int64_t i) const {
    int32_t L = len[rows[i]];
    return L < fanout ? L : fanout;
  }
};
struct SampleBeg {
  const int32_t* rows;
  int64_t* beg;
  int32_t* len;
  __device__ __forceinline__ void operator()(int64_t i, int64_t off, int64_t v) const {
    beg[rows[i]] = off;
    len[rows[i]] = static_cast<int32_t>(v);
  }
};

__global__ void __launch_bounds__(kFBlk) k_ns_sample(rtec_adj_t in, const int32_t* __restrict__ rows,
                                                     const int64_t* n_rows, int64_t max_rows, int32_t fanout,
                                                     uint64_t seed, int32_t hop, rtec_adj_t smp, uint32_t* bm_next) {
  RTEC_PDL_ENTRY();
  const int64_t nr = n_rows ? *n_rows : max_rows;
  int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int lane = lane_id();
  for (int64_t i = warp; i < nr; i += nw) {
    const int32_t v = rows[i];
    const int32_t L = in.len[v];
    const int64_t b = in.beg[v];
    const int32_t k = L < fanout ? L : fanout;
    const int64_t o = smp.beg[v];
    if (lane == 0) atomicOr(bm_next + (v >> 5), 1u << (v & 31));
    if (k == L) {  // keep every neighbour
      for (int32_t j = lane; j < L; j += 32) {
        int32_t u = in.nbr[b + j];
        smp.nbr[o + j] = u;
        atomicOr(bm_next + (u >> 5), 1u << (u & 31));
      }
      continue;
    }
    // Floyd: for j = L-k .. L-1 draw t in [0, j]; take t unless taken, else j.  Lane q keeps pick q.
    int32_t pick = -1;
    for (int32_t q = 0; q < k; ++q) {
      const int32_t j = L - k + q;
      const uint64_t h = mix64(seed ^ mix64((static_cast<uint64_t>(hop) << 56) ^ (static_cast<uint64_t>(v) << 24) ^
                                            static_cast<uint64_t>(j)));
      const int32_t t = static_cast<int32_t>(h % static_cast<uint64_t>(j + 1));
      const bool taken = __any_sync(0xffffffffu, lane < q && pick == t);
      if (lane == q) pick = taken ? j : t;
    }
    // ascending order of the picked positions (k <= 32: rank by comparison)
    int32_t rank = 0;
    for (int32_t q = 0; q < k; ++q) {
      int32_t other = __shfl_sync(0xffffffffu, pick, q);
      if (lane < k && other < pick) ++rank;
    }
    if (lane < k) {
      int32_t u = in.nbr[b + pick];
      smp.nbr[o + rank] = u;
      atomicOr(bm_next + (u >> 5), 1u << (u & 31));
    }
  }
}

}  // namespace rtec

extern "C" int rtec_ns_sample(const rtec_adj_t* in, const int32_t* rows, const int64_t* n_rows, int64_t max_rows,
                              int32_t fanout, uint64_t seed, int32_t hop, rtec_adj_t* sampled, uint32_t* bm_next,
                              int64_t n, void* ws, size_t ws_bytes, rtec_stream_t stream) {
  if (fanout < 1 || fanout > 32) {
    set_error("NS fanout %d outside [1, 32]", fanout);
    return RTEC_CONFIG_ERROR;
  }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  Ws w(ws, ws_bytes);
  RTEC_CUDA(cudaMemsetAsync(bm_next, 0, sizeof(uint32_t) * ((n + 31) / 32), s));
  RTEC_TRY(exclusive_scan(SampleCount{rows, in->len, fanout}, Count{n_rows, max_rows}, max_rows,
                          SampleBeg{rows, sampled->beg, sampled->len}, sampled->top, w, s));
  launch(k_ns_sample, kSMs * 8, kFBlk, 0, s, *in, rows, n_rows, max_rows, fanout, seed, hop, *sampled, bm_next);
  RTEC_LAUNCH_CHECK("k_ns_sample");
  return RTEC_OK;
}

extern "C" int rtec_bitmap_to_list(const uint32_t* bm, int64_t n, int32_t* list, int64_t* count, void* ws,
                                   size_t ws_bytes, rtec_stream_t stream) {
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  Ws w(ws, ws_bytes);
  const int64_t words = (n + 31) / 32;
  int64_t* woff = w.alloc<int64_t>(words + 1);
  RTEC_WS_CHECK(w);
  return bitmap_to_list(WordPop{bm, nullptr}, words, list, nullptr, count, woff, w, s);
}

// ------------------------------------------------------------------ ODEC (SPEC.md:473 run_odec)
// bm_out |= rows ∪ in-neighbours(rows): one level of the queries' L-hop in-subgraph.
namespace rtec {
__global__ void __launch_bounds__(kFBlk) k_in_expand(rtec_adj_t in, const int32_t* __restrict__ rows,
                                                     const int64_t* n_rows, int64_t max_rows, uint32_t* bm) {
  RTEC_PDL_ENTRY();
  const int64_t nr = n_rows ? *n_rows : max_rows;
  int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < nr; i += nw) {
    const int32_t v = rows[i];
    if (lane_id() == 0) atomicOr(bm + (v >> 5), 1u << (v & 31));
    const int64_t b = in.beg[v];
    const int32_t L = in.len[v];
    for (int32_t j0 = 0; j0 < L; j0 += 32) {
      const int32_t j = j0 + lane_id();
      const bool act = j < L;
      bm_set_warp(bm, act ? in.nbr[b + j] : 0, act);
    }
  }
}
}  // namespace rtec

extern "C" int rtec_in_expand(const rtec_adj_t* in, const int32_t* rows, const int64_t* n_rows, int64_t max_rows,
                              uint32_t* bm, rtec_stream_t stream) {
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (max_rows <= 0) return RTEC_OK;
  launch(k_in_expand, kSMs * 8, kFBlk, 0, s, *in, rows, n_rows, max_rows, bm);
  RTEC_LAUNCH_CHECK("k_in_expand");
  return RTEC_OK;
}
