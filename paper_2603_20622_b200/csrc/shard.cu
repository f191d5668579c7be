// shard.cu -- vertex-sharded execution: global degrees and the
// per-layer halo exchange of changed rows.
//
// Partitioning: owner(v) = v mod P.  Rank p's graph shard holds every edge
// whose dst it owns, in both directions (in-runs for aggregation, out-runs
// for frontier expansion), so Alg. 1 for an owned destination is purely
// local once the changed source rows of the previous layer are present.
// Every rank keeps a replica of each layer's input rows (H^0 = X ... H^{L-1})
// that the halo exchange refreshes; out-degrees (GCN's 1/sqrt(d_out(u)+off),
// models.py:98-99, and the Dg seed of the F1 rule) are global, maintained
// here from the globally applied set of each batch.
#include "prims.cuh"

namespace rtec {

constexpr int kSBlk = 256;

__device__ __forceinline__ bool owned_by(int32_t v, int32_t rank, int32_t count) {
  return count <= 1 || v % count == rank;
}

__global__ void k_shard_deg(const int32_t* __restrict__ src, const int32_t* __restrict__ dst,
                            const uint8_t* __restrict__ op, const uint8_t* __restrict__ gst, int64_t B, int32_t* gout,
                            int32_t* gin, uint32_t* bm_touch) {
  int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = tid - lane_id(); i0 < B; i0 += stride) {
    int64_t i = i0 + lane_id();
    bool act = i < B && gst[i];
    int32_t s = act ? src[i] : 0, d = act ? dst[i] : 0;
    if (act) {
      int32_t inc = op[i] == RTEC_OP_INSERT ? 1 : -1;  // graph.py:220-224
      atomicAdd(gout + s, inc);
      atomicAdd(gin + d, inc);
    }
    bm_set_warp(bm_touch, s, act);
    bm_set_warp(bm_touch, d, act);
  }
}

// touched vertices whose (in, out) degree changed -> DegreeDelta rows
// (ascending: words in order, bits in order); dg_bm word = out-degree changed
struct TouchedChanged {
  const uint32_t* touch;
  const int32_t* gout; const int32_t* gout_prev; const int32_t* gin; const int32_t* gin_prev;
  __device__ __forceinline__ uint32_t changed(int64_t w, uint32_t* dg) const {
    uint32_t t = touch[w], c = 0, o = 0;
    while (t) {
      int b = __ffs(t) - 1;
      t &= t - 1;
      int64_t v = w * 32 + b;
      bool oc = gout[v] != gout_prev[v];
      if (oc || gin[v] != gin_prev[v]) c |= 1u << b;
      if (oc) o |= 1u << b;
    }
    if (dg) *dg = o;
    return c;
  }
  __device__ __forceinline__ int64_t operator()(int64_t w) const { return __popc(changed(w, nullptr)); }
};
struct DeltaRows {
  TouchedChanged f;
  uint32_t* dg_bm;
  int32_t* dv; int32_t* doi; int32_t* dni; int32_t* doo; int32_t* dno;
  __device__ __forceinline__ void operator()(int64_t w, int64_t off, int64_t) const {
    uint32_t dg;
    uint32_t c = f.changed(w, &dg);
    dg_bm[w] = dg;
    while (c) {
      int b = __ffs(c) - 1;
      c &= c - 1;
      int32_t v = static_cast<int32_t>(w * 32 + b);
      dv[off] = v;
      doi[off] = f.gin_prev[v];
      dni[off] = f.gin[v];
      doo[off] = f.gout_prev[v];
      dno[off] = f.gout[v];
      ++off;
    }
  }
};

__global__ void k_shard_commit(const int32_t* __restrict__ src, const int32_t* __restrict__ dst,
                               const uint8_t* __restrict__ gst, int64_t B, const int32_t* gout, int32_t* gout_prev,
                               const int32_t* gin, int32_t* gin_prev, uint32_t* bm_touch, uint32_t* dg_bm) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < B; i += (int64_t)gridDim.x * blockDim.x) {
    if (!gst[i]) continue;
    int32_t s = src[i], d = dst[i];
    gout_prev[s] = gout[s];
    gin_prev[d] = gin[d];
    bm_touch[s >> 5] = 0;  // every touched bit belongs to some applied endpoint
    bm_touch[d >> 5] = 0;
    dg_bm[s >> 5] = 0;
  }
}

// ------------------------------------------------------------------ halo exchange
template <bool V4>
__global__ void __launch_bounds__(kSBlk) k_halo_pack(const float* __restrict__ H, int32_t d,
                                                     const int32_t* __restrict__ list, const int64_t* n_list,
                                                     int64_t max_rows, int32_t* send_ids, float* send_rows) {
  int64_t nr = n_list ? *n_list : max_rows;
  int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < nr; i += nw) {
    int32_t v = list[i];
    if (lane_id() == 0) send_ids[i] = v;
    const float* s = H + static_cast<int64_t>(v) * d;
    float* o = send_rows + i * d;
    if (V4) {
      for (int j = lane_id(); j < d / 4; j += 32)
        reinterpret_cast<float4*>(o)[j] = __ldg(reinterpret_cast<const float4*>(s) + j);
    } else {
      for (int j = lane_id(); j < d; j += 32) o[j] = __ldg(s + j);
    }
  }
}

template <bool V4>
__global__ void __launch_bounds__(kSBlk) k_halo_unpack(int32_t rank, int32_t count, int32_t d,
                                                       const int32_t* __restrict__ ids, const float* __restrict__ rows,
                                                       const int64_t* __restrict__ counts, int32_t world,
                                                       int64_t slot_cap, float* H, const float* __restrict__ local_log,
                                                       const int32_t* __restrict__ dst_slot, float* glog,
                                                       uint32_t* bm_chg, int32_t* chg_slot, int32_t* chg_list,
                                                       int64_t* n_chg) {
  int64_t total = static_cast<int64_t>(world) * slot_cap;
  int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  if (blockIdx.x == 0 && threadIdx.x == 0 && n_chg) {
    int64_t t = 0;
    for (int r = 0; r < world; ++r) t += counts[r];
    *n_chg = t;
  }
  for (int64_t k = warp; k < total; k += nw) {
    int r = static_cast<int>(k / slot_cap);
    int64_t j = k - static_cast<int64_t>(r) * slot_cap;
    if (j >= counts[r]) continue;
    int64_t pos = j;
    for (int q = 0; q < r; ++q) pos += counts[q];
    int32_t u = ids[k];
    bool mine = owned_by(u, rank, count);
    if (glog && lane_id() == 0) {
      atomicOr(bm_chg + (u >> 5), 1u << (u & 31));
      chg_slot[u] = static_cast<int32_t>(pos);
      chg_list[pos] = u;
    }
    float* hrow = H + static_cast<int64_t>(u) * d;
    const float* src = rows + k * d;
    float* lrow = glog ? glog + pos * d : nullptr;
    const float* own_old = (glog && mine) ? local_log + static_cast<int64_t>(dst_slot[u]) * d : nullptr;
    if (V4) {
      for (int c = lane_id(); c < d / 4; c += 32) {
        float4 nv = __ldg(reinterpret_cast<const float4*>(src) + c);
        if (mine) {
          if (lrow) reinterpret_cast<float4*>(lrow)[c] = __ldg(reinterpret_cast<const float4*>(own_old) + c);
        } else {
          if (lrow) reinterpret_cast<float4*>(lrow)[c] = reinterpret_cast<const float4*>(hrow)[c];
          reinterpret_cast<float4*>(hrow)[c] = nv;
        }
      }
    } else {
      for (int c = lane_id(); c < d; c += 32) {
        float nv = __ldg(src + c);
        if (mine) {
          if (lrow) lrow[c] = __ldg(own_old + c);
        } else {
          if (lrow) lrow[c] = hrow[c];
          hrow[c] = nv;
        }
      }
    }
  }
}

}  // namespace rtec

using namespace rtec;

extern "C" {

int rtec_shard_degrees(int64_t n, const int32_t* src, const int32_t* dst, const uint8_t* op, const uint8_t* gstatus,
                       int64_t B, int32_t* gout, const int32_t* gout_prev, int32_t* gin, const int32_t* gin_prev,
                       uint32_t* bm_touch, uint32_t* dg_bm, int32_t* d_vertex, int32_t* d_old_in, int32_t* d_new_in,
                       int32_t* d_old_out, int32_t* d_new_out, int64_t* n_delta, void* ws, size_t ws_bytes,
                       rtec_stream_t stream) {
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  RTEC_PROF("shard_degrees", s);
  int64_t words = (n + 31) / 32;
  if (B > 0) k_shard_deg<<<grid_for(B, kSBlk), kSBlk, 0, s>>>(src, dst, op, gstatus, B, gout, gin, bm_touch);
  RTEC_LAUNCH_CHECK("k_shard_deg");
  Ws w(ws, ws_bytes);
  TouchedChanged tc{bm_touch, gout, gout_prev, gin, gin_prev};
  return exclusive_scan(tc, Count{nullptr, words}, words,
                        DeltaRows{tc, dg_bm, d_vertex, d_old_in, d_new_in, d_old_out, d_new_out}, n_delta, w, s);
}

int rtec_shard_commit(const int32_t* src, const int32_t* dst, const uint8_t* gstatus, int64_t B, const int32_t* gout,
                      int32_t* gout_prev, const int32_t* gin, int32_t* gin_prev, uint32_t* bm_touch, uint32_t* dg_bm,
                      rtec_stream_t stream) {
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (B > 0)
    k_shard_commit<<<grid_for(B, kSBlk), kSBlk, 0, s>>>(src, dst, gstatus, B, gout, gout_prev, gin, gin_prev,
                                                        bm_touch, dg_bm);
  RTEC_LAUNCH_CHECK("k_shard_commit");
  return RTEC_OK;
}

int rtec_halo_pack(const float* H, int32_t d, const int32_t* list, const int64_t* n_list, int64_t max_rows,
                   int32_t* send_ids, float* send_rows, rtec_stream_t stream) {
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (max_rows <= 0) return RTEC_OK;
  RTEC_PROF("halo_pack", s);
  const int grid = grid_for(max_rows * 32, kSBlk, kSMs * 8);
  if (d % 4 == 0) k_halo_pack<true><<<grid, kSBlk, 0, s>>>(H, d, list, n_list, max_rows, send_ids, send_rows);
  else k_halo_pack<false><<<grid, kSBlk, 0, s>>>(H, d, list, n_list, max_rows, send_ids, send_rows);
  RTEC_LAUNCH_CHECK("k_halo_pack");
  return RTEC_OK;
}

int rtec_halo_unpack(const rtec_graph_t* g, int32_t d, const int32_t* recv_ids, const float* recv_rows,
                     const int64_t* counts, int32_t world, int64_t slot_cap, float* H, const float* local_log,
                     const int32_t* dst_slot, float* glog, uint32_t* bm_chg, int32_t* chg_slot, int32_t* chg_list,
                     int64_t* n_chg, rtec_stream_t stream) {
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (world < 1 || world > 64) {
    set_error("world size %d out of range", world);
    return RTEC_CONFIG_ERROR;
  }
  if (glog && (!bm_chg || !chg_slot || !chg_list || !local_log || !dst_slot)) {
    set_error("halo_unpack with a DeltaLog needs bm_chg, chg_slot, chg_list, local_log and dst_slot");
    return RTEC_CONFIG_ERROR;
  }
  RTEC_PROF("halo_unpack", s);
  if (glog) RTEC_CUDA(cudaMemsetAsync(bm_chg, 0, sizeof(uint32_t) * ((g->n + 31) / 32), s));
  int64_t total = static_cast<int64_t>(world) * slot_cap;
  const int grid = grid_for(total * 32, kSBlk, kSMs * 8);
  if (d % 4 == 0)
    k_halo_unpack<true><<<grid, kSBlk, 0, s>>>(g->part_rank, g->part_count, d, recv_ids, recv_rows, counts, world,
                                               slot_cap, H, local_log, dst_slot, glog, bm_chg, chg_slot, chg_list,
                                               n_chg);
  else
    k_halo_unpack<false><<<grid, kSBlk, 0, s>>>(g->part_rank, g->part_count, d, recv_ids, recv_rows, counts, world,
                                                slot_cap, H, local_log, dst_slot, glog, bm_chg, chg_slot, chg_list,
                                                n_chg);
  RTEC_LAUNCH_CHECK("k_halo_unpack");
  return RTEC_OK;
}

}  // extern "C"
