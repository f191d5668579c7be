// prims.cuh -- device-wide primitives used by the batch / frontier kernels:
// exclusive scans over functor-generated values and a (key u64, value u32)
// sort (single-CTA bitonic for small batches, LSD radix with 8-bit digits and
// stable warp-match ranking otherwise).  Counts may live on the device: the
// host passes an upper bound for the launch shape, kernels read the real count.
#pragma once
#include "common.cuh"

namespace rtec {

// ---------------------------------------------------------------- count helpers
struct Count {
  const int64_t* dev;  // device count or nullptr
  int64_t host;        // host count (upper bound when dev != nullptr)
  __device__ __forceinline__ int64_t get() const { return dev ? *dev : host; }
};

// ---------------------------------------------------------------- scan
constexpr int kScanBlock = 512;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanBlock * kScanItems;

template <typename T>
__device__ __forceinline__ T block_exclusive_scan(T v, T* smem_warp, T* total) {
  // 512 threads = 16 warps
  int lane = lane_id(), wid = warp_id();
  T x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) smem_warp[wid] = x;
  __syncthreads();
  if (wid == 0) {
    T w = lane < (kScanBlock / 32) ? smem_warp[lane] : T(0);
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      T y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < (kScanBlock / 32)) smem_warp[lane] = w;  // inclusive warp totals
  }
  __syncthreads();
  T warp_off = wid > 0 ? smem_warp[wid - 1] : T(0);
  if (total) *total = smem_warp[kScanBlock / 32 - 1];
  T r = warp_off + x - v;
  __syncthreads();
  return r;
}

// items per thread: 8 for large inputs; 1 below kScanSmall so mid-size scans (a batch of
// ~10^5 updates) still spread over >100 CTAs instead of a latency-bound handful
constexpr int64_t kScanSmall = 262144;
inline int scan_items_for(int64_t max_n) { return max_n <= kScanSmall ? 1 : kScanItems; }

inline int64_t scan_blocks_for(int64_t max_n) {
  const int64_t tile = static_cast<int64_t>(kScanBlock) * scan_items_for(max_n);
  return (max_n + tile - 1) / tile;
}

// whole scan in one CTA when the (host-side) bound fits one tile: one launch instead of three
template <typename F, typename O>
__global__ void __launch_bounds__(kScanBlock) k_scan_one(F f, Count cnt, O out, int64_t* total) {
  RTEC_PDL_ENTRY();
  __shared__ int64_t sw[kScanBlock / 32];
  int64_t n = cnt.get();
  int64_t vals[kScanItems];
  int64_t s = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    int64_t i = static_cast<int64_t>(threadIdx.x) * kScanItems + k;
    vals[k] = (i < n) ? f(i) : 0;
    s += vals[k];
  }
  int64_t tot;
  int64_t off = block_exclusive_scan<int64_t>(s, sw, &tot);
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    int64_t i = static_cast<int64_t>(threadIdx.x) * kScanItems + k;
    if (i < n) out(i, off, vals[k]);
    off += vals[k];
  }
  if (threadIdx.x == 0 && total) *total = tot;
}

// Single-pass scan with decoupled look-back: tiles are claimed in launch order from a
// counter (so every tile's predecessors are running or done), each tile publishes its
// aggregate, then walks back over its predecessors' published words until it meets an
// inclusive prefix.  Word = flag (bits 62-63: 1 aggregate, 2 inclusive prefix) | value.
// One kernel per scan instead of reduce + block-scan + down-sweep (the per-batch pipeline
// runs ~40 scans, most of them latency-bound).
constexpr unsigned long long kLbAgg = 1ull << 62, kLbPrefix = 2ull << 62, kLbMask = (1ull << 62) - 1;

template <typename F, typename O, int ITEMS>
__global__ void __launch_bounds__(kScanBlock) k_scan_1pass(F f, Count cnt, O out, int64_t* total,
                                                           unsigned long long* st, unsigned int* tile_ctr) {
  RTEC_PDL_ENTRY();
  __shared__ int64_t sw[kScanBlock / 32];
  __shared__ int64_t s_prefix;
  __shared__ unsigned int s_tile;
  const int64_t n = cnt.get();
  constexpr int64_t kT = static_cast<int64_t>(kScanBlock) * ITEMS;
  if (threadIdx.x == 0) s_tile = atomicAdd(tile_ctr, 1u);
  __syncthreads();
  const int64_t tile = s_tile;
  const int64_t ntiles = (n + kT - 1) / kT;
  if (tile >= (ntiles > 0 ? ntiles : 1)) return;  // tile 0 runs for n == 0 (writes the total)
  const int64_t base = tile * kT;
  int64_t vals[ITEMS];
  int64_t s = 0;
#pragma unroll
  for (int k = 0; k < ITEMS; ++k) {
    const int64_t i = base + static_cast<int64_t>(threadIdx.x) * ITEMS + k;
    vals[k] = (i < n) ? f(i) : 0;
    s += vals[k];
  }
  int64_t tot;
  int64_t off = block_exclusive_scan<int64_t>(s, sw, &tot);
  if (threadIdx.x < 32) {
    // warp-wide look-back: lane k reads the word of tile j - k, 32 predecessors per step
    volatile unsigned long long* vst = st;
    const int lane = threadIdx.x;
    int64_t excl = 0;
    if (tile == 0) {
      if (lane == 0) atomicExch(st, kLbPrefix | static_cast<unsigned long long>(tot));
    } else {
      if (lane == 0) atomicExch(st + tile, kLbAgg | static_cast<unsigned long long>(tot));
      for (int64_t j = tile - 1;;) {
        const int64_t idx = j - lane;
        const unsigned long long w = idx >= 0 ? vst[idx] : (kLbPrefix | 0ull);
        const unsigned pre = __ballot_sync(0xffffffffu, (w & kLbPrefix) != 0);
        const unsigned ready = __ballot_sync(0xffffffffu, w != 0);
        // lanes up to the nearest inclusive prefix (or all 32) must have published
        const unsigned need = pre ? ((pre & (0u - pre)) << 1) - 1u : 0xffffffffu;
        if ((ready & need) != need) continue;  // a predecessor is still scanning its tile
        int64_t v = (need >> lane) & 1u ? static_cast<int64_t>(w & kLbMask) : 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        excl += v;
        if (pre) break;
        j -= 32;
      }
      if (lane == 0) {
        __threadfence();
        atomicExch(st + tile, kLbPrefix | static_cast<unsigned long long>(excl + tot));
      }
    }
    if (lane == 0) {
      s_prefix = excl;
      if (total && tile == (ntiles > 0 ? ntiles - 1 : 0)) *total = excl + tot;
    }
  }
  __syncthreads();
  off += s_prefix;
#pragma unroll
  for (int k = 0; k < ITEMS; ++k) {
    const int64_t i = base + static_cast<int64_t>(threadIdx.x) * ITEMS + k;
    if (i < n) out(i, off, vals[k]);
    off += vals[k];
  }
}

// Exclusive scan: out(i, prefix, value) is called for every i < count; *total
// (device, may be null) receives the sum.  ws needs scan_blocks_for(max)+2 int64.
// wide: the functor is expensive (dependent global loads per item) -- never the one-CTA path,
// one item per thread over as many CTAs as it takes
template <typename F, typename O>
int exclusive_scan_bs(F f, Count cnt, int64_t max_n, O out, int64_t* total, int64_t* bs, cudaStream_t s,
                      bool wide = false) {
  if (wide) {
    const int64_t nb = (max_n + kScanBlock - 1) / kScanBlock;
    unsigned long long* st = reinterpret_cast<unsigned long long*>(bs);
    unsigned int* ctr = reinterpret_cast<unsigned int*>(bs + nb);
    RTEC_CUDA(cudaMemsetAsync(bs, 0, sizeof(int64_t) * (nb + 1), s));
    launch(k_scan_1pass<F, O, 1>, static_cast<unsigned>(nb > 0 ? nb : 1), kScanBlock, 0, s, f, cnt, out, total, st, ctr);
    RTEC_LAUNCH_CHECK("exclusive_scan");
    return RTEC_OK;
  }
  if (max_n <= kScanTile) {
    launch(k_scan_one<F, O>, 1, kScanBlock, 0, s, f, cnt, out, total);
    RTEC_LAUNCH_CHECK("exclusive_scan");
    return RTEC_OK;
  }
  const int64_t nb = scan_blocks_for(max_n);
  unsigned long long* st = reinterpret_cast<unsigned long long*>(bs);
  unsigned int* ctr = reinterpret_cast<unsigned int*>(bs + nb);
  RTEC_CUDA(cudaMemsetAsync(bs, 0, sizeof(int64_t) * (nb + 1), s));
  if (scan_items_for(max_n) == 1)
    launch(k_scan_1pass<F, O, 1>, static_cast<unsigned>(nb), kScanBlock, 0, s, f, cnt, out, total, st, ctr);
  else
    launch(k_scan_1pass<F, O, kScanItems>, static_cast<unsigned>(nb), kScanBlock, 0, s, f, cnt, out, total, st, ctr);
  RTEC_LAUNCH_CHECK("exclusive_scan");
  return RTEC_OK;
}

template <typename F, typename O>
int exclusive_scan(F f, Count cnt, int64_t max_n, O out, int64_t* total, Ws& ws, cudaStream_t s,
                   bool wide = false) {
  int64_t* bs = ws.alloc<int64_t>((wide ? (max_n + kScanBlock - 1) / kScanBlock : scan_blocks_for(max_n)) + 2);
  RTEC_WS_CHECK(ws);
  return exclusive_scan_bs(f, cnt, max_n, out, total, bs, s, wide);
}

// common out-functors
struct StorePrefix {
  int64_t* dst;
  __device__ __forceinline__ void operator()(int64_t i, int64_t off, int64_t) const { dst[i] = off; }
};

// ---------------------------------------------------------------- fills
// Up to four 4-byte-aligned spans (whole 32-bit words) set to a word pattern in ONE kernel
// launch: one graph node instead of one memset node per span on the per-batch chain.
struct FillSpan {
  void* p;
  int64_t bytes;  // multiple of 4
  uint32_t word;
};
struct Fill4 {
  FillSpan s[4];
  int n;
};
int fill_spans(const Fill4& f, cudaStream_t s);

// ---------------------------------------------------------------- sort
// Sorts (key, val) pairs ascending by key (stable w.r.t. input order) over
// bits [0, bits).  Result lands in keys_out/vals_out.  Needs sort_ws_bytes.
size_t sort_ws_bytes(int64_t max_n);
int sort_pairs(const uint64_t* keys_in, const uint32_t* vals_in, uint64_t* keys_out, uint32_t* vals_out,
               Count cnt, int64_t max_n, int bits, Ws& ws, cudaStream_t s);

inline int bits_for(uint64_t max_key) {
  int b = 0;
  while (b < 64 && (max_key >> b) != 0) ++b;
  return b < 1 ? 1 : b;
}

}  // namespace rtec
