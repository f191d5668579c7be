// prims.cu -- scan-of-block-sums and the (u64 key, u32 value) sort.
#include <stdarg.h>

#include <map>
#include <vector>

#include "prims.cuh"

#include <stdlib.h>

namespace rtec {

// ---------------------------------------------------------------- errors
static thread_local std::string g_last_error;

void set_error(const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
}

int cuda_status(cudaError_t e, const char* where) {
  set_error("CUDA error %s (%s) at %s", cudaGetErrorName(e), cudaGetErrorString(e), where);
  return RTEC_CUDA_ERROR;
}

const char* last_error_cstr() { return g_last_error.c_str(); }

// ---------------------------------------------------------------- timing hook
bool g_prof_on = false;
struct ProfRec {
  const char* name;
  cudaEvent_t a, b;
};
static std::vector<ProfRec> g_prof;
static std::vector<size_t> g_prof_open;

void prof_begin(const char* name, cudaStream_t s) {
  ProfRec r{name, nullptr, nullptr};
  cudaEventCreate(&r.a);
  cudaEventCreate(&r.b);
  cudaEventRecord(r.a, s);
  g_prof_open.push_back(g_prof.size());
  g_prof.push_back(r);
}

void prof_end(cudaStream_t s) {
  if (g_prof_open.empty()) return;
  size_t i = g_prof_open.back();
  g_prof_open.pop_back();
  cudaEventRecord(g_prof[i].b, s);
}

// "name count total_ms\n" lines, aggregated by name; syncs on the events.
std::string prof_report(bool reset) {
  std::map<std::string, std::pair<long, double>> agg;
  for (auto& r : g_prof) {
    float ms = 0.f;
    cudaEventSynchronize(r.b);
    cudaEventElapsedTime(&ms, r.a, r.b);
    auto& e = agg[r.name];
    e.first += 1;
    e.second += ms;
  }
  std::string out;
  char line[256];
  for (auto& kv : agg) {
    snprintf(line, sizeof(line), "%s %ld %.6f\n", kv.first.c_str(), kv.second.first, kv.second.second);
    out += line;
  }
  if (reset) {
    for (auto& r : g_prof) {
      cudaEventDestroy(r.a);
      cudaEventDestroy(r.b);
    }
    g_prof.clear();
    g_prof_open.clear();
  }
  return out;
}

// ---------------------------------------------------------------- per-device host state
int cur_device() {
  int d = 0;
  if (cudaGetDevice(&d) != cudaSuccess || d < 0 || d >= kMaxDevices) d = 0;
  return d;
}

int sm_count() {
  static int cache[kMaxDevices] = {0};
  const int d = cur_device();
  if (!cache[d]) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, d);
    cache[d] = v > 0 ? v : 148;
  }
  return cache[d];
}

bool pdl_on() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("RTEC_PDL");
    on = e ? (atoi(e) != 0) : 1;
  }
  return on != 0;
}

// side stream + fork / join events of the current device (the two-stream passes)
cudaStream_t side_stream() {
  static cudaStream_t st[kMaxDevices] = {};
  const int d = cur_device();
  if (!st[d]) cudaStreamCreateWithFlags(&st[d], cudaStreamNonBlocking);
  return st[d];
}
cudaEvent_t side_fork() {
  static cudaEvent_t e[kMaxDevices] = {};
  const int d = cur_device();
  if (!e[d]) cudaEventCreateWithFlags(&e[d], cudaEventDisableTiming);
  return e[d];
}
cudaEvent_t side_join() {
  static cudaEvent_t e[kMaxDevices] = {};
  const int d = cur_device();
  if (!e[d]) cudaEventCreateWithFlags(&e[d], cudaEventDisableTiming);
  return e[d];
}

// ---------------------------------------------------------------- small sort
// One CTA of 1024 threads, bitonic over (key, val) lexicographic; N <= 2048.
constexpr int kSmallSort = 2048;

__global__ void __launch_bounds__(1024) k_sort_small(const uint64_t* __restrict__ kin, const uint32_t* __restrict__ vin,
                                                     uint64_t* kout, uint32_t* vout, Count cnt) {
  RTEC_PDL_ENTRY();
  __shared__ uint64_t sk[kSmallSort];
  __shared__ uint32_t sv[kSmallSort];
  int64_t n = cnt.get();
  int N = 2;
  while (N < n) N <<= 1;
  for (int i = threadIdx.x; i < N; i += blockDim.x) {
    if (i < n) {
      sk[i] = kin[i];
      sv[i] = vin[i];
    } else {
      sk[i] = ~0ull;
      sv[i] = 0xffffffffu;
    }
  }
  __syncthreads();
  for (int size = 2; size <= N; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int t = threadIdx.x; t < N / 2; t += blockDim.x) {
        int lo = 2 * t - (t & (stride - 1));
        int hi = lo + stride;
        bool up = ((lo & size) == 0);
        uint64_t ka = sk[lo], kb = sk[hi];
        uint32_t va = sv[lo], vb = sv[hi];
        bool gt = (ka > kb) || (ka == kb && va > vb);
        if (gt == up) {
          sk[lo] = kb;
          sk[hi] = ka;
          sv[lo] = vb;
          sv[hi] = va;
        }
      }
      __syncthreads();
    }
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    kout[i] = sk[i];
    vout[i] = sv[i];
  }
}

// One CTA of 1024 threads, n <= 1024, one (key, val) per thread: LSD radix sort over `bits`
// with 8-bit digits in shared memory.  A pass ranks each element stably among equal digits
// (warp match + per-warp digit counts, warps in index order), then scatters; ~4 barriers per
// pass instead of the ~55 compare stages of a bitonic network.
__global__ void __launch_bounds__(1024) k_sort_reg(const uint64_t* __restrict__ kin, const uint32_t* __restrict__ vin,
                                                   uint64_t* kout, uint32_t* vout, Count cnt, int bits) {
  RTEC_PDL_ENTRY();
  __shared__ uint32_t whist[32][257];  // per-warp digit counts, then per-warp exclusive offsets
  __shared__ uint32_t boff[256];
  __shared__ uint64_t sk[1024];
  __shared__ uint32_t sv[1024];
  const int64_t n = cnt.get();
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const bool live = t < n;
  uint64_t key = live ? kin[t] : ~0ull;
  uint32_t val = live ? vin[t] : 0xffffffffu;
  const unsigned lt = (1u << lane) - 1u;
  for (int shift = 0; shift < bits; shift += 8) {
    for (int i = t; i < 32 * 257; i += 1024) (&whist[0][0])[i] = 0;
    __syncthreads();
    const int dg = live ? static_cast<int>((key >> shift) & 0xff) : 256;  // padding sorts last
    const unsigned peers = __match_any_sync(0xffffffffu, dg);
    const uint32_t rk = __popc(peers & lt);
    if ((__ffs(peers) - 1) == lane) whist[w][dg] = __popc(peers);
    __syncthreads();
    if (t < 257) {  // per digit: exclusive offsets over warps, total
      uint32_t run = 0;
      for (int q = 0; q < 32; ++q) {
        const uint32_t c = whist[q][t];
        whist[q][t] = run;
        run += c;
      }
      if (t < 256) boff[t] = run;
    }
    __syncthreads();
    if (t < 32) {  // exclusive scan of the 256 digit totals (8 per lane)
      uint32_t loc[8], sum = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        loc[j] = boff[t * 8 + j];
        sum += loc[j];
      }
      uint32_t inc = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
      }
      uint32_t ex = inc - sum;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        boff[t * 8 + j] = ex;
        ex += loc[j];
      }
    }
    __syncthreads();
    if (live) {
      const uint32_t pos = boff[dg] + whist[w][dg] + rk;
      sk[pos] = key;
      sv[pos] = val;
    }
    __syncthreads();
    if (live) {
      key = sk[t];
      val = sv[t];
    }
  }
  if (live) {
    kout[t] = key;
    vout[t] = val;
  }
}

// ---------------------------------------------------------------- fills
__global__ void k_fill4(Fill4 f) {
  RTEC_PDL_ENTRY();
  int64_t w[4], tot = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    w[k] = k < f.n ? f.s[k].bytes / 4 : 0;
    tot += w[k];
  }
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t j = i;
    int k = 0;
    while (j >= w[k]) {
      j -= w[k];
      ++k;
    }
    static_cast<uint32_t*>(f.s[k].p)[j] = f.s[k].word;
  }
}

int fill_spans(const Fill4& f, cudaStream_t s) {
  int64_t tot = 0;
  for (int k = 0; k < f.n; ++k) tot += f.s[k].bytes / 4;
  if (tot <= 0) return RTEC_OK;
  launch(k_fill4, grid_for(tot, 256, kSMs * 4), 256, 0, s, f);
  RTEC_LAUNCH_CHECK("k_fill4");
  return RTEC_OK;
}

// ---------------------------------------------------------------- radix sort
constexpr int kRxBlock = 256;
constexpr int kRxItems = 8;
constexpr int kRxBins = 256;
// items per thread: fewer for mid-size sorts (a batch of ~10^5 updates) so >100 CTAs take part
inline int rx_items_for(int64_t max_n) { return max_n <= 131072 ? 1 : (max_n <= 524288 ? 4 : kRxItems); }

template <int ITEMS>
__global__ void __launch_bounds__(kRxBlock) k_rx_hist(const uint64_t* __restrict__ keys, Count cnt, int shift,
                                                      int64_t ntiles, uint32_t* __restrict__ counts) {
  RTEC_PDL_ENTRY();
  __shared__ uint32_t hist[kRxBins];
  hist[threadIdx.x] = 0;
  __syncthreads();
  int64_t n = cnt.get();
  int64_t base = static_cast<int64_t>(blockIdx.x) * kRxBlock * ITEMS;
#pragma unroll
  for (int k = 0; k < ITEMS; ++k) {
    int64_t i = base + k * kRxBlock + threadIdx.x;
    if (i < n) atomicAdd(&hist[(keys[i] >> shift) & 0xff], 1u);
  }
  __syncthreads();
  counts[static_cast<int64_t>(threadIdx.x) * ntiles + blockIdx.x] = hist[threadIdx.x];
}

template <int ITEMS>
__global__ void __launch_bounds__(kRxBlock) k_rx_scatter(const uint64_t* __restrict__ kin, const uint32_t* __restrict__ vin,
                                                         uint64_t* __restrict__ kout, uint32_t* __restrict__ vout,
                                                         Count cnt, int shift, int64_t ntiles,
                                                         const int64_t* __restrict__ offsets) {
  RTEC_PDL_ENTRY();
  constexpr int kWarps = kRxBlock / 32;
  __shared__ uint32_t run[kRxBins];
  __shared__ uint32_t whist[kWarps][kRxBins];
  __shared__ int64_t goff[kRxBins];
  int t = threadIdx.x, lane = lane_id(), wid = warp_id();
  run[t] = 0;
  for (int w = 0; w < kWarps; ++w) whist[w][t] = 0;
  goff[t] = offsets[static_cast<int64_t>(t) * ntiles + blockIdx.x];
  __syncthreads();
  int64_t n = cnt.get();
  int64_t base = static_cast<int64_t>(blockIdx.x) * kRxBlock * ITEMS;
  unsigned lt_mask = (1u << lane) - 1u;
  for (int k = 0; k < ITEMS; ++k) {
    int64_t i = base + k * kRxBlock + t;
    bool valid = i < n;
    uint64_t key = valid ? kin[i] : 0;
    uint32_t val = valid ? vin[i] : 0;
    int d = valid ? static_cast<int>((key >> shift) & 0xff) : -1;
    unsigned peers = __match_any_sync(0xffffffffu, d);
    int rank_w = __popc(peers & lt_mask);
    if (valid && (__ffs(peers) - 1) == lane) whist[wid][d] = __popc(peers);
    __syncthreads();
    uint32_t pos = 0;
    if (valid) {
      pos = run[d] + rank_w;
      for (int w = 0; w < wid; ++w) pos += whist[w][d];
    }
    __syncthreads();
    {
      uint32_t add = 0;
      for (int w = 0; w < kWarps; ++w) {
        add += whist[w][t];
        whist[w][t] = 0;
      }
      run[t] += add;
    }
    if (valid) {
      int64_t o = goff[d] + pos;
      kout[o] = key;
      vout[o] = val;
    }
    __syncthreads();
  }
}

size_t sort_ws_bytes(int64_t max_n) {
  const int64_t tile = static_cast<int64_t>(kRxBlock) * rx_items_for(max_n);
  int64_t ntiles = (max_n + tile - 1) / tile;
  if (ntiles < 1) ntiles = 1;
  size_t b = 0;
  auto add = [&](size_t x) { b += (x + 255) & ~size_t(255); };
  add(sizeof(uint64_t) * max_n);
  add(sizeof(uint32_t) * max_n);
  add(sizeof(uint64_t) * max_n);
  add(sizeof(uint32_t) * max_n);
  add(sizeof(uint32_t) * kRxBins * ntiles);
  add(sizeof(int64_t) * kRxBins * ntiles);
  add(sizeof(int64_t) * (scan_blocks_for(kRxBins * ntiles) + 2));
  return b + 4096;
}

struct U32At {
  const uint32_t* p;
  __device__ __forceinline__ int64_t operator()(int64_t i) const { return p[i]; }
};

int sort_pairs(const uint64_t* keys_in, const uint32_t* vals_in, uint64_t* keys_out, uint32_t* vals_out,
               Count cnt, int64_t max_n, int bits, Ws& ws, cudaStream_t s) {
  if (max_n <= 0) return RTEC_OK;
  if (max_n <= 1024) {
    launch(k_sort_reg, 1, 1024, 0, s, keys_in, vals_in, keys_out, vals_out, cnt, bits);
    RTEC_LAUNCH_CHECK("k_sort_reg");
    return RTEC_OK;
  }
  if (max_n <= kSmallSort) {
    launch(k_sort_small, 1, 1024, 0, s, keys_in, vals_in, keys_out, vals_out, cnt);
    RTEC_LAUNCH_CHECK("k_sort_small");
    return RTEC_OK;
  }
  const int items = rx_items_for(max_n);
  const int64_t ntiles = (max_n + static_cast<int64_t>(kRxBlock) * items - 1) / (static_cast<int64_t>(kRxBlock) * items);
  uint64_t* ka = ws.alloc<uint64_t>(max_n);
  uint32_t* va = ws.alloc<uint32_t>(max_n);
  uint64_t* kb = ws.alloc<uint64_t>(max_n);
  uint32_t* vb = ws.alloc<uint32_t>(max_n);
  uint32_t* counts = ws.alloc<uint32_t>(kRxBins * ntiles);
  int64_t* offs = ws.alloc<int64_t>(kRxBins * ntiles);
  int64_t* bs = ws.alloc<int64_t>(scan_blocks_for(kRxBins * ntiles) + 2);
  RTEC_WS_CHECK(ws);
  int passes = (bits + 7) / 8;
  const uint64_t* ki = keys_in;
  const uint32_t* vi = vals_in;
  for (int p = 0; p < passes; ++p) {
    bool last = (p == passes - 1);
    uint64_t* ko = last ? keys_out : ((p & 1) ? kb : ka);
    uint32_t* vo = last ? vals_out : ((p & 1) ? vb : va);
    int shift = 8 * p;
    const unsigned grid = static_cast<unsigned>(ntiles);
    if (items == 1) launch(k_rx_hist<1>, grid, kRxBlock, 0, s, ki, cnt, shift, ntiles, counts);
    else if (items == 4) launch(k_rx_hist<4>, grid, kRxBlock, 0, s, ki, cnt, shift, ntiles, counts);
    else launch(k_rx_hist<kRxItems>, grid, kRxBlock, 0, s, ki, cnt, shift, ntiles, counts);
    RTEC_TRY(exclusive_scan_bs(U32At{counts}, Count{nullptr, kRxBins * ntiles}, kRxBins * ntiles,
                               StorePrefix{offs}, nullptr, bs, s));
    if (items == 1) launch(k_rx_scatter<1>, grid, kRxBlock, 0, s, ki, vi, ko, vo, cnt, shift, ntiles, offs);
    else if (items == 4) launch(k_rx_scatter<4>, grid, kRxBlock, 0, s, ki, vi, ko, vo, cnt, shift, ntiles, offs);
    else launch(k_rx_scatter<kRxItems>, grid, kRxBlock, 0, s, ki, vi, ko, vo, cnt, shift, ntiles, offs);
    RTEC_LAUNCH_CHECK("k_rx_scatter");
    ki = ko;
    vi = vo;
  }
  return RTEC_OK;
}

}  // namespace rtec
