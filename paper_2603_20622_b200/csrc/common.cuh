// common.cuh -- shared device/host helpers for librtec (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <string>
#include <utility>

#include "../../include/rtec.h"

namespace rtec {

constexpr int kWarp = 32;
constexpr int kMaxDevices = 64;

// SM count of the current device (148 on B200: 2 dies x 74), queried once per device;
// grids are sized in multiples of it
int sm_count();
#define kSMs (::rtec::sm_count())
// current device ordinal (0..kMaxDevices-1) for per-device host state
int cur_device();

// ---------------------------------------------------------------- errors
void set_error(const char* fmt, ...);
int cuda_status(cudaError_t e, const char* where);

#define RTEC_CUDA(call)                                   \
  do {                                                    \
    cudaError_t _e = (call);                              \
    if (_e != cudaSuccess) return ::rtec::cuda_status(_e, #call); \
  } while (0)

#define RTEC_LAUNCH_CHECK(name) RTEC_CUDA(cudaGetLastError())

#define RTEC_TRY(expr)              \
  do {                              \
    int _s = (expr);                \
    if (_s != RTEC_OK) return _s;   \
  } while (0)

// ---------------------------------------------------------------- kernel timing hook
// When enabled (rtec_prof_enable), launch sites bracket kernels with CUDA
// events on their stream; rtec_prof_report aggregates per kernel name.  Off by
// default (and never used inside CUDA-graph capture).
extern bool g_prof_on;
void prof_begin(const char* name, cudaStream_t s);
void prof_end(cudaStream_t s);
struct ProfScope {
  cudaStream_t s;
  bool on;
  ProfScope(const char* name, cudaStream_t st) : s(st), on(g_prof_on) {
    if (on) prof_begin(name, s);
  }
  ~ProfScope() {
    if (on) prof_end(s);
  }
};
#define RTEC_PROF(name, stream) ::rtec::ProfScope _rtec_prof_scope_##__LINE__(name, stream)

// ---------------------------------------------------------------- launches
// Programmatic dependent launch (PDL).  Every kernel begins with RTEC_PDL_ENTRY():
// griddepcontrol.wait blocks until the preceding grid in the stream has completed and
// its writes are visible (a no-op for a normal launch).  launch() issues every library
// kernel with programmatic stream serialization, so the next kernel of a dependent
// chain (and its CUDA-graph node, which keeps the programmatic edge) is launched as the
// predecessor's CTAs exit instead of after its completion is processed.  An explicit
// early griddepcontrol.launch_dependents (RTEC_PDL_TRIGGER=1 builds) makes the next
// grid's CTAs resident during the predecessor's last wave; measured slower on the
// two-stream passes (profiles/r02t_pdl_ab.md), so the default trigger is CTA exit.
// RTEC_PDL=0 turns the attribute off (plain stream order; A/B).
#ifndef RTEC_PDL_TRIGGER
#define RTEC_PDL_TRIGGER 0
#endif
#if RTEC_PDL_TRIGGER
#define RTEC_PDL_ENTRY() asm volatile("griddepcontrol.wait;\n\tgriddepcontrol.launch_dependents;" ::: "memory")
#else  // dependents launch as this grid's CTAs exit (no early residency)
#define RTEC_PDL_ENTRY() asm volatile("griddepcontrol.wait;" ::: "memory")
#endif
bool pdl_on();

template <typename... KArgs, typename... Args>
inline void launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_on() ? 1 : 0;
  (void)cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);  // errors: RTEC_LAUNCH_CHECK
}

// ---------------------------------------------------------------- side stream
// Library-owned side stream + fork / join events for independent passes inside one
// call (created once per process, on the device current at first use).  Fork and join
// are event records / waits, so a CUDA-graph capture of the caller's stream keeps them.
cudaStream_t side_stream();
cudaEvent_t side_fork();
cudaEvent_t side_join();

// ---------------------------------------------------------------- workspace
// Bump allocator over the caller's workspace; every chunk 256-B aligned.
struct Ws {
  uint8_t* base;
  size_t bytes;
  size_t off = 0;
  bool ok = true;
  Ws(void* p, size_t b) : base(static_cast<uint8_t*>(p)), bytes(b) {}
  template <typename T>
  T* alloc(int64_t count) {
    size_t need = (static_cast<size_t>(count > 0 ? count : 1) * sizeof(T) + 255) & ~size_t(255);
    if (off + need > bytes) {
      ok = false;
      return nullptr;
    }
    T* p = reinterpret_cast<T*>(base + off);
    off += need;
    return p;
  }
};

#define RTEC_WS_CHECK(ws)                                                                  \
  do {                                                                                     \
    if (!(ws).ok) {                                                                        \
      ::rtec::set_error("workspace too small (%zu bytes given, need more)", (ws).bytes);   \
      return RTEC_CONFIG_ERROR;                                                            \
    }                                                                                      \
  } while (0)

inline int grid_for(int64_t work, int block, int max_ctas = kSMs * 16) {
  int64_t g = (work + block - 1) / block;
  if (g < 1) g = 1;
  if (g > max_ctas) g = max_ctas;
  return static_cast<int>(g);
}

// ---------------------------------------------------------------- device helpers
__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ int warp_id() { return threadIdx.x >> 5; }

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// first index i in [lo, hi) with a[i] >= key (a ascending)
template <typename T, typename K>
__device__ __forceinline__ int64_t lower_bound_dev(const T* a, int64_t lo, int64_t hi, K key) {
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (a[mid] < key) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

__device__ __forceinline__ bool bm_test(const uint32_t* bm, int32_t v) {
  return (__ldg(bm + (v >> 5)) >> (v & 31)) & 1u;
}

// Warp-aggregated atomicOr of bit v (lanes sharing a word issue one atomic).
__device__ __forceinline__ void bm_set_warp(uint32_t* bm, int32_t v, bool active) {
  unsigned mask = __ballot_sync(0xffffffffu, active);
  if (!active) return;
  int word = v >> 5;
  unsigned peers = __match_any_sync(mask, word);
  uint32_t acc = __reduce_or_sync(peers, 1u << (v & 31));
  if ((__ffs(peers) - 1) == lane_id()) atomicOr(bm + word, acc);
}

__device__ __forceinline__ void atomic_min_i32(int32_t* p, int32_t v) { atomicMin(p, v); }

// Device status word: packed (position << 32 | code), all-ones = ok.  The
// smallest position wins (first offender in batch order); ties keep the
// smaller code.
constexpr uint64_t kErrOk = ~0ull;
__device__ __forceinline__ void report_error(uint64_t* err, int32_t code, int64_t pos) {
  unsigned long long packed = (static_cast<unsigned long long>(static_cast<uint32_t>(pos)) << 32) |
                              static_cast<uint32_t>(code);
  atomicMin(reinterpret_cast<unsigned long long*>(err), packed);
}
__device__ __forceinline__ bool err_set(const uint64_t* err) { return *((volatile const uint64_t*)err) != kErrOk; }

}  // namespace rtec
