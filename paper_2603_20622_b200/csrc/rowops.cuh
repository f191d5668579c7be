// rowops.cuh -- warp-cooperative feature-row accumulators.
// A warp owns one destination row; lane l holds chunks c = l + 32*k (k < K)
// of VEC consecutive floats (VEC = 4 -> 128-bit loads when d % 4 == 0).
#pragma once
#include "common.cuh"

namespace rtec {

template <int VEC>
struct VecT;
template <>
struct VecT<4> {
  using T = float4;
};
template <>
struct VecT<2> {
  using T = float2;
};
template <>
struct VecT<1> {
  using T = float;
};

// L2 eviction-priority policy for streaming traffic (read/written once per
// batch): keeps it from displacing re-used gathered rows in L2.
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ float4 ld_stream_f4(const float4* a, uint64_t pol) {
  float4 v;
  asm volatile("ld.global.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ void st_stream_f4(float4* a, float4 v, uint64_t pol) {
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.v4.f32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(a), "f"(v.x),
               "f"(v.y), "f"(v.z), "f"(v.w), "l"(pol)
               : "memory");
}
__device__ __forceinline__ int32_t ld_stream_i32(const int32_t* a, uint64_t pol) {
  int32_t v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(v) : "l"(a), "l"(pol));
  return v;
}

// 16-byte global -> shared async copy with an L2 eviction-priority hint; completion
// (cp_async_wait_all) makes it visible to the issuing thread
__device__ __forceinline__ void cp_async16_hint(void* smem, const void* gmem, uint64_t pol) {
  const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

template <int VEC, int K>
struct RowAcc {
  float v[K][VEC];
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int k = 0; k < K; ++k)
#pragma unroll
      for (int j = 0; j < VEC; ++j) v[k][j] = 0.f;
  }
  __device__ __forceinline__ static bool has(int k, int d) { return ((lane_id() + 32 * k) * VEC) < d; }
  __device__ __forceinline__ static void load(const float* __restrict__ row, int d, float (&r)[K][VEC]) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      int c = lane_id() + 32 * k;
      if (c * VEC < d) {
        if constexpr (VEC == 4) {
          float4 x = __ldg(reinterpret_cast<const float4*>(row) + c);
          r[k][0] = x.x; r[k][1] = x.y; r[k][2] = x.z; r[k][3] = x.w;
        } else if constexpr (VEC == 2) {
          float2 x = __ldg(reinterpret_cast<const float2*>(row) + c);
          r[k][0] = x.x; r[k][1] = x.y;
        } else {
          r[k][0] = __ldg(row + c);
        }
      } else {
#pragma unroll
        for (int j = 0; j < VEC; ++j) r[k][j] = 0.f;
      }
    }
  }
  // row -> this lane's chunks of a shared-memory stage, asynchronously (VEC == 4): keeps a
  // prefetched row out of registers across a gather loop; read back with from_stage
  __device__ __forceinline__ static void stage_async(float* stage, const float* row, int d, uint64_t pol) {
    static_assert(VEC == 4, "stage_async needs 16-byte chunks");
#pragma unroll
    for (int k = 0; k < K; ++k) {
      int c = lane_id() + 32 * k;
      if (c * VEC < d) cp_async16_hint(stage + c * VEC, row + c * VEC, pol);
    }
  }
  // row already resident in shared memory (e.g. completed bulk copy)
  __device__ __forceinline__ static void from_stage_sync(const float* stage, int d, float (&r)[K][VEC]) {
    static_assert(VEC == 4, "16-byte chunks");
#pragma unroll
    for (int k = 0; k < K; ++k) {
      int c = lane_id() + 32 * k;
      if (c * VEC < d) {
        float4 x = *reinterpret_cast<const float4*>(stage + c * VEC);
        r[k][0] = x.x; r[k][1] = x.y; r[k][2] = x.z; r[k][3] = x.w;
      } else {
        r[k][0] = r[k][1] = r[k][2] = r[k][3] = 0.f;
      }
    }
  }
  __device__ __forceinline__ static void from_stage(const float* stage, int d, float (&r)[K][VEC]) {
    cp_async_wait_all();
#pragma unroll
    for (int k = 0; k < K; ++k) {
      int c = lane_id() + 32 * k;
      if (c * VEC < d) {
        float4 x = *reinterpret_cast<const float4*>(stage + c * VEC);
        r[k][0] = x.x; r[k][1] = x.y; r[k][2] = x.z; r[k][3] = x.w;
      } else {
        r[k][0] = r[k][1] = r[k][2] = r[k][3] = 0.f;
      }
    }
  }
  // plain (non-__ldg) load for rows written earlier in the same kernel
  __device__ __forceinline__ static void load_rw(const float* row, int d, float (&r)[K][VEC]) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      int c = lane_id() + 32 * k;
      if (c * VEC < d) {
        if constexpr (VEC == 4) {
          float4 x = reinterpret_cast<const float4*>(row)[c];
          r[k][0] = x.x; r[k][1] = x.y; r[k][2] = x.z; r[k][3] = x.w;
        } else if constexpr (VEC == 2) {
          float2 x = reinterpret_cast<const float2*>(row)[c];
          r[k][0] = x.x; r[k][1] = x.y;
        } else {
          r[k][0] = row[c];
        }
      } else {
#pragma unroll
        for (int j = 0; j < VEC; ++j) r[k][j] = 0.f;
      }
    }
  }
  // streaming (evict-first) row load / store, VEC == 4 only; falls back otherwise
  __device__ __forceinline__ static void load_stream(const float* row, int d, float (&r)[K][VEC], uint64_t pol) {
    if constexpr (VEC == 4) {
#pragma unroll
      for (int k = 0; k < K; ++k) {
        int c = lane_id() + 32 * k;
        if (c * VEC < d) {
          float4 x = ld_stream_f4(reinterpret_cast<const float4*>(row) + c, pol);
          r[k][0] = x.x; r[k][1] = x.y; r[k][2] = x.z; r[k][3] = x.w;
        } else {
          r[k][0] = r[k][1] = r[k][2] = r[k][3] = 0.f;
        }
      }
    } else {
      load_rw(row, d, r);
    }
  }
  __device__ __forceinline__ void store_stream(float* row, int d, uint64_t pol) const {
    if constexpr (VEC == 4) {
#pragma unroll
      for (int k = 0; k < K; ++k) {
        int c = lane_id() + 32 * k;
        if (c * VEC < d)
          st_stream_f4(reinterpret_cast<float4*>(row) + c, make_float4(v[k][0], v[k][1], v[k][2], v[k][3]), pol);
      }
    } else {
      store(row, d);
    }
  }
  __device__ __forceinline__ void fma(const float (&r)[K][VEC], float s) {
#pragma unroll
    for (int k = 0; k < K; ++k)
#pragma unroll
      for (int j = 0; j < VEC; ++j) v[k][j] = fmaf(s, r[k][j], v[k][j]);
  }
  __device__ __forceinline__ void add(const float (&r)[K][VEC]) {
#pragma unroll
    for (int k = 0; k < K; ++k)
#pragma unroll
      for (int j = 0; j < VEC; ++j) v[k][j] += r[k][j];
  }
  __device__ __forceinline__ void store(float* row, int d) const {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      int c = lane_id() + 32 * k;
      if (c * VEC < d) {
        if constexpr (VEC == 4) {
          reinterpret_cast<float4*>(row)[c] = make_float4(v[k][0], v[k][1], v[k][2], v[k][3]);
        } else if constexpr (VEC == 2) {
          reinterpret_cast<float2*>(row)[c] = make_float2(v[k][0], v[k][1]);
        } else {
          row[c] = v[k][0];
        }
      }
    }
  }
  // Columns [col0, col0 + w) of row i into the tcgen05 A-operand image:
  // [tile][kb][128][32] with the SW128 16-byte-chunk XOR swizzle.  The slice
  // ending at d_total also writes the zero padding d_total .. nkb*32.
  __device__ __forceinline__ void store_tiled(float* A, int64_t i, int col0, int w, int d_total, int nkb) const {
    const int64_t tile = i >> 7;
    const int r = static_cast<int>(i & 127);
    float* tbase = A + tile * static_cast<int64_t>(nkb) * 4096;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      int cl = (lane_id() + 32 * k) * VEC;
      if (cl < w) {
        int c = col0 + cl;
        int kb = c >> 5, cc = c & 31;
        float* blk = tbase + kb * 4096 + r * 32 + ((((cc >> 2) ^ (r & 7)) << 2) | (cc & 3));
        if constexpr (VEC == 4) {
          st_stream_f4(reinterpret_cast<float4*>(blk), make_float4(v[k][0], v[k][1], v[k][2], v[k][3]),
                       l2_evict_first_policy());
        } else if constexpr (VEC == 2) {
          *reinterpret_cast<float2*>(blk) = make_float2(v[k][0], v[k][1]);
        } else {
          *blk = v[k][0];
        }
      }
    }
    if (col0 + w >= d_total) {
      for (int c = d_total + lane_id(); c < nkb * 32; c += 32) {  // zero padding
        int kb = c >> 5, cc = c & 31;
        tbase[kb * 4096 + r * 32 + ((((cc >> 2) ^ (r & 7)) << 2) | (cc & 3))] = 0.f;
      }
    }
  }
};

// dispatch for a feature slice of width w <= 64: float2 lanes when even
#define RTEC_SLICE_DISPATCH(w, ...)                                                 \
  [&]() -> bool {                                                                  \
    if ((w) <= 64 && ((w) % 2) == 0) { constexpr int VEC = 2, K = 1; __VA_ARGS__; return true; } \
    if ((w) <= 64) { constexpr int VEC = 1, K = 2; __VA_ARGS__; return true; }      \
    return false;                                                                  \
  }()

// dispatch (VEC, K) from the row width; returns false if unsupported
#define RTEC_ROW_DISPATCH(d, ...)                                         \
  [&]() -> bool {                                                         \
    if ((d) % 4 == 0) {                                                   \
      int _k = ((d) / 4 + 31) / 32;                                       \
      if (_k <= 1) { constexpr int VEC = 4, K = 1; __VA_ARGS__; return true; } \
      if (_k <= 2) { constexpr int VEC = 4, K = 2; __VA_ARGS__; return true; } \
      if (_k <= 4) { constexpr int VEC = 4, K = 4; __VA_ARGS__; return true; } \
      if (_k <= 5) { constexpr int VEC = 4, K = 5; __VA_ARGS__; return true; } \
      return false;                                                       \
    }                                                                     \
    int _k = ((d) + 31) / 32;                                             \
    if (_k <= 1) { constexpr int VEC = 1, K = 1; __VA_ARGS__; return true; }   \
    if (_k <= 4) { constexpr int VEC = 1, K = 4; __VA_ARGS__; return true; }   \
    if (_k <= 8) { constexpr int VEC = 1, K = 8; __VA_ARGS__; return true; }   \
    if (_k <= 20) { constexpr int VEC = 1, K = 20; __VA_ARGS__; return true; } \
    return false;                                                         \
  }()

}  // namespace rtec
