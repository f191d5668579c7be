// gemm_tc.cu -- the dense per-layer update on tcgen05 tensor cores.
//
// Y[i] = act(A[i] · W^T) for the affected rows only (operators.py:180 ->
// linalg.matvec, linalg.py:22), fp32-accurate via 3xTF32:
//     a·w ≈ a_hi·w_hi + a_hi·w_lo + a_lo·w_hi     (hi = cvt.rna.tf32(x), lo = x - hi)
// all three products accumulated in one TMEM accumulator (128 lanes x N fp32).
//
// Data layout (no tensor maps needed): the producer of A (the aggregation
// kernel) writes rows straight into a tile-major, 128B-swizzled image
//     A[tile][kb][128 rows][32 fp32]   (16 KB per block, SW128 K-major atoms)
// and the weights are split + swizzled once per layer into
//     Bhi/Blo[kb][Npad rows][32 fp32].
// Each K-block is therefore one contiguous chunk fetched with a single 1-D
// bulk async copy (cp.async.bulk -> UBLKCP) completing on an mbarrier.
//
// Persistent CTAs (one per SM, 128 threads), 2-stage smem ring:
//   stage = A (raw -> lo in place, 16 KB) + A_hi (16 KB) + Bhi + Blo (Npad*128 B each)
// thread 0 issues the bulk copies one step ahead and the 12 MMAs per K-block
// (4 k-steps x 3 products, tcgen05.mma.cta_group::1.kind::tf32, M=128, N=Npad),
// tcgen05.commit frees the stage; all 128 threads split hi/lo and run the
// epilogue (tcgen05.ld 32x32b.x32 -> act -> scatter rows + DeltaLog capture).
#include "prims.cuh"
#include "gemm_tc.cuh"

namespace rtec {

constexpr int kTM = 128;                    // UMMA M (rows per tile)
constexpr int kTK = 32;                     // fp32 per K-block (one 128 B swizzle row)
constexpr int kABlockBytes = kTM * kTK * 4; // 16 KB

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\tLAB_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE;\n\tbra LAB_WAIT;\n\tDONE:\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void fence_barrier_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// SW128 K-major UMMA shared-memory descriptor (cute::UMMA::SmemDescriptor layout)
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);  // start address
  d |= static_cast<uint64_t>(1) << 16;                // LBO (unused for SW128 K-major)
  d |= static_cast<uint64_t>(1024 >> 4) << 32;        // SBO: 8 rows x 128 B
  d |= static_cast<uint64_t>(1) << 46;                // version 1 (sm_100)
  d |= static_cast<uint64_t>(2) << 61;                // SWIZZLE_128B
  return d;
}

__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

#define RTEC_TMEM_LD32(taddr, r)                                                                                  \
  asm volatile(                                                                                                   \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18," \
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                                               \
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),           \
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),     \
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),   \
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])    \
      : "r"(taddr))

// float offset of element (row r in tile, column c in K-block) in a SW128 block of 32-float rows
__host__ __device__ __forceinline__ int64_t sw128_off(int r, int c) {
  return static_cast<int64_t>(r) * 32 + ((((c >> 2) ^ (r & 7)) << 2) | (c & 3));
}



__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Warp-specialised persistent kernel (256 threads):
//   warp 0      producer: bulk-copies A / Bhi / Blo of each K-block into a ring of S stages
//   warp 1      MMA issuer: 12 tcgen05.mma per K-block into one of two TMEM accumulators
//   warps 2-3   splitters: A -> (hi, lo) in shared memory, fence.proxy.async, arrive
//   warps 4-7   epilogue: tcgen05.ld -> act -> global rows (+ DeltaLog), overlapping the
//               next tile's main loop thanks to the double-buffered accumulator
// mbarriers: full[s] (tx), split[s] (64 arrivals), empty[s] (tcgen05.commit),
//            tfull[2] (tcgen05.commit), tempty[2] (128 arrivals)
constexpr int kMaxStages = 4;

__global__ void __launch_bounds__(256, 1) k_gemm_tc(TcArgs g, int S) {
  extern __shared__ uint8_t smem_raw[];
  if (g.err && err_set(g.err)) return;
  const int64_t nrows = g.n_rows ? *g.n_rows : g.max_rows;
  const int64_t ntiles = (nrows + kTM - 1) / kTM;
  if (static_cast<int64_t>(blockIdx.x) >= ntiles) return;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t bbytes = static_cast<uint32_t>(g.npad) * kTK * 4;
  const uint32_t stage_bytes = 2 * kABlockBytes + 2 * bbytes;
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(base + S * stage_bytes);
  uint64_t* full = bars;
  uint64_t* split = bars + kMaxStages;
  uint64_t* empty = bars + 2 * kMaxStages;
  uint64_t* tfull = bars + 3 * kMaxStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  uint32_t ncols = 32;
  while (ncols < static_cast<uint32_t>(2 * g.npad)) ncols <<= 1;

  if (tid == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(full + i, 1);
      mbar_init(split + i, 64);
      mbar_init(empty + i, 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(tfull + i, 1);
      mbar_init(tempty + i, 128);
    }
    fence_barrier_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(ncols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t taddr = *tmem_slot;
  const int64_t my_tiles = (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x;
  const int64_t J = my_tiles * g.nkb;

  if (warp == 0) {
    if (lane == 0) {
      for (int64_t j = 0; j < J; ++j) {
        const int s = static_cast<int>(j % S);
        const int64_t u = j / S;
        if (u > 0) mbar_wait(empty + s, static_cast<uint32_t>((u - 1) & 1));
        const int64_t tile = blockIdx.x + (j / g.nkb) * gridDim.x;
        const int kb = static_cast<int>(j % g.nkb);
        uint8_t* st = base + s * stage_bytes;
        mbar_expect_tx(full + s, kABlockBytes + 2 * bbytes);
        bulk_g2s(st, g.A + (tile * g.nkb + kb) * (kABlockBytes / 4), kABlockBytes, full + s);
        bulk_g2s(st + 2 * kABlockBytes, g.Bhi + static_cast<int64_t>(kb) * g.npad * kTK, bbytes, full + s);
        bulk_g2s(st + 2 * kABlockBytes + bbytes, g.Blo + static_cast<int64_t>(kb) * g.npad * kTK, bbytes, full + s);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(g.npad >> 3) << 17) |
                             (static_cast<uint32_t>(kTM >> 4) << 24);
      for (int64_t t = 0; t < my_tiles; ++t) {
        const int b = static_cast<int>(t & 1);
        const int64_t ub = t >> 1;
        if (ub > 0) mbar_wait(tempty + b, static_cast<uint32_t>((ub - 1) & 1));
        tc_fence_after();
        const uint32_t acc_addr = taddr + static_cast<uint32_t>(b * g.npad);
        for (int kb = 0; kb < g.nkb; ++kb) {
          const int64_t j = t * g.nkb + kb;
          const int s = static_cast<int>(j % S);
          mbar_wait(split + s, static_cast<uint32_t>((j / S) & 1));
          tc_fence_after();
          const uint32_t a_lo = smem_u32(base + s * stage_bytes);
          const uint32_t a_hi = a_lo + kABlockBytes;
          const uint32_t b_hi = a_lo + 2 * kABlockBytes;
          const uint32_t b_lo = b_hi + bbytes;
#pragma unroll
          for (int k = 0; k < kTK / 8; ++k) {
            const uint32_t off = k * 32;
            const uint32_t acc = (kb > 0 || k > 0) ? 1u : 0u;
            mma_tf32(acc_addr, sw128_desc(a_hi + off), sw128_desc(b_hi + off), idesc, acc);
            mma_tf32(acc_addr, sw128_desc(a_hi + off), sw128_desc(b_lo + off), idesc, 1u);
            mma_tf32(acc_addr, sw128_desc(a_lo + off), sw128_desc(b_hi + off), idesc, 1u);
          }
          mma_commit(empty + s);  // smem stage reusable once these MMAs retire
        }
        mma_commit(tfull + b);    // accumulator b complete
      }
    }
  } else if (warp < 4) {
    const int st_id = tid - 64;  // 0..63
    for (int64_t j = 0; j < J; ++j) {
      const int s = static_cast<int>(j % S);
      mbar_wait(full + s, static_cast<uint32_t>((j / S) & 1));
      float4* raw = reinterpret_cast<float4*>(base + s * stage_bytes);
      float4* hi = reinterpret_cast<float4*>(base + s * stage_bytes + kABlockBytes);
#pragma unroll 4
      for (int q = 0; q < kABlockBytes / 16 / 64; ++q) {
        const int idx = st_id + 64 * q;
        float4 x = raw[idx];
        float4 h = make_float4(tf32_rna(x.x), tf32_rna(x.y), tf32_rna(x.z), tf32_rna(x.w));
        hi[idx] = h;
        raw[idx] = make_float4(x.x - h.x, x.y - h.y, x.z - h.z, x.w - h.w);
      }
      fence_proxy_async();
      mbar_arrive(split + s);
    }
  } else {
    // epilogue: thread owns accumulator row r = tid - 128 (TMEM lane r; warp w%4 -> lanes 32*(w%4))
    const int r = tid - 128;
    const uint32_t lane_base = static_cast<uint32_t>((warp & 3) * 32) << 16;
    for (int64_t t = 0; t < my_tiles; ++t) {
      const int b = static_cast<int>(t & 1);
      mbar_wait(tfull + b, static_cast<uint32_t>((t >> 1) & 1));
      tc_fence_after();
      const int64_t tile = blockIdx.x + t * gridDim.x;
      const int64_t i = tile * kTM + r;
      const bool valid = i < nrows;
      const int64_t dst = valid ? (g.y_rows ? static_cast<int64_t>(g.y_rows[i]) : i) : 0;
      for (int c0 = 0; c0 < g.npad; c0 += 32) {
        uint32_t rr[32];
        RTEC_TMEM_LD32(taddr + lane_base + static_cast<uint32_t>(b * g.npad + c0), rr);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (!valid) continue;
        float y[32];
#pragma unroll
        for (int q = 0; q < 32; ++q) {
          float v = __uint_as_float(rr[q]);
          y[q] = g.act == 1 ? fmaxf(v, 0.f) : v;
        }
        if (g.Yt) {  // chained GEMM input: SW128 tile image (zero padding beyond d_out)
          float* blk = g.Yt + ((tile * g.nkb_out + c0 / 32) * kTM) * kTK;
#pragma unroll
          for (int q = 0; q < 32; q += 4) {
            float4 v4 = make_float4(c0 + q < g.d_out ? y[q] : 0.f, c0 + q + 1 < g.d_out ? y[q + 1] : 0.f,
                                    c0 + q + 2 < g.d_out ? y[q + 2] : 0.f, c0 + q + 3 < g.d_out ? y[q + 3] : 0.f);
            *reinterpret_cast<float4*>(blk + sw128_off(r, q)) = v4;
          }
        } else {
          float* yrow = g.Y + dst * g.ldy;
          if ((g.d_out & 3) == 0 && c0 + 32 <= g.d_out && (g.ldy & 3) == 0) {
            float4* y4 = reinterpret_cast<float4*>(yrow + c0);
            if (g.log) {
              float4 old[8];
#pragma unroll
              for (int q = 0; q < 8; ++q) old[q] = y4[q];
              float4* l4 = reinterpret_cast<float4*>(g.log + i * g.d_out + c0);
#pragma unroll
              for (int q = 0; q < 8; ++q) l4[q] = old[q];
            }
#pragma unroll
            for (int q = 0; q < 8; ++q) y4[q] = make_float4(y[4 * q], y[4 * q + 1], y[4 * q + 2], y[4 * q + 3]);
          } else {
            for (int q = 0; q < 32 && c0 + q < g.d_out; ++q) {
              if (g.log) g.log[i * g.d_out + c0 + q] = yrow[c0 + q];
              yrow[c0 + q] = y[q];
            }
          }
        }
      }
      tc_fence_before();
      mbar_arrive(tempty + b);
    }
  }
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols));
  }
}

// W [d_out, d_in] -> Bhi/Blo [nkb][npad][32] swizzled, zero padded
__global__ void k_prep_b(const float* __restrict__ W, int d_in, int d_out, int nkb, int npad, float* Bhi, float* Blo) {
  int64_t total = static_cast<int64_t>(nkb) * npad * kTK;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    int kb = static_cast<int>(e / (static_cast<int64_t>(npad) * kTK));
    int rem = static_cast<int>(e % (static_cast<int64_t>(npad) * kTK));
    int n = rem / kTK, c = rem % kTK;
    int k = kb * kTK + c;
    float w = (n < d_out && k < d_in) ? W[static_cast<int64_t>(n) * d_in + k] : 0.f;
    float h = tf32_rna(w);
    float l = tf32_rna(w - h);
    int64_t o = static_cast<int64_t>(kb) * npad * kTK + sw128_off(n, c);
    Bhi[o] = h;
    Blo[o] = l;
  }
}

static int gemm_tc_stages(int npad) {
  size_t stage = 2 * kABlockBytes + 2 * static_cast<size_t>(npad) * kTK * 4;
  int S = static_cast<int>((227 * 1024 - 1024 - 256) / stage);
  return S < kMaxStages ? S : kMaxStages;
}
size_t gemm_tc_smem(int npad) {
  return gemm_tc_stages(npad) * (2 * kABlockBytes + 2 * static_cast<size_t>(npad) * kTK * 4) + 1024 + 256;
}

int gemm_tc_launch(const TcArgs& g, cudaStream_t s) {
  if (g.max_rows <= 0) return RTEC_OK;
  size_t smem = gemm_tc_smem(g.npad);
  static int configured = 0;
  if (!configured) {
    RTEC_CUDA(cudaFuncSetAttribute(k_gemm_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    configured = 1;
  }
  int64_t tiles = (g.max_rows + kTM - 1) / kTM;
  int grid = static_cast<int>(tiles < kSMs ? tiles : kSMs);
  RTEC_PROF("k_gemm_tc", s);
  k_gemm_tc<<<grid, 256, smem, s>>>(g, gemm_tc_stages(g.npad));
  RTEC_LAUNCH_CHECK("k_gemm_tc");
  return RTEC_OK;
}

}  // namespace rtec

using namespace rtec;

extern "C" {

// Split + swizzle fp32 weights W[d_out, d_in] into the tcgen05 3xTF32 operand
// image (Bhi, Blo each nkb*npad*32 floats; nkb = ceil(d_in/32), npad = d_out
// rounded up to 16).  Returns ShapeError if d_out > 256.
int rtec_gemm_prepare_weights(const float* W, int32_t d_in, int32_t d_out, float* Bhi, float* Blo,
                              rtec_stream_t stream) {
  if (d_out <= 0 || d_out > 256 || d_in <= 0) {
    set_error("tcgen05 update GEMM supports 1 <= d_out <= 256 (got %d)", d_out);
    return RTEC_SHAPE_ERROR;
  }
  int nkb = (d_in + kTK - 1) / kTK;
  int npad = (d_out + 15) / 16 * 16;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  k_prep_b<<<grid_for(static_cast<int64_t>(nkb) * npad * kTK, 256), 256, 0, s>>>(W, d_in, d_out, nkb, npad, Bhi, Blo);
  RTEC_LAUNCH_CHECK("k_prep_b");
  return RTEC_OK;
}

}  // extern "C"
