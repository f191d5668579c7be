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
// Persistent CTAs (one per SM, 16 warps, see k_gemm_tc): an A ring (raw -> lo
// in place + hi, 32 KB per K-block) and a B ring of (K-block, N-half) stages,
// one producer lane issuing the bulk copies, one MMA lane issuing 12
// tcgen05.mma per (K-block, N-half) into a double-buffered TMEM accumulator,
// six splitter warps and eight epilogue warps (tcgen05.ld -> act -> rows
// staged through swizzled shared memory -> float4 stores; the DeltaLog copy of
// the old rows runs before the accumulator is ready).
#include "prims.cuh"
#include "gemm_tc.cuh"
#include "async.cuh"

#include <stdlib.h>

namespace rtec {

constexpr int kTM = 128;                    // UMMA M (rows per tile)
constexpr int kTK = 32;                     // fp32 per K-block (one 128 B swizzle row)
constexpr int kABlockBytes = kTM * kTK * 4; // 16 KB

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



__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.b32 %0, 1, 0, P;\n\t}" : "=r"(pred));
  return pred != 0;
}


// Warp-specialised persistent kernel (512 threads), separate operand rings:
//   warp 0      A producer: bulk-copies each A K-block (16 KB) into the A ring
//   warp 2      B producer: each (K-block, N-half) of Bhi/Blo into the B ring
//   warp 1      MMA issuer: per (K-block, N-half) 12 tcgen05.mma into one of two TMEM
//               accumulators (columns [half0, npad) of buffer t&1)
//   warps 3-7   splitters: A -> (hi, lo) in shared memory, fence.proxy.async, arrive
//   warps 8-15  epilogue: tcgen05.ld -> act -> global rows (+ DeltaLog), overlapping the
//               next tile's main loop thanks to the double-buffered accumulator
// Splitting B by N-halves keeps the B stage at 32 KB for N = 256, so the rings
// are 3 A stages + 4 B stages deep instead of 2 monolithic 96 KB stages.
// mbarriers: a_full (tx), a_split (160 arrivals), a_empty (tcgen05.commit),
//            b_full (tx), b_empty (commit), tfull[2] (commit), tempty[2] (256 arrivals)
constexpr int kMaxA = 6, kMaxB = 8;
constexpr int kSplitThreads = 160;
constexpr int kEpiBytes = 8 * 32 * 32 * 4;              // 8 epilogue warps x 32 rows x 32 cols

struct TcShape {
  int probe;        // timing probes (-DRTEC_GEMM_PROBES builds only; wrong results): 1 no B refills,
                    // 2 no A refills, 4 no split, 8 no epilogue, 16 no MMAs
  int SA, SB;       // ring depths
  int nh;           // N halves (1 or 2)
  int h0;           // width of half 0 (multiple of 16); half 1 = npad - h0
  uint32_t bstage;  // bytes of one B stage (hi + lo of the wider half)
  uint32_t oldb;    // fused deltas: per-warp double-buffered old-row staging (bytes, all warps)
};

constexpr int kOldBytes = 8 * 2 * 32 * 32 * 4;  // 8 epilogue warps x 2 buffers x 32 rows x 32 cols

// RTEC_GEMM_NWIDE env: 1 one N <= 256 MMA per (K-step, product) when the shared memory leaves
// a double-buffered 64 KB B ring (no fused deltas), 0 (default) two N-halves.  Measured on
// c2-gcn layer 2 (profiles/r02k_gemm_wide.md): tensor pipe 30 -> 40 % active but 1.77 ->
// 1.83 ms -- the shallower B ring (2 x 64 KB instead of 4 x 32 KB) costs more than the halved
// MMA issues / A re-reads save
static bool gemm_n_wide() {
  static int w = -1;
  if (w < 0) {
    const char* e = getenv("RTEC_GEMM_NWIDE");
    w = e ? atoi(e) : 0;
  }
  return w != 0;
}

// RTEC_GEMM_SA env: A-ring stages (A/B; 0: the defaults below)
static int gemm_a_stages() {
  static int a = -1;
  if (a < 0) {
    const char* e = getenv("RTEC_GEMM_SA");
    a = e ? atoi(e) : 0;
  }
  return a;
}

static TcShape tc_shape(int npad, bool fused) {
  TcShape sh;
  sh.probe = 0;
#ifdef RTEC_GEMM_PROBES  // bottleneck probes for tools/gemm_probe.sh (build with -DRTEC_GEMM_PROBES)
  {
    const char* e = getenv("RTEC_GEMM_PROBE");
    sh.probe = e ? atoi(e) : 0;
  }
#endif
  // N > 128 runs in two N-halves (32 KB B stages, deep rings) unless the whole N fits one
  // MMA with a double-buffered B ring: half the MMA issues and ~25 % fewer shared-memory
  // operand reads (A is read once per K-step instead of once per N-half)
  const bool wide = gemm_n_wide() && !fused && npad > 128;
  sh.nh = (npad > 128 && !wide) ? 2 : 1;
  sh.h0 = sh.nh == 2 ? ((npad / 2 + 15) / 16) * 16 : npad;
  sh.bstage = 2u * static_cast<uint32_t>(sh.h0) * kTK * 4;
  sh.oldb = fused ? kOldBytes : 0;
  const int budget = 227 * 1024 - 1024 - 512 - kEpiBytes - static_cast<int>(sh.oldb);
  sh.SA = (fused || wide) ? 2 : 3;  // measured: 2..4 A stages perform alike; the B ring gets the rest
  const int sa_env = gemm_a_stages();
  if (sa_env >= 2 && sa_env <= kMaxA) sh.SA = sa_env;
  sh.SB = (budget - sh.SA * 2 * kABlockBytes) / static_cast<int>(sh.bstage);
  if (sh.SB > kMaxB) sh.SB = kMaxB;
  if (sh.SB < 2) {  // keep a double-buffered B ring
    sh.SB = 2;
    sh.SA = (budget - sh.SB * static_cast<int>(sh.bstage)) / (2 * kABlockBytes);
  }
  return sh;
}

__global__ void __launch_bounds__(512, 1) k_gemm_tc(TcArgs g, TcShape sh) {
  RTEC_PDL_ENTRY();
  extern __shared__ uint8_t smem_raw[];
  if (g.err && err_set(g.err)) return;
  const int64_t nrows = g.n_rows ? *g.n_rows : g.max_rows;
  const int64_t ntiles = (nrows + kTM - 1) / kTM;
  if (static_cast<int64_t>(blockIdx.x) >= ntiles) return;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* aring = base;                                      // SA x (lo 16 KB | hi 16 KB)
  uint8_t* bring = base + sh.SA * 2 * kABlockBytes;           // SB x (hi | lo)
  float* epi = reinterpret_cast<float*>(bring + sh.SB * sh.bstage);   // epilogue transpose staging
  float* olds = epi + kEpiBytes / 4;                                    // fused deltas: old rows
  uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(olds) + sh.oldb);
  uint64_t* a_full = bars;
  uint64_t* a_split = a_full + kMaxA;
  uint64_t* a_empty = a_split + kMaxA;
  uint64_t* b_full = a_empty + kMaxA;
  uint64_t* b_empty = b_full + kMaxB;
  uint64_t* tfull = b_empty + kMaxB;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  uint32_t ncols = 32;
  while (ncols < static_cast<uint32_t>(2 * g.npad)) ncols <<= 1;

  if (tid == 0) {
    for (int i = 0; i < sh.SA; ++i) {
      mbar_init(a_full + i, 1);
      mbar_init(a_split + i, kSplitThreads);
      mbar_init(a_empty + i, 1);
    }
    for (int i = 0; i < sh.SB; ++i) {
      mbar_init(b_full + i, 1);
      mbar_init(b_empty + i, 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(tfull + i, 1);
      mbar_init(tempty + i, 256);
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
  const int64_t J = my_tiles * g.nkb;  // A stages consumed by this CTA

  if (warp == 0) {
    if (lane == 0) {  // A producer: one 16 KB K-block of the tile image per stage
      for (int64_t j = 0; j < J; ++j) {
        const int sa = static_cast<int>(j % sh.SA);
        if (j >= sh.SA) mbar_wait(a_empty + sa, static_cast<uint32_t>(((j / sh.SA) - 1) & 1));
        const int64_t tile = blockIdx.x + (j / g.nkb) * gridDim.x;
        const int kb = static_cast<int>(j % g.nkb);
        if ((sh.probe & 2) && j >= g.nkb) { mbar_arrive(a_full + sa); continue; }
        mbar_expect_tx(a_full + sa, kABlockBytes);
        bulk_g2s(aring + sa * 2 * kABlockBytes, g.A + (tile * g.nkb + kb) * (kABlockBytes / 4), kABlockBytes,
                 a_full + sa);
      }
    }
  } else if (warp == 2) {
    if (lane == 0) {  // B producer (its own lane, so a full B ring never stalls the A loads)
      const int64_t JB = J * sh.nh;
      for (int64_t jb = 0; jb < JB; ++jb) {
        const int kb = static_cast<int>((jb / sh.nh) % g.nkb);
        const int h = static_cast<int>(jb % sh.nh);
        const int sb = static_cast<int>(jb % sh.SB);
        if (jb >= sh.SB) mbar_wait(b_empty + sb, static_cast<uint32_t>(((jb / sh.SB) - 1) & 1));
        const int n0 = h == 0 ? 0 : sh.h0;
        const int nw = h == 0 ? sh.h0 : g.npad - sh.h0;
        const uint32_t hb = static_cast<uint32_t>(nw) * kTK * 4;
        uint8_t* st = bring + sb * sh.bstage;
        const int64_t off = (static_cast<int64_t>(kb) * g.npad + n0) * kTK;
        if ((sh.probe & 1) && jb >= static_cast<int64_t>(g.nkb) * sh.nh) { mbar_arrive(b_full + sb); continue; }
        mbar_expect_tx(b_full + sb, 2 * hb);
        bulk_g2s(st, g.Bhi + off, hb, b_full + sb);
        bulk_g2s(st + sh.bstage / 2, g.Blo + off, hb, b_full + sb);
      }
    }
  } else if (warp == 1) {
    // MMA warp: all lanes walk the (uniform) schedule so descriptors live in uniform
    // registers; one elected lane issues each tcgen05.mma / commit
    int64_t j = 0, jb = 0;
    for (int64_t t = 0; t < my_tiles; ++t) {
      const int b = static_cast<int>(t & 1);
      const int64_t ub = t >> 1;
      if (ub > 0) mbar_wait(tempty + b, static_cast<uint32_t>((ub - 1) & 1));
      tc_fence_after();
      for (int kb = 0; kb < g.nkb; ++kb, ++j) {
        const int sa = static_cast<int>(j % sh.SA);
        mbar_wait(a_split + sa, static_cast<uint32_t>((j / sh.SA) & 1));
        tc_fence_after();
        const uint64_t dalo = sw128_desc(smem_u32(aring + sa * 2 * kABlockBytes));
        const uint64_t dahi = dalo + (kABlockBytes >> 4);
        for (int h = 0; h < sh.nh; ++h, ++jb) {
          const int sb = static_cast<int>(jb % sh.SB);
          mbar_wait(b_full + sb, static_cast<uint32_t>((jb / sh.SB) & 1));
          tc_fence_after();
          const int n0 = h == 0 ? 0 : sh.h0;
          const int nw = h == 0 ? sh.h0 : g.npad - sh.h0;
          const uint64_t dbhi = sw128_desc(smem_u32(bring + sb * sh.bstage));
          const uint64_t dblo = dbhi + ((sh.bstage / 2) >> 4);
          const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(nw >> 3) << 17) |
                                 (static_cast<uint32_t>(kTM >> 4) << 24);
          const uint32_t acc_addr = taddr + static_cast<uint32_t>(b * g.npad + n0);
          if (elect_one()) {
#pragma unroll
            for (int k = 0; k < ((sh.probe & 16) ? 0 : kTK / 8); ++k) {
              const uint64_t off = static_cast<uint64_t>(k * 32) >> 4;  // +32 B along K per k-step
              const uint32_t acc = (kb > 0 || k > 0) ? 1u : 0u;
              mma_tf32(acc_addr, dahi + off, dbhi + off, idesc, acc);
              mma_tf32(acc_addr, dahi + off, dblo + off, idesc, 1u);
              mma_tf32(acc_addr, dalo + off, dbhi + off, idesc, 1u);
            }
            mma_commit(b_empty + sb);  // B stage reusable once these MMAs retire
          }
          __syncwarp();
        }
        if (elect_one()) mma_commit(a_empty + sa);
        __syncwarp();
      }
      if (elect_one()) mma_commit(tfull + b);  // accumulator b complete
      __syncwarp();
    }
  } else if (warp < 8) {
    const int st_id = tid - 96;  // warps 3-7: 0..159
    for (int64_t j = 0; j < J; ++j) {
      const int sa = static_cast<int>(j % sh.SA);
      mbar_wait(a_full + sa, static_cast<uint32_t>((j / sh.SA) & 1));
      float4* raw = reinterpret_cast<float4*>(aring + sa * 2 * kABlockBytes);
      float4* hi = reinterpret_cast<float4*>(aring + sa * 2 * kABlockBytes + kABlockBytes);
      for (int idx = st_id; idx < ((sh.probe & 4) && j >= g.nkb ? 0 : kABlockBytes / 16); idx += kSplitThreads) {
        float4 x = raw[idx];
        float4 hv = make_float4(tf32_rna(x.x), tf32_rna(x.y), tf32_rna(x.z), tf32_rna(x.w));
        hi[idx] = hv;
        // lo rounded to tf32 too (the MMA would truncate it): half an ulp of the residual
        raw[idx] = make_float4(tf32_rna(x.x - hv.x), tf32_rna(x.y - hv.y), tf32_rna(x.z - hv.z),
                               tf32_rna(x.w - hv.w));
      }
      fence_proxy_async();
      mbar_arrive(a_split + sa);
    }
  } else {
    // epilogue (warps 8-15): warp w reads TMEM lanes 32*(w%4).. (its 32 rows) and the
    // column half (w-8)/4 of the accumulator.  Row-major outputs are staged through
    // shared memory (16-byte chunks XOR-swizzled by row) so each float4 store
    // instruction writes 4 rows x 128 contiguous bytes.
    const int wq = warp & 3;
    const int half = (warp - 8) >> 2;
    const int r = wq * 32 + lane;
    const uint32_t lane_base = static_cast<uint32_t>(wq * 32) << 16;
    float* stg = epi + (warp - 8) * 32 * 32;
    const int nchunk = g.npad / 32 + (g.npad % 32 ? 1 : 0);
    const int cbeg = half == 0 ? 0 : (nchunk / 2), cend = half == 0 ? (nchunk / 2) : nchunk;
    for (int64_t t = 0; t < my_tiles; ++t) {
      const int b = static_cast<int>(t & 1);
      const int64_t tile = blockIdx.x + t * gridDim.x;
      const int64_t i = tile * kTM + r;
      const bool valid = i < nrows;
      const int64_t dst =
          valid ? (g.y_rows ? static_cast<int64_t>(g.y_rows[i]) : i) / (g.ydiv > 1 ? g.ydiv : 1) : -1;
      const int64_t row0 = tile * kTM + wq * 32;  // first row of this warp
      if (g.log && !g.Yt) {
        // DeltaLog capture of this tile's rows (this warp's column half) does not
        // depend on the MMA: copy the pre-batch rows while the tile accumulates
        const int c_lo = cbeg * 32, c_hi = min(cend * 32, g.d_out);
        for (int q0 = 0; q0 < 32; q0 += 4) {
          float v[4][4];
          int64_t dq[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            dq[u] = __shfl_sync(0xffffffffu, dst, q0 + u);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const int c = c_lo + lane + 32 * k;
              v[u][k] = (dq[u] >= 0 && c < c_hi) ? __ldcg(g.Y + dq[u] * g.ldy + c) : 0.f;
            }
          }
#pragma unroll
          for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const int c = c_lo + lane + 32 * k;
              if (dq[u] >= 0 && c < c_hi) __stcs(g.log + (row0 + q0 + u) * g.d_out + c, v[u][k]);
            }
        }
      }
      // fused deltas: pre-batch rows of this warp's 32 rows, one 32-column chunk at a
      // time, copied asynchronously into shared memory one chunk ahead
      const bool fused = g.delta_next != nullptr && !g.Yt;
      float c_new = 1.f, c_old = 1.f;
      float* oldw = olds + (warp - 8) * 2 * 32 * 32;
      const int sub = lane >> 3, ch = lane & 7;  // 4 rows per instruction, 8 lanes x 16 B per row
      auto prefetch_old = [&](int cc) {
        float* ob = oldw + ((cc - cbeg) & 1) * 32 * 32;
        const int col = cc * 32 + ch * 4;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int q = 4 * u + sub;
          const int64_t dq = __shfl_sync(0xffffffffu, dst, q);
          if (dq >= 0 && col + 4 <= g.d_out) cp_async16(ob + q * 32 + ch * 4, g.Y + dq * g.ldy + col);
        }
        cp_async_commit();
      };
      if (fused) {
        if (dst >= 0) {
          const int32_t dn = g.deg_new[dst], dp = g.deg_old[dst];
          c_new = dn > 0 ? (g.coeff_gcn ? 1.0f / sqrtf(static_cast<float>(dn) + g.deg_off) : 1.f) : 0.f;
          c_old = dp > 0 ? (g.coeff_gcn ? 1.0f / sqrtf(static_cast<float>(dp) + g.deg_off) : 1.f) : 0.f;
        }
        if (cbeg < cend) prefetch_old(cbeg);  // independent of the MMA: overlaps the wait below
      }
      mbar_wait(tfull + b, static_cast<uint32_t>((t >> 1) & 1));
      tc_fence_after();
      for (int cc = cbeg; cc < ((sh.probe & 8) ? cbeg : cend); ++cc) {
        const int c0 = cc * 32;
        if (fused) {
          if (cc + 1 < cend) {
            prefetch_old(cc + 1);
            cp_async_wait<1>();
          } else {
            cp_async_wait<0>();
          }
        }
        uint32_t rr[32];
        RTEC_TMEM_LD32(taddr + lane_base + static_cast<uint32_t>(b * g.npad + c0), rr);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        float y[32];
        bool finite = true;
#pragma unroll
        for (int q = 0; q < 32; ++q) {
          float v = __uint_as_float(rr[q]);
          finite = finite && isfinite(v);  // padding columns accumulate zeros
          y[q] = g.act == 1 ? fmaxf(v, 0.f) : v;
        }
        if (!finite && valid && g.nerr)
          report_error(g.nerr, RTEC_NUMERIC_ERROR, g.y_rows ? static_cast<int64_t>(g.y_rows[i]) : i);
        if (g.Yt) {  // chained GEMM input: SW128 tile image (zero padding beyond d_out)
          if (!valid) continue;
          float* blk = g.Yt + ((tile * g.nkb_out + c0 / 32) * kTM) * kTK;
#pragma unroll
          for (int q = 0; q < 32; q += 4) {
            float4 v4 = make_float4(c0 + q < g.d_out ? y[q] : 0.f, c0 + q + 1 < g.d_out ? y[q + 1] : 0.f,
                                    c0 + q + 2 < g.d_out ? y[q + 2] : 0.f, c0 + q + 3 < g.d_out ? y[q + 3] : 0.f);
            *reinterpret_cast<float4*>(blk + sw128_off(r, q)) = v4;
          }
          continue;
        }
        // stage: row `lane`, chunk c at 16-byte slot (c ^ (lane & 7))
#pragma unroll
        for (int c = 0; c < 8; ++c)
          *reinterpret_cast<float4*>(stg + lane * 32 + ((c ^ (lane & 7)) << 2)) =
              make_float4(y[4 * c], y[4 * c + 1], y[4 * c + 2], y[4 * c + 3]);
        __syncwarp();
        const int col = c0 + ch * 4;
        if (fused) {
          const float* ob = oldw + ((cc - cbeg) & 1) * 32 * 32;
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int q = 4 * u + sub;
            const int64_t dq = __shfl_sync(0xffffffffu, dst, q);
            const float cn = __shfl_sync(0xffffffffu, c_new, q);
            const float co = __shfl_sync(0xffffffffu, c_old, q);
            const float4 v4 = *reinterpret_cast<const float4*>(stg + q * 32 + ((ch ^ (q & 7)) << 2));
            if (dq < 0 || col + 4 > g.d_out) continue;
            const float4 o4 = *reinterpret_cast<const float4*>(ob + q * 32 + ch * 4);
            *reinterpret_cast<float4*>(g.Y + dq * g.ldy + col) = v4;
            __stcg(reinterpret_cast<float4*>(g.delta_next + dq * g.d_out + col),
                   make_float4(cn * v4.x - co * o4.x, cn * v4.y - co * o4.y, cn * v4.z - co * o4.z,
                               cn * v4.w - co * o4.w));
          }
          __syncwarp();
          continue;
        }
        const bool full4 = (g.d_out & 3) == 0 && (g.ldy & 3) == 0;
#pragma unroll
        for (int q0 = 0; q0 < 32; q0 += 4) {
          const int q = q0 + sub;
          const int64_t dq = __shfl_sync(0xffffffffu, dst, q);
          const float4 v4 = *reinterpret_cast<const float4*>(stg + q * 32 + ((ch ^ (q & 7)) << 2));
          if (dq < 0) continue;
          float* yp = g.Y + dq * g.ldy + col;
          if (full4 && col + 4 <= g.d_out) {
            *reinterpret_cast<float4*>(yp) = v4;
          } else {
            const float e[4] = {v4.x, v4.y, v4.z, v4.w};
            for (int k = 0; k < 4 && col + k < g.d_out; ++k) yp[k] = e[k];
          }
        }
        __syncwarp();
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
  RTEC_PDL_ENTRY();
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

// gathered rows -> SW128 A image: one warp per row, lane = 4 consecutive columns (scalar
// loads: rows of odd 16-byte alignment such as d = 602 are read coalesced), one float4
// store per lane into its swizzled 16-byte slot
__global__ void k_pack_rows(const float* __restrict__ X, int64_t ld, int d, const int32_t* __restrict__ rows,
                            const int64_t* n_rows, int64_t n_all, float* __restrict__ img, int nkb, const uint64_t* err) {
  RTEC_PDL_ENTRY();
  if (err && err_set(err)) return;
  const int64_t nr = n_rows ? *n_rows : n_all;
  int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int kw = nkb * kTK;
  for (int64_t i = warp; i < nr; i += nw) {
    const int64_t src = rows ? static_cast<int64_t>(rows[i]) : i;
    const float* xr = X + src * ld;
    const int64_t tile = i / kTM;
    const int r = static_cast<int>(i % kTM);
    for (int c = lane * 4; c < kw; c += 128) {
      float4 v;
      v.x = c < d ? __ldg(xr + c) : 0.f;
      v.y = c + 1 < d ? __ldg(xr + c + 1) : 0.f;
      v.z = c + 2 < d ? __ldg(xr + c + 2) : 0.f;
      v.w = c + 3 < d ? __ldg(xr + c + 3) : 0.f;
      const int kb = c / kTK, cc = c % kTK;
      *reinterpret_cast<float4*>(img + ((tile * nkb + kb) * kTM) * kTK + sw128_off(r, cc)) = v;
    }
  }
}

int gemm_tc_pack_rows(const float* X, int64_t ld, int d, const int32_t* rows, const int64_t* n_rows, int64_t n_all,
                      float* img, int nkb, const uint64_t* err, cudaStream_t s) {
  if (n_all <= 0) return RTEC_OK;
  RTEC_PROF("k_pack_rows", s);
  launch(k_pack_rows, grid_for(n_all * 32, 256, kSMs * 8), 256, 0, s, X, ld, d, rows, n_rows, n_all, img, nkb, err);
  RTEC_LAUNCH_CHECK("k_pack_rows");
  return RTEC_OK;
}

size_t gemm_tc_smem(int npad, bool fused) {
  TcShape sh = tc_shape(npad, fused);
  return static_cast<size_t>(sh.SA) * 2 * kABlockBytes + static_cast<size_t>(sh.SB) * sh.bstage + kEpiBytes +
         sh.oldb + 1024 + 512;
}

int gemm_tc_launch(const TcArgs& g, cudaStream_t s) {
  if (g.max_rows <= 0) return RTEC_OK;
  const bool fused = g.delta_next && !g.Yt;
  size_t smem = gemm_tc_smem(g.npad, fused);
  static bool configured[kMaxDevices] = {};  // a function attribute is per device
  const int dev = cur_device();
  if (!configured[dev]) {
    RTEC_CUDA(cudaFuncSetAttribute(k_gemm_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    configured[dev] = true;
  }
  int64_t tiles = (g.max_rows + kTM - 1) / kTM;
  int grid = static_cast<int>(tiles < kSMs ? tiles : kSMs);
  RTEC_PROF("k_gemm_tc", s);
  launch(k_gemm_tc, grid, 512, smem, s, g, tc_shape(g.npad, fused));
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
  launch(k_prep_b, grid_for(static_cast<int64_t>(nkb) * npad * kTK, 256), 256, 0, s, W, d_in, d_out, nkb, npad, Bhi, Blo);
  RTEC_LAUNCH_CHECK("k_prep_b");
  return RTEC_OK;
}

}  // extern "C"
