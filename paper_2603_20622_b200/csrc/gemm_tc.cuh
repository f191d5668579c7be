// gemm_tc.cuh -- launcher interface of the tcgen05 3xTF32 update GEMM (gemm_tc.cu).
#pragma once
#include "common.cuh"

namespace rtec {

struct TcArgs {
  const float* A;    // [tiles][nkb][128][32] SW128-swizzled A image
  const float* Bhi;  // [nkb][npad][32] swizzled weights (tf32 hi / lo)
  const float* Blo;
  int nkb, npad, d_out;
  const int64_t* n_rows;  // device row count (or null -> max_rows)
  int64_t max_rows;
  int act;                // 0 none, 1 relu
  float* Y;               // row-major output (scattered by y_rows) ...
  int64_t ldy;
  const int32_t* y_rows;
  float* log;             // DeltaLog of overwritten Y rows (or null)
  float* Yt;              // ... or a tile-layout output feeding a chained GEMM
  int nkb_out;
  const uint64_t* err;
  // fused source deltas of the next layer (sum aggregators): instead of the DeltaLog,
  // delta_next[y_rows[i]] = c_new * h_new - c_old * h_old with c from the out-degrees
  // (GCN 1/sqrt(deg + off), others 1; 0 for a vertex without out-edges)
  float* delta_next;
  const int32_t* deg_new;
  const int32_t* deg_old;
  int coeff_gcn;
  float deg_off;
  int ydiv;  // > 1: Y rows stored per owned vertex at y_rows[i] / ydiv (sharded final layer)
  // non-finite pre-activation output -> NumericError at the row's vertex id (linalg.py:22-29
  // matvec "non-finite result"); null: not checked
  uint64_t* nerr;
};

int gemm_tc_launch(const TcArgs& g, cudaStream_t s);

// rows of a row-major [*, ld] matrix (rows[i], or i when rows is null; i < *n_rows or
// n_all) -> the SW128 A image [tiles][nkb][128][32] with zero K padding beyond d
int gemm_tc_pack_rows(const float* X, int64_t ld, int d, const int32_t* rows, const int64_t* n_rows, int64_t n_all,
                      float* img, int nkb, const uint64_t* err, cudaStream_t s);

__host__ __device__ __forceinline__ int tc_nkb_of(int d) { return (d + 31) / 32; }
__host__ __device__ __forceinline__ int tc_npad_of(int d) { return (d + 15) / 16 * 16; }

}  // namespace rtec
