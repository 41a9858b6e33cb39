// scfa_internal.h — declarations shared between the .cu translation units.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/scfa_b200.h"

namespace scfa {

// Index sentinels (reference pkg/src/scfa/tensors.py:22-24 plus out-of-range slots).
constexpr int32_t kQueryPad = -1;         // QUERY_PAD
constexpr int32_t kKeyPad = 1000000000;   // KEY_PAD = 10**9
constexpr int32_t kColOob = 0x7fffffff;   // key slot past the end of a buffer
constexpr int32_t kQHashOob = -3;         // bucket sentinel of a query slot past the end
constexpr int32_t kKHashOob = -2;         // bucket sentinel of a key slot past the end

struct AttnLaunch {
  int mode;  // 0 fwd, 1 dq, 2 dkdv, 3 fused bwd (dq + dkdv)
  int D;
  int BH;
  int H;             // heads (for the boundary-layout epilogue)
  int T_out;         // boundary-layout sequence length
  int out_boundary;  // 1: epilogue scatters rows to (B, T_out, H, D) by original position
  int T_rows, T_cols, T_rows_pad, T_cols_pad;
  const void* x0;
  const void* x1;
  const void* y0;
  const void* y1;
  const int* row_idx;   // original position per stationary row slot (output routing)
  const int* row_runs;  // (BH, T_rows_pad) int2: visible streamed-slot run [lo, hi)
  const float* lse2;
  const float* delta;
  const int* x_rows;   // gather mode: global row of each stationary slot (BH, T_rows_pad); null = tiled
  const int* y_rows;   // gather mode: global row of each streamed slot (BH, T_cols_pad)
  const int* out_rows; // optional output routing table of the stationary slots (BH, T_rows_pad)
  long long x_nrows;   // rows of the x / out row tables (gather mode)
  long long y_nrows;   // rows of the y row tables
  void* x_out;         // FWD gather mode: stationary Q rows written back in kernel order (BH, T_rows, D)
  const void* x0_tiled;  // DQ gather mode: Q already in kernel order (BH, T_rows, D): tiled loads, only dO gathered
  const void* o_src;   // DQ: O rows (same addressing as dO) for the fused delta = rowsum(dO * O)
  float* delta_out;    // DQ: delta per query slot (BH, T_rows_pad)
  const uint16_t* list;
  const int* list_count;
  int list_stride;
  int n_row_blocks;
  __nv_bfloat16* out_o;
  float* out0;
  float* out1;
  float* out_lse2;
  const int* col_idx;  // BWD: original position per streamed (query) slot (BH, T_cols_pad)
  float* out2;         // BWD: dQ (zero-filled; reduced into)
  int T_out_cols;      // BWD: boundary length of the dQ rows
  float scale;
  int32_t* err_flag;  // FWD: SCFA_ERR_NUMERIC when an output row or its l is non-finite (softmax.py:63-64)
};

int launch_attention(const AttnLaunch& L, cudaStream_t stream);

// Item order of a tile list: after the n = B*H*n_row_blocks counts and the work-counter pair
// of a count buffer (8-byte aligned), n {item, tile count} pairs, most tiles first (LPT: the
// longest items are handed out first, so the grid's last items are its shortest).
__host__ __device__ inline int64_t item_order_offset(int64_t n_items) { return n_items + 2 + (n_items & 1); }
struct OrderJob {
  int32_t* count;  // the list's count buffer (counts, pair, order)
  int n_rb;        // row blocks per slice
  int lpt;         // 0: keep the default order (last row block first, cycling over slices)
};
int launch_item_order(const OrderJob* jobs, int n_jobs, int BH, cudaStream_t stream);
int encode_tensor_map(CUtensorMap* map, int dtype_bytes, int rank, const void* base, const cuuint64_t* dims,
                      const cuuint64_t* strides_bytes, const cuuint32_t* box);
int encode_tensor_map_bf16_3d(CUtensorMap* map, const void* base, const cuuint64_t* dims,
                              const cuuint64_t* strides_bytes, const cuuint32_t* box,
                              const cuuint32_t* elem_strides);
void set_error(const char* fmt, ...);

}  // namespace scfa
