// scfa_sched.cu — tile schedules.
//
// 1. Exact tile lists for the tcgen05 kernels.  The reference schedules a
//    contiguous key-block range per query block — [0, j_stop) for the QK and
//    dense kernels (causal_j_stops, _kernel.py:45-53) and a causally refined
//    bucket band [j_start, j_stop) for hash (hash_tile_ranges, _kernel.py:56-79)
//    — and then masks.  Here a tile is listed only if it contains at least one
//    visible pair; that is decided exactly per tile from the sorted index /
//    bucket vectors, and tiles whose pairs are all visible are flagged so the
//    kernel skips the per-element mask there.
// 2. The reference's own schedule at any BlockSpec, used to report
//    FlashOutputs.tiles_computed with the reference's meaning.
#include "scfa_common.cuh"
#include "scfa_internal.h"

namespace scfa {

constexpr int kMaxBlockRows = 128;
constexpr int kMaxColBlocks = 4096;

struct Summary {
  int min_i, max_i, min_h, max_h;
};

// one warp per (bh, block): min/max of index and bucket over all slots of the block
__global__ void block_summary_kernel(const int32_t* __restrict__ idx, const int32_t* __restrict__ hash, int64_t T_pad,
                                     int block, int64_t n_blk, int64_t total, Summary* __restrict__ out) {
  const int64_t w = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= total) return;
  const int64_t bh = w / n_blk, blk = w - bh * n_blk;
  const int32_t* ip = idx + bh * T_pad + blk * block;
  const int32_t* hp = hash ? hash + bh * T_pad + blk * block : nullptr;
  int mn = 0x7fffffff, mx = -0x7fffffff - 1, hmn = 0x7fffffff, hmx = -0x7fffffff - 1;
  for (int i = lane; i < block; i += 32) {
    const int v = ip[i];
    mn = min(mn, v);
    mx = max(mx, v);
    if (hp) {
      const int hv = hp[i];
      hmn = min(hmn, hv);
      hmx = max(hmx, hv);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    hmn = min(hmn, __shfl_xor_sync(0xffffffffu, hmn, o));
    hmx = max(hmx, __shfl_xor_sync(0xffffffffu, hmx, o));
  }
  if (lane == 0) {
    Summary r;
    r.min_i = mn;
    r.max_i = mx;
    r.min_h = hp ? hmn : 0;
    r.max_h = hp ? hmx : 0;
    out[w] = r;
  }
}

SCFA_DEVICE bool causal_ok(int qi, int ki, bool excl) { return excl ? (qi > ki) : (qi >= ki); }

// Tile classification: 0 empty, 1 partial (mask needed), 2 full.
// rows = stationary side (queries if rows_are_queries), cols = streamed side.
__global__ void __launch_bounds__(128) tile_list_kernel(
    const int32_t* __restrict__ q_idx, const int32_t* __restrict__ q_hash, const int32_t* __restrict__ k_idx,
    const int32_t* __restrict__ k_hash, int64_t T_q, int64_t T_kv, int64_t Tq_pad, int64_t Tkv_pad,
    int rows_are_queries, int row_block, int col_block, int flags, const Summary* __restrict__ row_sum,
    const Summary* __restrict__ col_sum, int n_row_blocks, int n_col_blocks, uint16_t* __restrict__ list,
    int32_t* __restrict__ list_count, int64_t list_stride, unsigned long long* tiles_total) {
  __shared__ int r_idx[kMaxBlockRows];
  __shared__ int r_hash[kMaxBlockRows];
  __shared__ uint8_t cls[kMaxColBlocks];
  const int rb = blockIdx.x;
  const int64_t bh = blockIdx.y;
  const bool excl = (flags & SCFA_FLAG_EXCLUDE_SELF) != 0;
  const bool use_hash = (flags & SCFA_FLAG_HASH) != 0;
  const bool rq = rows_are_queries != 0;
  const int32_t* ri = rq ? q_idx + bh * Tq_pad : k_idx + bh * Tkv_pad;
  const int32_t* rh = rq ? q_hash + bh * Tq_pad : k_hash + bh * Tkv_pad;
  const int32_t* ci = rq ? k_idx + bh * Tkv_pad : q_idx + bh * Tq_pad;
  const int32_t* ch = rq ? k_hash + bh * Tkv_pad : q_hash + bh * Tq_pad;
  const int64_t T_rows = rq ? T_q : T_kv, T_cols = rq ? T_kv : T_q;
  const int row0 = rb * row_block;
  const int n_r = static_cast<int>((T_rows - row0) < row_block ? (T_rows - row0) : row_block);
  for (int i = threadIdx.x; i < row_block; i += blockDim.x) {
    r_idx[i] = ri[row0 + i];
    if (use_hash) r_hash[i] = rh[row0 + i];
  }
  __syncthreads();
  const Summary rs = row_sum[bh * n_row_blocks + rb];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = blockDim.x >> 5;
  for (int cb = warp; cb < n_col_blocks; cb += nw) {
    const Summary cs = col_sum[bh * n_col_blocks + cb];
    // query/key views of the two summaries
    const Summary& qs = rq ? rs : cs;
    const Summary& ks = rq ? cs : rs;
    int c = 0;
    bool maybe = causal_ok(qs.max_i, ks.min_i, excl);
    if (use_hash) maybe = maybe && max(qs.min_h, ks.min_h) <= min(qs.max_h, ks.max_h);
    if (maybe) {
      const bool all_vis = causal_ok(qs.min_i, ks.max_i, excl) &&
                           (!use_hash || (qs.min_h == qs.max_h && ks.min_h == ks.max_h && qs.min_h == ks.min_h));
      if (all_vis) {
        c = 2;
      } else if (!use_hash) {
        c = 1;  // sorted indices: max_q vs min_k decides non-emptiness exactly
      } else {
        // exact bucket test: per column bucket g, the row run of g is contiguous and
        // sorted by index, so one binary search finds the extreme row of the run.
        const int col0 = cb * col_block;
        bool hit = false;
        for (int j = lane; j < col_block && !hit; j += 32) {
          const int64_t col = col0 + j;
          if (col >= T_cols) break;
          const int g = ch[col], cidx = ci[col];
          int lo = 0, hi = n_r;
          if (rq) {  // last query row with bucket g (largest index in the run)
            while (lo < hi) { const int mid = (lo + hi) >> 1; if (r_hash[mid] <= g) lo = mid + 1; else hi = mid; }
            const int r = lo - 1;
            hit = (r >= 0 && r_hash[r] == g && causal_ok(r_idx[r], cidx, excl));
          } else {   // first key row with bucket g (smallest index in the run)
            while (lo < hi) { const int mid = (lo + hi) >> 1; if (r_hash[mid] < g) lo = mid + 1; else hi = mid; }
            hit = (lo < n_r && r_hash[lo] == g && causal_ok(cidx, r_idx[lo], excl));
          }
        }
        c = __any_sync(0xffffffffu, hit) ? 1 : 0;
      }
    }
    if (lane == 0) cls[cb] = static_cast<uint8_t>(c);
  }
  __syncthreads();
  if (warp == 0) {
    uint16_t* out = list + (bh * n_row_blocks + rb) * list_stride;
    int n = 0;
    for (int c0 = 0; c0 < n_col_blocks; c0 += 32) {
      const int cb = c0 + lane;
      const int c = cb < n_col_blocks ? cls[cb] : 0;
      const uint32_t bal = __ballot_sync(0xffffffffu, c != 0);
      const int pos = n + __popc(bal & ((1u << lane) - 1u));
      if (c) out[pos] = static_cast<uint16_t>(cb | (c == 2 ? 0x8000 : 0));
      n += __popc(bal);
    }
    if (lane == 0) {
      list_count[bh * n_row_blocks + rb] = n;
      if (tiles_total) atomicAdd(tiles_total, static_cast<unsigned long long>(n));
    }
  }
}

// ---- the reference schedule (reporting only) ----

SCFA_DEVICE void blk_minmax(const int32_t* a, int64_t lo, int64_t hi, int* mn, int* mx) {
  int x = 0x7fffffff, y = -0x7fffffff - 1;
  for (int64_t i = lo; i < hi; ++i) { x = min(x, a[i]); y = max(y, a[i]); }
  *mn = x;
  *mx = y;
}

__global__ void ref_schedule_kernel(const int32_t* __restrict__ q_idx, const int32_t* __restrict__ q_hash,
                                    const int32_t* __restrict__ k_idx, const int32_t* __restrict__ k_hash,
                                    int64_t T_q, int64_t T_kv, int64_t Tq_pad, int64_t Tkv_pad, int64_t B_m,
                                    int64_t B_n, int use_hash, int32_t* j_start, int32_t* j_stop, int64_t* tiles) {
  __shared__ unsigned long long acc;
  const int64_t bh = blockIdx.x;
  const int32_t* qi = q_idx + bh * Tq_pad;
  const int32_t* ki = k_idx + bh * Tkv_pad;
  const int32_t* qh = use_hash ? q_hash + bh * Tq_pad : nullptr;
  const int32_t* kh = use_hash ? k_hash + bh * Tkv_pad : nullptr;
  const int64_t nQ = (T_q + B_m - 1) / B_m, nK = (T_kv + B_n - 1) / B_n;
  if (threadIdx.x == 0) acc = 0;
  __syncthreads();
  unsigned long long mine = 0;
  for (int64_t i = threadIdx.x; i < nQ; i += blockDim.x) {
    const int64_t lo = i * B_m, hi = min(T_q, lo + B_m);
    int mnq, mxq;
    blk_minmax(qi, lo, hi, &mnq, &mxq);
    int64_t js = 0, je;
    if (!use_hash) {
      // searchsorted(min_k, max_q, 'right'), min_k non-decreasing
      int64_t a = 0, b = nK;
      while (a < b) {
        const int64_t mid = (a + b) >> 1;
        int mn, mx;
        blk_minmax(ki, mid * B_n, min(T_kv, (mid + 1) * B_n), &mn, &mx);
        if (mn <= mxq) a = mid + 1; else b = mid;
      }
      je = a;
    } else {
      int mnqh, mxqh;
      blk_minmax(qh, lo, hi, &mnqh, &mxqh);
      int64_t a = 0, b = nK;  // searchsorted(max_kh, min_qh, 'left')
      while (a < b) {
        const int64_t mid = (a + b) >> 1;
        int mn, mx;
        blk_minmax(kh, mid * B_n, min(T_kv, (mid + 1) * B_n), &mn, &mx);
        if (mx < mnqh) a = mid + 1; else b = mid;
      }
      js = a;
      a = 0, b = nK;  // searchsorted(min_kh, max_qh, 'right')
      while (a < b) {
        const int64_t mid = (a + b) >> 1;
        int mn, mx;
        blk_minmax(kh, mid * B_n, min(T_kv, (mid + 1) * B_n), &mn, &mx);
        if (mn <= mxqh) a = mid + 1; else b = mid;
      }
      const int64_t jh = a;
      je = js;
      for (int64_t j = jh - 1; j >= js; --j) {
        int mn, mx;
        blk_minmax(ki, j * B_n, min(T_kv, (j + 1) * B_n), &mn, &mx);
        if (mn <= mxq) { je = j + 1; break; }
      }
    }
    if (je < js) je = js;
    if (j_start) j_start[bh * nQ + i] = static_cast<int32_t>(js);
    if (j_stop) j_stop[bh * nQ + i] = static_cast<int32_t>(je);
    mine += static_cast<unsigned long long>(je - js);
  }
  atomicAdd(&acc, mine);
  __syncthreads();
  if (threadIdx.x == 0 && tiles) tiles[bh] = static_cast<int64_t>(acc);
}

}  // namespace scfa

using namespace scfa;

extern "C" int scfa_build_tile_lists(const int32_t* q_idx, const int32_t* q_hash, const int32_t* k_idx,
                                     const int32_t* k_hash, int64_t BH, int64_t T_q, int64_t T_kv, int64_t Tq_pad,
                                     int64_t Tkv_pad, int rows_are_queries, int row_block, int col_block, int flags,
                                     uint16_t* list, int32_t* list_count, int64_t list_stride,
                                     unsigned long long* tiles_total, void* workspace, int64_t workspace_bytes,
                                     void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const bool rq = rows_are_queries != 0;
  const int64_t T_rows = rq ? T_q : T_kv, T_cols = rq ? T_kv : T_q;
  const int64_t n_rb = (T_rows + row_block - 1) / row_block;
  const int64_t n_cb = (T_cols + col_block - 1) / col_block;
  if (row_block > kMaxBlockRows || n_cb > kMaxColBlocks || n_cb > list_stride || n_cb > 32767) {
    set_error("tile list: sequence too long for the schedule builder");
    return SCFA_ERR_SHAPE;
  }
  const int64_t Tr_pad = rq ? Tq_pad : Tkv_pad, Tc_pad = rq ? Tkv_pad : Tq_pad;
  if (n_rb * row_block > Tr_pad || n_cb * col_block > Tc_pad) {
    set_error("tile list: padded vectors shorter than the block grid");
    return SCFA_ERR_SHAPE;
  }
  if (BH == 0 || n_rb == 0) return SCFA_OK;
  const bool use_hash = (flags & SCFA_FLAG_HASH) != 0;
  const int64_t bytes = BH * (n_rb + n_cb) * static_cast<int64_t>(sizeof(Summary));
  if (workspace == nullptr || workspace_bytes < bytes || (reinterpret_cast<uintptr_t>(workspace) & 15)) {
    set_error("tile list: workspace must be >= %lld bytes, 16-byte aligned", static_cast<long long>(bytes));
    return SCFA_ERR_SHAPE;
  }
  Summary* sums = static_cast<Summary*>(workspace);
  Summary* rsum = sums;
  Summary* csum = sums + BH * n_rb;
  const int32_t* ri = rq ? q_idx : k_idx;
  const int32_t* rh = rq ? q_hash : k_hash;
  const int32_t* ci = rq ? k_idx : q_idx;
  const int32_t* chh = rq ? k_hash : q_hash;
  {
    const int64_t tot = BH * n_rb;
    block_summary_kernel<<<static_cast<unsigned>((tot * 32 + 255) / 256), 256, 0, s>>>(
        ri, use_hash ? rh : nullptr, Tr_pad, row_block, n_rb, tot, rsum);
  }
  if (n_cb > 0) {
    const int64_t tot = BH * n_cb;
    block_summary_kernel<<<static_cast<unsigned>((tot * 32 + 255) / 256), 256, 0, s>>>(
        ci, use_hash ? chh : nullptr, Tc_pad, col_block, n_cb, tot, csum);
  }
  dim3 grid(static_cast<unsigned>(n_rb), static_cast<unsigned>(BH));
  tile_list_kernel<<<grid, 128, 0, s>>>(q_idx, use_hash ? q_hash : q_idx, k_idx, use_hash ? k_hash : k_idx, T_q,
                                        T_kv, Tq_pad, Tkv_pad, rows_are_queries, row_block, col_block, flags, rsum,
                                        csum, static_cast<int>(n_rb), static_cast<int>(n_cb), list, list_count,
                                        list_stride, tiles_total);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("tile list: %s", cudaGetErrorString(e));
    return SCFA_ERR_CUDA;
  }
  return SCFA_OK;
}

extern "C" int scfa_ref_schedule(const int32_t* q_idx, const int32_t* q_hash, const int32_t* k_idx,
                                 const int32_t* k_hash, int64_t BH, int64_t T_q, int64_t T_kv, int64_t Tq_pad,
                                 int64_t Tkv_pad, int64_t B_m, int64_t B_n, int flags, int32_t* j_start,
                                 int32_t* j_stop, int64_t* tiles, void* stream) {
  if (B_m < 1 || B_n < 1) { set_error("block sizes must be >= 1"); return SCFA_ERR_SHAPE; }
  if (BH == 0) return SCFA_OK;
  ref_schedule_kernel<<<static_cast<unsigned>(BH), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      q_idx, q_hash, k_idx, k_hash, T_q, T_kv, Tq_pad, Tkv_pad, B_m, B_n, (flags & SCFA_FLAG_HASH) ? 1 : 0, j_start,
      j_stop, tiles);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("ref_schedule: %s", cudaGetErrorString(e));
    return SCFA_ERR_CUDA;
  }
  return SCFA_OK;
}
