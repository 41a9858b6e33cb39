// scfa_sched.cu — visibility runs and tile schedules.
//
// 1. Visibility runs.  Both sides of every (b, h) slice are sorted — keys by
//    position (QK / dense, pads at the tail) or by (bucket, position) (hash,
//    sort_by_bucket hash_sparse.py:89-133).  The keys a query sees,
//    {k : k_hash == q_hash and k_idx <(=) q_idx} (_tile_mask, _kernel.py:82-89),
//    are therefore ONE contiguous run of key slots: the prefix of the query's
//    bucket run cut at the causal boundary.  Likewise the queries a key is seen
//    by form one run of query slots.  scfa_build_schedule stores that run,
//    [lo, hi), per row slot; the attention kernels turn it into their
//    per-element mask with two subtractions per tile, with no binary search and no
//    per-column index traffic.
// 2. Exact tile lists.  The reference schedules a contiguous key-block range per
//    query block — [0, j_stop) for QK / dense (causal_j_stops, _kernel.py:45-53)
//    and a causally refined bucket band for hash (hash_tile_ranges,
//    _kernel.py:56-79) — and masks inside it.  Here a (row block, column block)
//    tile is listed iff some row's run intersects it, and flagged "full" (bit 15)
//    iff every row's run covers it, so the kernel skips the mask there.
// 3. The reference's own schedule at any BlockSpec, used to report
//    FlashOutputs.tiles_computed with the reference's meaning.
#include <cstdlib>

#ifndef SCFA_LPT_LISTS
#define SCFA_LPT_LISTS 5  // bit z: list z (fwd, dq, dkdv) handed out longest first (dQ: measured slower)
#endif

#include "scfa_common.cuh"
#include "scfa_internal.h"

namespace scfa {

constexpr int kRowBlock = 128;
constexpr int kMaxColBlocks = 2048;  // 131072 streamed slots at 64-slot tiles

// first i in [0, n) with a[i] >= x / > x  (a ascending on [0, n))
SCFA_DEVICE int g_lower(const int32_t* __restrict__ a, int n, int x) {
  int lo = 0;
  while (n > 0) {
    const int h = n >> 1;
    if (__ldg(a + lo + h) < x) { lo += h + 1; n -= h + 1; } else { n = h; }
  }
  return lo;
}
SCFA_DEVICE int g_upper(const int32_t* __restrict__ a, int n, int x) {
  int lo = 0;
  while (n > 0) {
    const int h = n >> 1;
    if (__ldg(a + lo + h) <= x) { lo += h + 1; n -= h + 1; } else { n = h; }
  }
  return lo;
}

// One thread per row slot.  dir 0: rows = queries, run in key-slot space;
// dir 1: rows = keys, run in query-slot space.  Row slots past the true
// length get the empty run.
__global__ void __launch_bounds__(256) runs_kernel(const int32_t* __restrict__ q_idx, const int32_t* __restrict__ q_hash,
                                                   const int32_t* __restrict__ k_idx, const int32_t* __restrict__ k_hash,
                                                   int T_q, int T_kv, int Tq_pad, int Tkv_pad, int flags,
                                                   int2* __restrict__ q_runs, int2* __restrict__ k_runs) {
  const int dir = blockIdx.y;
  const int64_t bh = blockIdx.z;
  const int slot = blockIdx.x * blockDim.x + threadIdx.x;
  const bool excl = (flags & SCFA_FLAG_EXCLUDE_SELF) != 0;
  const bool use_hash = (flags & SCFA_FLAG_HASH) != 0;
  const int32_t* qi = q_idx + bh * Tq_pad;
  const int32_t* ki = k_idx + bh * Tkv_pad;
  const int32_t* qh = use_hash ? q_hash + bh * Tq_pad : nullptr;
  const int32_t* kh = use_hash ? k_hash + bh * Tkv_pad : nullptr;
  if (dir == 0) {
    if (q_runs == nullptr || slot >= Tq_pad) return;
    int2 r = make_int2(0, 0);
    if (slot < T_q && T_kv > 0) {
      const int x = qi[slot];
      if (!use_hash) {  // keys ascending, pads (10^9) at the tail
        r.y = excl ? g_lower(ki, T_kv, x) : g_upper(ki, T_kv, x);
      } else {          // bucket run [a, e), sorted by position inside
        const int g = qh[slot];
        const int a = g_lower(kh, T_kv, g);
        const int e = a + g_upper(kh + a, T_kv - a, g);
        r.x = a;
        r.y = a + (excl ? g_lower(ki + a, e - a, x) : g_upper(ki + a, e - a, x));
      }
    }
    q_runs[bh * Tq_pad + slot] = r;
  } else {
    if (k_runs == nullptr || slot >= Tkv_pad) return;
    int2 r = make_int2(0, 0);
    if (slot < T_kv && T_q > 0) {
      const int x = ki[slot];
      if (!use_hash) {  // real queries ascending, then pads (-1) at the tail
        int n_real = 0, n = T_q;
        while (n > 0) {
          const int h = n >> 1;
          if (__ldg(qi + n_real + h) >= 0) { n_real += h + 1; n -= h + 1; } else { n = h; }
        }
        r.x = excl ? g_upper(qi, n_real, x) : g_lower(qi, n_real, x);
        r.y = n_real;
      } else {
        const int g = kh[slot];
        const int a = g_lower(qh, T_q, g);
        const int e = a + g_upper(qh + a, T_q - a, g);
        r.x = a + (excl ? g_upper(qi + a, e - a, x) : g_lower(qi + a, e - a, x));
        r.y = e;
      }
    }
    k_runs[bh * Tkv_pad + slot] = r;
  }
}

struct ListJob {
  const int2* runs;  // row runs (BH, T_rows_pad)
  uint16_t* list;    // (BH, n_rb, stride)
  int32_t* count;    // (BH, n_rb)
  int64_t stride;
  int T_rows, T_rows_pad, n_rb, n_cb, col_block, col_shift;  // col_block = 1 << col_shift
};

struct ListJobs {
  ListJob job[3];
  unsigned long long* tiles;  // [3] accumulated, may be null
  int BH;
};

// One warp per (list, slice, row block): the same lists as tile_list_kernel without shared
// memory or block barriers.  Every sorted problem here has run starts that never decrease
// along the rows (keys / queries sorted by position, or by (bucket, position) with each
// bucket's runs inside its own slot range), so the union of the rows' column-block ranges
// is an interval merge: a prefix max of the range ends says which blocks each row adds.
// When the union is one interval (QK, dense, shared-id hash: always) the lanes write it
// together; otherwise each row writes the blocks it adds; a decreasing start (never seen)
// falls back to one ballot per column block.  Lists and counts are bit-identical to
// tile_list_kernel's.
__global__ void __launch_bounds__(128) tile_list_warp_kernel(const __grid_constant__ ListJobs jobs, int n_rb_max) {
  const int lane = threadIdx.x & 31;
  // 32-bit index math (3 * BH * n_rb < 2^31, checked by the launcher); column blocks are
  // powers of two, so the block of a column is a shift
  const int w = static_cast<int>(blockIdx.x) * 4 + (threadIdx.x >> 5);
  const int per_z = jobs.BH * n_rb_max;
  const int z = w / per_z;
  if (z >= 3) return;
  const int rem = w - z * per_z;
  const int bh = rem / n_rb_max, rb = rem - bh * n_rb_max;
  const ListJob& J = jobs.job[z];
  if (J.list == nullptr || rb >= J.n_rb) return;
  if (rb == 0 && bh == 0 && lane < 2) J.count[static_cast<int64_t>(jobs.BH) * J.n_rb + lane] = 0;
  const int B = J.col_block, sh = J.col_shift, n_cb = J.n_cb;
  // rows 4 * lane .. 4 * lane + 3 of the block, in order
  int lo[4], hi[4];
  bool ne[4];
  int my_full_lo = 0, my_full_hi = n_cb;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int row = rb * kRowBlock + 4 * lane + i;
    const int2 r = (row < J.T_rows_pad) ? J.runs[static_cast<int64_t>(bh) * J.T_rows_pad + row] : make_int2(0, 0);
    ne[i] = r.y > r.x;
    lo[i] = ne[i] ? r.x >> sh : 0;
    hi[i] = ne[i] ? ((r.y - 1) >> sh) + 1 : 0;
    my_full_lo = max(my_full_lo, ne[i] ? (r.x + B - 1) >> sh : 0);
    my_full_hi = min(my_full_hi, ne[i] ? r.y >> sh : 0);
  }
  const int flo = static_cast<int>(__reduce_max_sync(0xffffffffu, static_cast<unsigned>(my_full_lo)));
  const int fhi = static_cast<int>(__reduce_min_sync(0xffffffffu, static_cast<unsigned>(my_full_hi)));
  // per lane: max end and max start of its rows; a start below an earlier row's start is a
  // decreasing start
  int lmax_hi = 0, lmax_lo = -1, lmin_lo = 0x7fffffff;
  bool mono = true;
#pragma unroll
  for (int i = 0; i < 4; ++i)
    if (ne[i]) {
      mono &= lo[i] >= lmax_lo;
      lmax_lo = max(lmax_lo, lo[i]);
      lmax_hi = max(lmax_hi, hi[i]);
      lmin_lo = min(lmin_lo, lo[i]);
    }
  // exclusive prefix max (over lanes) of ends and starts
  int px_hi = lmax_hi, px_lo = lmax_lo;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int a = __shfl_up_sync(0xffffffffu, px_hi, o), b = __shfl_up_sync(0xffffffffu, px_lo, o);
    if (lane >= o) {
      px_hi = max(px_hi, a);
      px_lo = max(px_lo, b);
    }
  }
  int prev_hi = __shfl_up_sync(0xffffffffu, px_hi, 1), prev_lo = __shfl_up_sync(0xffffffffu, px_lo, 1);
  if (lane == 0) {
    prev_hi = 0;
    prev_lo = -1;
  }
  mono &= (lmin_lo == 0x7fffffff) || lmin_lo >= prev_lo;  // this lane's first start vs every earlier row
  const bool all_mono = __all_sync(0xffffffffu, mono);
  uint16_t* out = J.list + (static_cast<int64_t>(bh) * J.n_rb + rb) * J.stride;
  auto entry = [&](int cb) { return static_cast<uint16_t>(cb | ((cb >= flo && cb < fhi) ? 0x8000 : 0)); };
  int total;
  if (all_mono) {
    int add = 0, run_hi = prev_hi;  // blocks this lane's rows add to the union
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (ne[i]) {
        add += max(0, hi[i] - max(lo[i], run_hi));
        run_hi = max(run_hi, hi[i]);
      }
    int pos = add;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int a = __shfl_up_sync(0xffffffffu, pos, o);
      if (lane >= o) pos += a;
    }
    total = __shfl_sync(0xffffffffu, pos, 31);
    pos -= add;
    const int u_lo = static_cast<int>(__reduce_min_sync(0xffffffffu, static_cast<unsigned>(lmin_lo)));
    const int u_hi = __shfl_sync(0xffffffffu, px_hi, 31);
    if (total > 0 && total == u_hi - u_lo) {  // one interval: written by all lanes
      for (int j = lane; j < total; j += 32) out[j] = entry(u_lo + j);
    } else {
      run_hi = prev_hi;
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (ne[i]) {
          for (int cb = max(lo[i], run_hi); cb < hi[i]; ++cb) out[pos++] = entry(cb);
          run_hi = max(run_hi, hi[i]);
        }
    }
  } else {  // general: one ballot per column block
    total = 0;
    for (int cb = 0; cb < n_cb; ++cb) {
      bool hit = false;
#pragma unroll
      for (int i = 0; i < 4; ++i) hit |= ne[i] && lo[i] <= cb && cb < hi[i];
      if (__any_sync(0xffffffffu, hit)) {
        if (lane == 0) out[total] = entry(cb);
        ++total;
      }
    }
  }
  if (lane == 0) {
    J.count[static_cast<int64_t>(bh) * J.n_rb + rb] = total;
    if (total == 0) out[0] = 0;  // the attention kernels prefetch an item's first entry unconditionally
    if (jobs.tiles) atomicAdd(jobs.tiles + z, static_cast<unsigned long long>(total));
  }
}

// One CTA (128 threads = 128 rows) per (row block, slice, list).  Each row adds its
// run's column-block range to a difference array; a block scan turns it into the
// set of non-empty tiles, listed in ascending order.  The full-tile range is the
// intersection of every row's fully covered blocks.
__global__ void __launch_bounds__(128) tile_list_kernel(const __grid_constant__ ListJobs jobs) {
  __shared__ int diff[kMaxColBlocks + 8];
  __shared__ int warp_tot[4];
  __shared__ int full_lo, full_hi;
  const int z = blockIdx.z;
  const ListJob& J = jobs.job[z];
  const int rb = blockIdx.x;
  const int64_t bh = blockIdx.y;
  if (J.list == nullptr || rb >= J.n_rb) return;
  if (rb == 0 && bh == 0 && threadIdx.x < 2) J.count[static_cast<int64_t>(gridDim.y) * J.n_rb + threadIdx.x] = 0;
  const int n_cb = J.n_cb, B = J.col_block;
  for (int i = threadIdx.x; i <= n_cb; i += blockDim.x) diff[i] = 0;
  if (threadIdx.x == 0) {
    full_lo = 0;
    full_hi = n_cb;
  }
  __syncthreads();
  const int row = rb * kRowBlock + threadIdx.x;
  const int2 r = (row < J.T_rows_pad) ? J.runs[bh * J.T_rows_pad + row] : make_int2(0, 0);
  // Rows of a bucket share run starts (and neighbours share ends): aggregate equal
  // addresses within the warp before the shared-memory atomics, and reduce the full-tile
  // bounds per warp, so no address sees 128 serialized updates.
  const bool nonempty = r.y > r.x;
  const int a_lo = nonempty ? r.x / B : -1 - static_cast<int>(threadIdx.x & 31);
  const int a_hi = nonempty ? (r.y - 1) / B + 1 : -1 - static_cast<int>(threadIdx.x & 31);
  {
    const unsigned lo_peers = __match_any_sync(0xffffffffu, a_lo);
    if (nonempty && (lo_peers & ((1u << (threadIdx.x & 31)) - 1u)) == 0) atomicAdd(&diff[a_lo], __popc(lo_peers));
    const unsigned hi_peers = __match_any_sync(0xffffffffu, a_hi);
    if (nonempty && (hi_peers & ((1u << (threadIdx.x & 31)) - 1u)) == 0) atomicAdd(&diff[a_hi], -__popc(hi_peers));
  }
  const int my_lo = nonempty ? (r.x + B - 1) / B : n_cb;  // first fully covered block
  const int my_hi = nonempty ? r.y / B : 0;                // one past the last fully covered block
  const int w_lo = __reduce_max_sync(0xffffffffu, static_cast<unsigned>(nonempty ? my_lo : 0)) ;
  const int w_hi = static_cast<int>(__reduce_min_sync(0xffffffffu, static_cast<unsigned>(my_hi)));
  if ((threadIdx.x & 31) == 0) {
    atomicMax(&full_lo, w_lo);
    atomicMin(&full_hi, w_hi);
  }
  __syncthreads();
  // ---- ascending compaction of {cb : prefix(diff)[cb] > 0}; thread i owns a chunk
  const int per = (n_cb + blockDim.x - 1) / blockDim.x;
  const int c0 = threadIdx.x * per, c1 = min(n_cb, c0 + per);
  int run = 0, mine = 0;
  for (int c = c0; c < c1; ++c) run += diff[c];
  // exclusive scan of the chunk sums -> running coverage at c0
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int incl = run;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) warp_tot[warp] = incl;
  __syncthreads();
  int cover = incl - run;
  for (int w = 0; w < warp; ++w) cover += warp_tot[w];
  {
    int c = cover;
    for (int i = c0; i < c1; ++i) {
      c += diff[i];
      mine += (c > 0);
    }
  }
  __syncthreads();  // warp_tot reused below
  int pos = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, pos, o);
    if (lane >= o) pos += v;
  }
  if (lane == 31) warp_tot[warp] = pos;
  __syncthreads();
  pos -= mine;
  for (int w = 0; w < warp; ++w) pos += warp_tot[w];
  uint16_t* out = J.list + (bh * J.n_rb + rb) * J.stride;
  const int flo = full_lo, fhi = full_hi;
  {
    int c = cover;
    for (int i = c0; i < c1; ++i) {
      c += diff[i];
      if (c > 0) out[pos++] = static_cast<uint16_t>(i | ((i >= flo && i < fhi) ? 0x8000 : 0));
    }
  }
  if (threadIdx.x == blockDim.x - 1) {
    if (pos == 0) out[0] = 0;  // the attention kernels prefetch an item's first entry unconditionally
    J.count[bh * J.n_rb + rb] = pos;
    if (jobs.tiles) atomicAdd(jobs.tiles + z, static_cast<unsigned long long>(pos));
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

extern "C" int scfa_build_schedule(const int32_t* q_idx, const int32_t* q_hash, const int32_t* k_idx,
                                   const int32_t* k_hash, int64_t BH, int64_t T_q, int64_t T_kv, int64_t Tq_pad,
                                   int64_t Tkv_pad, int flags, int32_t* q_runs, int32_t* k_runs, int runs_ready,
                                   uint16_t* list_fwd,
                                   int32_t* count_fwd, int64_t stride_fwd, uint16_t* list_dq, int32_t* count_dq,
                                   int64_t stride_dq, uint16_t* list_dkdv, int32_t* count_dkdv, int64_t stride_dkdv,
                                   unsigned long long* tiles, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (Tq_pad < ((T_q + 127) / 128) * 128 || Tkv_pad < ((T_kv + 127) / 128) * 128 || BH > 65535) {
    set_error("schedule: padded vectors shorter than the block grid (or too many slices)");
    return SCFA_ERR_SHAPE;
  }
  // (no rows, no runs: an empty side of the problem — e.g. every query dropped — needs none)
  if ((list_fwd || list_dq) && q_runs == nullptr && T_q > 0) {
    set_error("schedule: query-row lists need q_runs");
    return SCFA_ERR_PARAM;
  }
  if (list_dkdv && k_runs == nullptr && T_kv > 0) {
    set_error("schedule: key-row lists need k_runs");
    return SCFA_ERR_PARAM;
  }
  if (BH == 0) return SCFA_OK;
  ListJobs jobs{};
  const int n_rb_q = static_cast<int>((T_q + 127) / 128), n_rb_k = static_cast<int>((T_kv + 127) / 128);
  const int64_t n_cb128_k = (T_kv + 127) / 128, n_cb64_k = (T_kv + 63) / 64, n_cb64_q = (T_q + 63) / 64;
  auto set = [&](int z, const int32_t* runs, uint16_t* list, int32_t* count, int64_t stride, int64_t T_rows,
                 int64_t T_rows_pad, int64_t n_cb, int B) -> int {
    if (!list) return SCFA_OK;
    if (n_cb > kMaxColBlocks || n_cb > 32767 || stride < n_cb || !count) {
      set_error("schedule: sequence too long for the tile lists (or list stride < column blocks)");
      return SCFA_ERR_SHAPE;
    }
    ListJob& J = jobs.job[z];
    J.runs = reinterpret_cast<const int2*>(runs);
    J.list = list;
    J.count = count;
    J.stride = stride;
    J.T_rows = static_cast<int>(T_rows);
    J.T_rows_pad = static_cast<int>(T_rows_pad);
    J.n_rb = static_cast<int>((T_rows + 127) / 128);
    J.n_cb = static_cast<int>(n_cb);
    J.col_block = B;
    J.col_shift = (B == 128) ? 7 : 6;
    return SCFA_OK;
  };
  int rc = set(0, q_runs, list_fwd, count_fwd, stride_fwd, T_q, Tq_pad, n_cb128_k, 128);
  rc = rc ? rc : set(1, q_runs, list_dq, count_dq, stride_dq, T_q, Tq_pad, n_cb64_k, 64);
  rc = rc ? rc : set(2, k_runs, list_dkdv, count_dkdv, stride_dkdv, T_kv, Tkv_pad, n_cb64_q, 64);
  if (rc) return rc;
  jobs.tiles = tiles;
  const int64_t Tmax_pad = Tq_pad > Tkv_pad ? Tq_pad : Tkv_pad;
  int2* q_out = (runs_ready & 1) ? nullptr : reinterpret_cast<int2*>(q_runs);
  int2* k_out = (runs_ready & 2) ? nullptr : reinterpret_cast<int2*>(k_runs);
  if (q_out || k_out) {
    dim3 grid(static_cast<unsigned>((Tmax_pad + 255) / 256), 2, static_cast<unsigned>(BH));
    runs_kernel<<<grid, 256, 0, s>>>(q_idx, (flags & SCFA_FLAG_HASH) ? q_hash : nullptr, k_idx,
                                     (flags & SCFA_FLAG_HASH) ? k_hash : nullptr, static_cast<int>(T_q),
                                     static_cast<int>(T_kv), static_cast<int>(Tq_pad), static_cast<int>(Tkv_pad), flags,
                                     q_out, k_out);
  }
  const int n_rb = n_rb_q > n_rb_k ? n_rb_q : n_rb_k;
  jobs.BH = static_cast<int>(BH);
  if ((list_fwd || list_dq || list_dkdv) && n_rb > 0) {
    static const bool cta_lists = getenv("SCFA_CTA_LISTS") != nullptr;  // diagnostics: the per-CTA kernel
    if (cta_lists) {
      dim3 grid(static_cast<unsigned>(n_rb), static_cast<unsigned>(BH), 3);
      tile_list_kernel<<<grid, 128, 0, s>>>(jobs);
    } else {
      const int64_t warps = 3 * BH * n_rb;
      if (warps >= (1LL << 31) - 4) {
        set_error("schedule: too many (slice, row block) items for the list kernel");
        return SCFA_ERR_SHAPE;
      }
      tile_list_warp_kernel<<<static_cast<unsigned>((warps + 3) / 4), 128, 0, s>>>(jobs, n_rb);
    }
    // the longest items first (count buffers hold the order after the work-counter pair)
    static const int lpt_mask = getenv("SCFA_LPT") ? atoi(getenv("SCFA_LPT")) : SCFA_LPT_LISTS;  // A/B knob
    OrderJob oj[3] = {};
    for (int z = 0; z < 3; ++z)
      if (jobs.job[z].list) oj[z] = OrderJob{jobs.job[z].count, jobs.job[z].n_rb, (lpt_mask >> z) & 1};
    if (launch_item_order(oj, 3, static_cast<int>(BH), s) != SCFA_OK) {
      set_error("schedule: item order launch failed");
      return SCFA_ERR_CUDA;
    }
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("schedule: %s", cudaGetErrorString(e));
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
