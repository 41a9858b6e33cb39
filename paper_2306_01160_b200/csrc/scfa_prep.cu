// scfa_prep.cu — index preparation for the SCFA path (HBM-bound integer / byte work).
//
//   qk_compact   : stable keep-first permutation per (b, h)   (qk_sparse.py:41-71)
//   hash_sort    : stable LSD radix sort by bucket per (b, h) (hash_sparse.py:89-133)
//   gather_rows  : row gather fused with (B,T,H,D)->(B,H,T,D)  (take_along_axis + to_heads)
//   scatter_rows : inverse routing fused with from_heads       (qk_postprocess / hash_scatter)
//   build_aux    : padded int32 index / bucket vectors         (pad_index, qk_sparse.py:74-83)
//   pack_index, validate_*, bwd_prep (delta = rowsum(dO*O), lse2)
#include <cstdarg>
#include <cstdio>

#include <cooperative_groups.h>

#include "scfa_common.cuh"
#include "scfa_internal.h"

namespace scfa {

// ------------------------------------------------------------------ helpers

SCFA_DEVICE double load_num(const void* p, int dt, int64_t i) {
  switch (dt) {
    case SCFA_DT_F32: return static_cast<double>(static_cast<const float*>(p)[i]);
    case SCFA_DT_F64: return static_cast<const double*>(p)[i];
    case SCFA_DT_U8: return static_cast<double>(static_cast<const uint8_t*>(p)[i]);
    case SCFA_DT_I32: return static_cast<double>(static_cast<const int32_t*>(p)[i]);
    default: return static_cast<double>(static_cast<const int64_t*>(p)[i]);
  }
}

SCFA_DEVICE int64_t load_int(const void* p, int dt, int64_t i) {
  switch (dt) {
    case SCFA_DT_I32: return static_cast<const int32_t*>(p)[i];
    case SCFA_DT_I64: return static_cast<const int64_t*>(p)[i];
    case SCFA_DT_U8: return static_cast<const uint8_t*>(p)[i];
    case SCFA_DT_F32: return static_cast<int64_t>(static_cast<const float*>(p)[i]);
    default: return static_cast<int64_t>(static_cast<const double*>(p)[i]);
  }
}

SCFA_DEVICE void flag_error(int32_t* err, int code) {
  if (err) atomicCAS(err, 0, code);
}

SCFA_DEVICE uint32_t lanemask_lt() {
  uint32_t r;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
  return r;
}

// Block-wide exclusive scan of one int per warp (<= 32 warps); returns the
// exclusive prefix for the calling warp and the block total in *total.
SCFA_DEVICE int warp_offsets(int warp_val, int* sm /*32+1*/, int* total) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = (blockDim.x + 31) >> 5;
  if (lane == 0) sm[warp] = warp_val;
  __syncthreads();
  if (warp == 0) {
    int v = lane < nwarps ? sm[lane] : 0;
    int incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int n = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += n;
    }
    sm[lane] = incl - v;
    if (lane == 31) sm[32] = incl;
  }
  __syncthreads();
  int r = sm[warp];
  *total = sm[32];
  __syncthreads();
  return r;
}

// ------------------------------------------------------------------ QK compaction

__global__ void qk_compact_kernel(const void* keep, int dt, int64_t T, int64_t H, int64_t sb, int64_t st,
                                  int64_t sh, int32_t* perm, int32_t* rank, int32_t* counts, int32_t* err) {
  __shared__ int sm[33];
  const int64_t bh = blockIdx.x;
  const int64_t b = bh / H, h = bh % H;
  const int64_t base = b * sb + h * sh;
  const int lane = threadIdx.x & 31;

  // pass 1: kept count (and {0,1} check)
  int cnt = 0;
  for (int64_t t = threadIdx.x; t < T; t += blockDim.x) {
    const double v = load_num(keep, dt, base + t * st);
    if (v == 1.0) ++cnt;
    else if (v != 0.0) flag_error(err, SCFA_ERR_SHAPE);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  int total_kept;
  warp_offsets(cnt, sm, &total_kept);
  if (threadIdx.x == 0) counts[bh] = total_kept;

  // pass 2: slots.  kept t -> #kept before t ; dropped t -> total_kept + #dropped before t
  int running = 0;
  for (int64_t c0 = 0; c0 < T; c0 += blockDim.x) {
    const int64_t t = c0 + threadIdx.x;
    const bool kept = (t < T) && (load_num(keep, dt, base + t * st) == 1.0);
    const uint32_t bal = __ballot_sync(0xffffffffu, kept);
    const int in_warp = __popc(bal & lanemask_lt());
    int chunk_total;
    const int woff = warp_offsets(lane == 0 ? __popc(bal) : 0, sm, &chunk_total);
    if (t < T) {
      const int kb = running + woff + in_warp;
      const int slot = kept ? kb : total_kept + static_cast<int>(t - kb);
      perm[bh * T + slot] = static_cast<int32_t>(t);
      rank[bh * T + t] = slot;
    }
    running += chunk_total;
  }
}

// ------------------------------------------------------------------ fused QK preparation
//
// The fused QK fwd + bwd's whole index preparation for one (b, h) slice per CTA, static sizes
// (every position has a slot: kept positions first in position order, then the dropped
// ones, qk_sparse.py:41-71 with the buffer = T instead of the max kept count):
//   perm / rank                       compact()'s argsort(~kept, stable) and its inverse
//   q_idx / k_idx (padded)            pad_index (qk_sparse.py:74-83): QUERY_PAD / KEY_PAD
//   row tables                        slot -> row of the caller's (B, T, H, D) tensors
//   visibility runs                   causal (k_idx <= q_idx, _kernel.py:82-89): a kept query
//                                     at position t sees key slots [0, #kept keys <= t); a
//                                     kept key at t is seen by query slots [#kept q < t, #kept q)
// Keep vectors are read once (every thread a contiguous segment of positions, all loads in
// flight), one block scan per side gives the kept-before counts, and both sides' prefix
// counts sit in shared memory so the runs need no search.  Replaces two compaction passes,
// two aux builds, two row maps and the runs kernel (seven launches) by one.
constexpr int kQkPrepThreads = 1024;
constexpr int kQkPrepMaxT = 16384;

SCFA_DEVICE int block_excl_scan(int v, int* sm, int* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int n = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += n;
  }
  if (lane == 31) sm[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const int w = (lane < static_cast<int>(blockDim.x >> 5)) ? sm[lane] : 0;
    int wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int n = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += n;
    }
    sm[lane] = wi - w;
    if (lane == 31) sm[32] = wi;
  }
  __syncthreads();
  const int r = sm[warp] + incl - v;
  *total = sm[32];
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(kQkPrepThreads) qk_prepare_kernel(
    const void* keep_q, int dtq, int64_t sbq, int64_t stq, int64_t shq, const void* keep_k, int dtk, int64_t sbk,
    int64_t stk, int64_t shk, int T_Q, int T_KV, int Tq_pad, int Tkv_pad, int H, int32_t* perm_q, int32_t* rank_q,
    int32_t* perm_k, int32_t* rank_k, int32_t* q_idx, int32_t* k_idx, int2* q_runs, int2* k_runs, int32_t* q_rows,
    int32_t* k_rows, int32_t* counts, int BH, int32_t* err) {
  // Position t = c * 1024 + threadIdx.x (chunk c): a warp covers 32 consecutive positions, so
  // the keep loads, rank stores and (kept or dropped runs of) slot stores are coalesced.
  extern __shared__ __align__(16) int qsm[];
  int* pq = qsm;                                  // [T_Q + 1]: kept queries before position t
  int* pk = pq + T_Q + 1;                         // [T_KV + 1]: kept keys before position t
  int* wc = pk + T_KV + 1;                        // [2][kChunks * 32]: per (chunk, warp) kept counts
  int* red = wc + 2 * (kQkPrepMaxT / 32);         // 33 ints scan scratch
  constexpr int kChunks = kQkPrepMaxT / kQkPrepThreads;
  const int bh = blockIdx.x;
  const int b = bh / H, h = bh - b * H;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t lt = lanemask_lt();
  uint32_t bq = 0, bk = 0;  // keep bit of this thread's position in each chunk
  bool bad = false;
  constexpr int kBatch = 8;
#pragma unroll
  for (int c0 = 0; c0 < kChunks; c0 += kBatch) {
    double vq[kBatch], vk[kBatch];
#pragma unroll
    for (int j2 = 0; j2 < kBatch; ++j2) {  // a batch of loads in flight per side
      const int t = (c0 + j2) * kQkPrepThreads + threadIdx.x;
      vq[j2] = (t < T_Q) ? load_num(keep_q, dtq, b * sbq + h * shq + static_cast<int64_t>(t) * stq) : 0.0;
      vk[j2] = (t < T_KV) ? load_num(keep_k, dtk, b * sbk + h * shk + static_cast<int64_t>(t) * stk) : 0.0;
    }
#pragma unroll
    for (int j2 = 0; j2 < kBatch; ++j2) {
      bad |= !(vq[j2] == 0.0 || vq[j2] == 1.0) || !(vk[j2] == 0.0 || vk[j2] == 1.0);
      bq |= (vq[j2] == 1.0 ? 1u : 0u) << (c0 + j2);
      bk |= (vk[j2] == 1.0 ? 1u : 0u) << (c0 + j2);
    }
  }
  if (bad) flag_error(err, SCFA_ERR_SHAPE);  // keep entries must be 0 or 1 (qk_sparse.py:54-55)
  // per (chunk, warp) counts in position order, one block scan over them per side
#pragma unroll
  for (int c = 0; c < kChunks; ++c) {
    const uint32_t balq = __ballot_sync(0xffffffffu, (bq >> c) & 1u);
    const uint32_t balk = __ballot_sync(0xffffffffu, (bk >> c) & 1u);
    if (lane == 0) {
      wc[c * 32 + warp] = __popc(balq);
      wc[kChunks * 32 + c * 32 + warp] = __popc(balk);
    }
  }
  __syncthreads();
  int nq = 0, nk = 0;
  {  // 512 entries per side: threads [0, 512) scan q, then k
    const int e = threadIdx.x & (kChunks * 32 - 1);
    const int vq0 = (threadIdx.x < kChunks * 32) ? wc[e] : 0;
    const int oq = block_excl_scan(vq0, red, &nq);
    const int vk0 = (threadIdx.x < kChunks * 32) ? wc[kChunks * 32 + e] : 0;
    const int ok = block_excl_scan(vk0, red, &nk);
    if (threadIdx.x < kChunks * 32) {
      wc[e] = oq;
      wc[kChunks * 32 + e] = ok;
    }
  }
  __syncthreads();
#pragma unroll
  for (int c = 0; c < kChunks; ++c) {
    const int t = c * kQkPrepThreads + threadIdx.x;
    const uint32_t balq = __ballot_sync(0xffffffffu, (bq >> c) & 1u);
    const uint32_t balk = __ballot_sync(0xffffffffu, (bk >> c) & 1u);
    if (t < T_Q) pq[t] = wc[c * 32 + warp] + __popc(balq & lt);
    if (t < T_KV) pk[t] = wc[kChunks * 32 + c * 32 + warp] + __popc(balk & lt);
  }
  if (threadIdx.x == 0) {
    pq[T_Q] = nq;
    pk[T_KV] = nk;
    counts[bh] = nq;
    counts[BH + bh] = nk;
  }
  __syncthreads();
  const size_t oqs = static_cast<size_t>(bh) * Tq_pad, oks = static_cast<size_t>(bh) * Tkv_pad;
#pragma unroll
  for (int c = 0; c < kChunks; ++c) {
    const int t = c * kQkPrepThreads + threadIdx.x;
    if (t < T_Q) {  // queries: slot, padded idx, row, run
      const bool kept = (bq >> c) & 1u;
      const int before = pq[t];
      const int slot = kept ? before : nq + (t - before);
      perm_q[static_cast<size_t>(bh) * T_Q + slot] = t;
      rank_q[static_cast<size_t>(bh) * T_Q + t] = slot;
      q_idx[oqs + slot] = kept ? t : kQueryPad;
      q_rows[oqs + slot] = (b * T_Q + t) * H + h;
      const int hi = (T_KV == 0) ? 0 : (t + 1 <= T_KV ? pk[t + 1] : nk);  // keys at positions <= t
      q_runs[oqs + slot] = kept ? make_int2(0, hi) : make_int2(0, 0);
    }
    if (t < T_KV) {  // keys: seen by the kept queries at positions >= t; dropped: (nq, nq)
      const bool kept = (bk >> c) & 1u;
      const int before = pk[t];
      const int slot = kept ? before : nk + (t - before);
      perm_k[static_cast<size_t>(bh) * T_KV + slot] = t;
      rank_k[static_cast<size_t>(bh) * T_KV + t] = slot;
      k_idx[oks + slot] = kept ? t : kKeyPad;
      k_rows[oks + slot] = (b * T_KV + t) * H + h;
      const int lo = (T_Q == 0) ? 0 : (t <= T_Q ? pq[t] : nq);
      k_runs[oks + slot] = (T_Q == 0) ? make_int2(0, 0) : (kept ? make_int2(lo, nq) : make_int2(nq, nq));
    }
  }
  // pad slots past the lengths: out-of-range idx, empty runs, a valid row (slot 0's)
  __syncthreads();
  for (int s2 = T_Q + threadIdx.x; s2 < Tq_pad; s2 += blockDim.x) {
    q_idx[oqs + s2] = kQueryPad;
    q_runs[oqs + s2] = make_int2(0, 0);
    q_rows[oqs + s2] = (T_Q > 0) ? (b * T_Q + perm_q[static_cast<size_t>(bh) * T_Q]) * H + h : 0;
  }
  for (int s2 = T_KV + threadIdx.x; s2 < Tkv_pad; s2 += blockDim.x) {
    k_idx[oks + s2] = kColOob;
    k_runs[oks + s2] = make_int2(0, 0);
    k_rows[oks + s2] = (T_KV > 0) ? (b * T_KV + perm_k[static_cast<size_t>(bh) * T_KV]) * H + h : 0;
  }
}

// ------------------------------------------------------------------ hash radix sort

constexpr int kSortThreads = 1024;

struct SortSmem {
  uint16_t wcnt[32][256];
  int bin_base[256];
  int tile_tot[256];
  int hist[256];
  int red[33];
  long long mx[2];
};

__global__ void __launch_bounds__(kSortThreads) hash_sort_kernel(
    const void* hash, int hdt, int64_t T, int64_t H, int64_t sb, int64_t st, int64_t sh, const void* pos, int pdt,
    int64_t ps_bh, int64_t ps_t, int32_t* perm, int32_t* rank, int32_t* scratch, int32_t* err) {
  __shared__ SortSmem S;
  const int64_t bh = blockIdx.x;
  const int64_t b = bh / H, h = bh % H;
  const int64_t hbase = b * sb + h * sh;
  const int64_t pbase = bh * ps_bh;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // validate and find the largest key of each kind
  long long mh = 0, mp = 0;
  for (int64_t t = threadIdx.x; t < T; t += blockDim.x) {
    const long long hv = load_int(hash, hdt, hbase + t * st);
    if (hv < 0 || hv > 0x7fffffffLL) flag_error(err, SCFA_ERR_SHAPE);
    mh = max(mh, hv);
    if (pos) {
      const long long pv = load_int(pos, pdt, pbase + t * ps_t);
      if (pv < 0 || pv > 0x7fffffffLL) flag_error(err, SCFA_ERR_SHAPE);
      mp = max(mp, pv);
    }
  }
  if (threadIdx.x == 0) { S.mx[0] = 0; S.mx[1] = 0; }
  __syncthreads();
  atomicMax(reinterpret_cast<unsigned long long*>(&S.mx[0]), static_cast<unsigned long long>(max(mh, 0LL)));
  atomicMax(reinterpret_cast<unsigned long long*>(&S.mx[1]), static_cast<unsigned long long>(max(mp, 0LL)));
  __syncthreads();
  const long long max_h = S.mx[0], max_p = S.mx[1];
  auto nbytes = [](long long m) { int n = 0; while (m > 0) { ++n; m >>= 8; } return n; };
  const int pos_passes = pos ? nbytes(max_p) : 0;
  const int hash_passes = nbytes(max_h);
  const int passes = pos_passes + hash_passes;

  // the final pass must land in `perm`
  int32_t* bufs[2] = {perm + bh * T, scratch + bh * T};
  int cur = (passes & 1) ? 1 : 0;
  for (int64_t s = threadIdx.x; s < T; s += blockDim.x) bufs[cur][s] = static_cast<int32_t>(s);
  __syncthreads();

  for (int p = 0; p < passes; ++p) {
    const bool by_pos = p < pos_passes;
    const int shift = 8 * (by_pos ? p : p - pos_passes);
    const int32_t* src = bufs[cur];
    int32_t* dst = bufs[cur ^ 1];
    auto digit = [&](int32_t t) -> int {
      const long long key = by_pos ? load_int(pos, pdt, pbase + t * ps_t) : load_int(hash, hdt, hbase + t * st);
      return static_cast<int>((key >> shift) & 255);
    };
    for (int i = threadIdx.x; i < 256; i += blockDim.x) S.hist[i] = 0;
    for (int i = threadIdx.x; i < 32 * 256; i += blockDim.x) (&S.wcnt[0][0])[i] = 0;
    __syncthreads();
    for (int64_t s = threadIdx.x; s < T; s += blockDim.x) atomicAdd(&S.hist[digit(src[s])], 1);
    __syncthreads();
    if (threadIdx.x == 0) {
      int acc = 0;
      for (int i = 0; i < 256; ++i) { S.bin_base[i] = acc; acc += S.hist[i]; }
    }
    __syncthreads();
    for (int64_t c0 = 0; c0 < T; c0 += blockDim.x) {
      const int64_t s = c0 + threadIdx.x;
      const bool act = s < T;
      const int32_t val = act ? src[s] : 0;
      const int d = act ? digit(val) : 256 + lane;  // inactive lanes never match a real digit
      const uint32_t same = __match_any_sync(0xffffffffu, d);
      const int r_in = __popc(same & lanemask_lt());
      if (act && r_in == 0) S.wcnt[warp][d] = static_cast<uint16_t>(__popc(same));
      __syncthreads();
      if (threadIdx.x < 256) {
        int acc = 0;
        for (int w = 0; w < 32; ++w) {
          const int c = S.wcnt[w][threadIdx.x];
          S.wcnt[w][threadIdx.x] = static_cast<uint16_t>(acc);
          acc += c;
        }
        S.tile_tot[threadIdx.x] = acc;
      }
      __syncthreads();
      if (act) dst[S.bin_base[d] + S.wcnt[warp][d] + r_in] = val;
      __syncthreads();
      if (threadIdx.x < 256) {
        S.bin_base[threadIdx.x] += S.tile_tot[threadIdx.x];
        for (int w = 0; w < 32; ++w) S.wcnt[w][threadIdx.x] = 0;
      }
      __syncthreads();
    }
    cur ^= 1;
  }
  // cur == 0 now (perm)
  for (int64_t s = threadIdx.x; s < T; s += blockDim.x) rank[bh * T + perm[bh * T + s]] = static_cast<int32_t>(s);
}

// ------------------------------------------------------------------ fused hash preparation
//
// Shared bucket ids (q_hash is k_hash, T_Q == T_KV, positions = arange — the
// reference's own bench / LM setting, cli.py:481-487): one CTA per (b, h) slice
// does, with the slice's keys cached in shared memory,
//   sort_by_bucket's stable argsort (hash_sparse.py:89-94)        -> perm, rank
//   the sorted idx / hash vectors (hash_sparse.py:127-133, padded) -> idx_*, hash_*
//   the visibility runs (scfa_sched.cu runs_kernel), which for shared ids are
//   O(1) per slot: a query slot s in bucket run [a, e) sees key slots [a, s)
//   ([a, s] without exclude_self) and key slot s is seen by query slots (s, e).
// That replaces hash_sort + 2 x build_aux + runs_kernel (four launches, three
// re-reads of the ids from HBM) by one launch.

constexpr int kPrepMaxT = 16384;

struct PrepSmem {
  int cnt[256][33];  // per (digit, warp) counts, then exclusive offsets (digit-major);
                     // row padded to 33 so a warp's lanes (one warp column, many digits)
                     // fall in different banks
  int red[33];
  long long mx;
};

SCFA_DEVICE int lower_bound_s(const int32_t* a, int n, int x) {
  int lo = 0;
  while (n > 0) {
    const int h = n >> 1;
    if (a[lo + h] < x) { lo += h + 1; n -= h + 1; } else { n = h; }
  }
  return lo;
}

// Stable LSD radix pass (8-bit digit) of the slice: warp w owns the contiguous slot
// segment [w * seg, (w + 1) * seg) of `src` and walks it in order, so
//   slot = sum of counts of smaller digits (all warps) + counts of this digit in
//          earlier warps + this warp's running count + rank among equal lanes,
// which is exactly argsort(kind="stable").  Two walks, three __syncthreads.
SCFA_DEVICE void radix_pass(PrepSmem& S, const int32_t* key, int T, int shift, const int32_t* src, int32_t* dst,
                           int32_t* sorted_key, int32_t* rank = nullptr) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int seg = (((T + 31) / 32) + 31) & ~31;
  const int s0 = warp * seg, s1 = min(T, s0 + seg);
  for (int i = threadIdx.x; i < 256 * 33; i += blockDim.x) (&S.cnt[0][0])[i] = 0;
  __syncthreads();
  for (int base = s0; base < s1; base += 32) {
    const int s = base + lane;
    const bool act = s < s1;
    const int d = act ? ((key[src ? src[s] : s] >> shift) & 255) : 256 + lane;
    const uint32_t peers = __match_any_sync(0xffffffffu, d);
    if (act && (peers & lanemask_lt()) == 0) S.cnt[d][warp] += __popc(peers);
    __syncwarp();  // the next group leader of digit d (another lane) reads this count
  }
  __syncthreads();
  {  // exclusive scan of cnt in (digit, warp) order: 8 entries per thread
    int* flat = &S.cnt[0][0];
    const int i0 = threadIdx.x * 8;  // flat (digit, warp) index; entry f lives at (f / 32) * 33 + f % 32
    const int a0 = (i0 >> 5) * 33 + (i0 & 31);
    int loc[8], sum = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) { loc[i] = flat[a0 + i]; sum += loc[i]; }
    int incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int n = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += n;
    }
    if (lane == 31) S.red[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      const int v = S.red[lane];
      int w = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int n = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += n;
      }
      S.red[lane] = w - v;
    }
    __syncthreads();
    int acc = S.red[warp] + incl - sum;
#pragma unroll
    for (int i = 0; i < 8; ++i) { flat[a0 + i] = acc; acc += loc[i]; }
  }
  __syncthreads();
  for (int base = s0; base < s1; base += 32) {
    const int s = base + lane;
    const bool act = s < s1;
    const int32_t val = act ? (src ? src[s] : s) : 0;
    const int d = act ? ((key[val] >> shift) & 255) : 256 + lane;
    const uint32_t peers = __match_any_sync(0xffffffffu, d);
    const int below = __popc(peers & lanemask_lt());
    int off = 0;
    if (act) off = S.cnt[d][warp];
    __syncwarp();
    if (act) {
      dst[off + below] = val;
      if (sorted_key) sorted_key[off + below] = key[val];
      if (rank) rank[val] = off + below;
      if (below == 0) S.cnt[d][warp] = off + __popc(peers);
    }
    __syncwarp();
  }
  __syncthreads();
}

// Item order of the tile lists (one CTA per list): the attention kernels' default order
// (last row block first, cycling over slices) stably re-sorted by tile count, longest first —
// an LPT schedule: with items handed out dynamically, the last ones left are the shortest, so
// the streams of a persistent grid finish close together.  One 8-bit counting pass (counts
// above 255 share the top class).  Lists of more than kPrepMaxT items keep the default order.
struct OrderJobs {
  OrderJob job[3];
  int BH;
  int cap;  // items per shared-memory array (the largest sorted list)
};

__global__ void __launch_bounds__(kSortThreads) item_order_kernel(const __grid_constant__ OrderJobs J) {
  extern __shared__ __align__(16) uint8_t dsm[];
  PrepSmem& S = *reinterpret_cast<PrepSmem*>(dsm);
  int32_t* key = reinterpret_cast<int32_t*>(dsm + sizeof(PrepSmem));
  const OrderJob& o = J.job[blockIdx.x];
  if (o.count == nullptr) return;
  const int n = J.BH * o.n_rb;
  int32_t* order = o.count + item_order_offset(n);
  auto item_of = [&](int w) {  // scfa_attn.cu item_of: last row block first, cycling over slices
    const int rb = o.n_rb - 1 - w / J.BH, bh = w - (w / J.BH) * J.BH;
    return bh * o.n_rb + rb;
  };
  if (n > J.cap || !o.lpt) {
    for (int w = threadIdx.x; w < n; w += blockDim.x) {
      const int it = item_of(w);
      order[2 * w] = it;
      order[2 * w + 1] = o.count[it];
    }
    return;
  }
  int32_t* sorted = key + J.cap;
  for (int w = threadIdx.x; w < n; w += blockDim.x) key[w] = 255 - min(o.count[item_of(w)], 255);
  __syncthreads();
  radix_pass(S, key, n, 0, nullptr, sorted, nullptr, nullptr);  // stable: equal counts keep their order
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    const int it = item_of(sorted[j]);
    order[2 * j] = it;
    order[2 * j + 1] = o.count[it];
  }
}

int launch_item_order(const OrderJob* jobs, int n_jobs, int BH, cudaStream_t stream) {
  OrderJobs J{};
  int cap = 0;  // shared memory sized for the lists actually sorted (at most kPrepMaxT items)
  for (int i = 0; i < n_jobs && i < 3; ++i) {
    J.job[i] = jobs[i];
    const int n = BH * jobs[i].n_rb;
    if (jobs[i].count && jobs[i].lpt && n <= kPrepMaxT && n > cap) cap = n;
  }
  J.BH = BH;
  J.cap = (cap + 31) & ~31;
  const size_t smem = sizeof(PrepSmem) + 2 * static_cast<size_t>(J.cap) * sizeof(int32_t);
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(item_order_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(sizeof(PrepSmem) + 2 * kPrepMaxT * sizeof(int32_t))) != cudaSuccess)
      return SCFA_ERR_CUDA;
    attr = true;
  }
  item_order_kernel<<<3, kSortThreads, smem, stream>>>(J);
  return cudaGetLastError() == cudaSuccess ? SCFA_OK : SCFA_ERR_CUDA;
}

// Kernel 1 (one CTA per slice): keys cached in shared memory, stable LSD radix
// passes -> perm; the final pass also writes the sorted ids.  With one pass (ids <
// 256, every bench / LM bucket count) the pass's digit offsets ARE the bucket runs:
// bounds[bh][g] = first slot of bucket g, bounds[bh][256] = T.  bounds[bh][0] = -1
// flags a multi-pass sort (the finishing kernel then searches the sorted ids).
__global__ void __launch_bounds__(kSortThreads) hash_prepare_sort_kernel(
    const void* hash, int hdt, int T, int T_pad, int64_t H, int64_t sb, int64_t st, int64_t sh, int32_t* perm,
    int32_t* rank, int32_t* scratch, int32_t* sorted_hash, int32_t* err) {
  extern __shared__ __align__(16) uint8_t dsm[];
  PrepSmem& S = *reinterpret_cast<PrepSmem*>(dsm);
  int32_t* key = reinterpret_cast<int32_t*>(dsm + sizeof(PrepSmem));
  const int64_t bh = blockIdx.x;
  const int64_t b = bh / H, h = bh % H;
  const int64_t hbase = b * sb + h * sh;

  constexpr int kMaxPer = kPrepMaxT / kSortThreads;
  long long v[kMaxPer];
#pragma unroll
  for (int i = 0; i < kMaxPer; ++i) {  // all loads in flight before any use
    const int t = threadIdx.x + i * kSortThreads;
    v[i] = t < T ? load_int(hash, hdt, hbase + t * st) : 0;
  }
  long long mh = 0;
  bool bad = false;
#pragma unroll
  for (int i = 0; i < kMaxPer; ++i) {
    const int t = threadIdx.x + i * kSortThreads;
    if (t < T) {
      bad |= (v[i] < 0 || v[i] > 0x7fffffffLL);
      const long long c = v[i] < 0 ? 0 : (v[i] > 0x7fffffffLL ? 0x7fffffffLL : v[i]);
      key[t] = static_cast<int32_t>(c);
      mh = max(mh, c);
    }
  }
  if (bad) flag_error(err, SCFA_ERR_SHAPE);
  if (threadIdx.x == 0) S.mx = 0;
  __syncthreads();
  atomicMax(reinterpret_cast<unsigned long long*>(&S.mx), static_cast<unsigned long long>(mh));
  __syncthreads();
  int passes = 0;
  for (long long m = S.mx; m > 0; m >>= 8) ++passes;

  int32_t* P = perm + bh * T;
  int32_t* X = scratch + bh * (T + 257);  // radix ping-pong, then the slice's bucket bounds
  int32_t* bounds = X + T;
  int32_t* SH = sorted_hash + bh * T_pad;
  if (passes == 0) {
    for (int s = threadIdx.x; s < T; s += blockDim.x) { P[s] = s; SH[s] = 0; rank[bh * T + s] = s; }
    if (threadIdx.x <= 256) bounds[threadIdx.x] = (threadIdx.x == 0) ? 0 : T;
    return;
  }
  for (int p = 0; p < passes; ++p) {  // the final pass lands in perm; pass 0 reads the identity
    const bool last = p == passes - 1;
    const bool to_perm = ((passes - 1 - p) & 1) == 0;
    radix_pass(S, key, T, 8 * p, p == 0 ? nullptr : (to_perm ? X : P), to_perm ? P : X, last ? SH : nullptr,
               last ? rank + bh * T : nullptr);
  }
  // radix_pass leaves each digit's end offset in S.cnt[d][31] (after the last walk)
  if (threadIdx.x < 256) {
    const int start = threadIdx.x == 0 ? 0 : S.cnt[threadIdx.x - 1][31];
    bounds[threadIdx.x] = (passes == 1) ? start : -1;
  }
  if (threadIdx.x == 0) bounds[256] = T;
}

// Kernel 1, cluster form (the common case: every id < 256, one counting pass): a cluster
// of kSortCluster CTAs per slice, each owning a contiguous quarter of the positions, so a
// slice is sorted by 4x the SMs.  Each CTA counts its quarter per (digit, warp); the
// clusters' per-digit totals are exchanged through distributed shared memory, giving
// every CTA its global slot base per digit (stable: lower quarters first, then warps in
// order, then lanes).  Multi-pass ids (>= 256) fall back to the single-CTA path in CTA 0.
constexpr int kSortCluster = 4;

struct ClusterSortSmem {
  int ctot[256];   // this CTA's count per digit
  int dbase[256];  // global first slot of each digit
  int before[256];  // slots of each digit in lower-ranked CTAs
  int wsum[8];
  unsigned long long mx;
};

__global__ void __cluster_dims__(kSortCluster, 1, 1) __launch_bounds__(kSortThreads, 2)
    hash_prepare_sort_cluster_kernel(const void* hash, int hdt, int T, int T_pad, int64_t H, int64_t sb, int64_t st,
                                     int64_t sh, int32_t* perm, int32_t* rank, int32_t* scratch,
                                     int32_t* sorted_hash, int32_t* err) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ __align__(16) uint8_t dsm[];
  PrepSmem& S = *reinterpret_cast<PrepSmem*>(dsm);
  ClusterSortSmem& C = *reinterpret_cast<ClusterSortSmem*>(dsm + sizeof(PrepSmem));
  int32_t* key = reinterpret_cast<int32_t*>(dsm + sizeof(PrepSmem) + sizeof(ClusterSortSmem));
  const int crank = static_cast<int>(cluster.block_rank());
  const int64_t bh = blockIdx.x / kSortCluster;
  const int64_t b = bh / H, h = bh % H;
  const int64_t hbase = b * sb + h * sh;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int segT = ((T + kSortCluster - 1) / kSortCluster + 31) & ~31;
  const int s0 = min(T, crank * segT), s1 = min(T, s0 + segT), nloc = s1 - s0;
  int32_t* P = perm + bh * T;
  int32_t* R = rank + bh * T;
  int32_t* X = scratch + bh * (T + 257);
  int32_t* bounds = X + T;
  int32_t* SH = sorted_hash + bh * T_pad;

  // ---- this CTA's keys, validity and max
  long long mh = 0;
  bool bad = false;
  for (int i = threadIdx.x; i < nloc; i += blockDim.x) {
    const long long v = load_int(hash, hdt, hbase + static_cast<int64_t>(s0 + i) * st);
    bad |= (v < 0 || v > 0x7fffffffLL);
    const long long c = v < 0 ? 0 : (v > 0x7fffffffLL ? 0x7fffffffLL : v);
    key[i] = static_cast<int32_t>(c);
    mh = max(mh, c);
  }
  if (bad) flag_error(err, SCFA_ERR_SHAPE);
  if (threadIdx.x == 0) C.mx = 0;
  for (int i = threadIdx.x; i < 256 * 33; i += blockDim.x) (&S.cnt[0][0])[i] = 0;
  __syncthreads();
  atomicMax(&C.mx, static_cast<unsigned long long>(mh));
  // ---- one counting pass (ids < 256, the common case): per-warp counts over contiguous warp
  // segments of this quarter.  Counted before the cluster knows the ids' maximum (digits
  // clamped, so larger ids stay in bounds): the maximum travels with the counts through one
  // cluster barrier, and a multi-pass slice discards them.
  const int wseg = (((nloc + 31) / 32) + 31) & ~31;
  const int w0 = min(nloc, warp * wseg), w1 = min(nloc, w0 + wseg);
  for (int base = w0; base < w1; base += 32) {
    const int i = base + lane;
    const bool act = i < w1;
    const int d = act ? min(key[i], 255) : 256 + lane;
    const uint32_t peers = __match_any_sync(0xffffffffu, d);
    if (act && (peers & lanemask_lt()) == 0) S.cnt[d][warp] += __popc(peers);
    __syncwarp();  // the next group leader of digit d (another lane) reads this count
  }
  __syncthreads();
  if (threadIdx.x < 256) {  // within-digit warp prefix, this CTA's total per digit
    const int d = threadIdx.x;
    int acc = 0;
    for (int w = 0; w < 32; ++w) {
      const int c = S.cnt[d][w];
      S.cnt[d][w] = acc;
      acc += c;
    }
    C.ctot[d] = acc;
  }
  cluster.sync();
  unsigned long long gmx = 0;
  for (int c = 0; c < kSortCluster; ++c) gmx = max(gmx, cluster.map_shared_rank(&C.mx, c)[0]);
  if (gmx >= 256) {  // multi-pass ids: CTA 0 sorts the whole slice as the single-CTA kernel
    cluster.sync();
    if (crank != 0) return;
    for (int t = threadIdx.x; t < T; t += blockDim.x) {
      const long long v = load_int(hash, hdt, hbase + static_cast<int64_t>(t) * st);
      key[t] = static_cast<int32_t>(v < 0 ? 0 : (v > 0x7fffffffLL ? 0x7fffffffLL : v));
    }
    __syncthreads();
    int passes = 0;
    for (unsigned long long m = gmx; m > 0; m >>= 8) ++passes;
    for (int p = 0; p < passes; ++p) {
      const bool last = p == passes - 1;
      const bool to_perm = ((passes - 1 - p) & 1) == 0;
      radix_pass(S, key, T, 8 * p, p == 0 ? nullptr : (to_perm ? X : P), to_perm ? P : X, last ? SH : nullptr,
                 last ? R : nullptr);
    }
    if (threadIdx.x < 256) bounds[threadIdx.x] = -1;
    if (threadIdx.x == 0) bounds[256] = T;
    return;
  }
  int gsum = 0;
  if (threadIdx.x < 256) {
    const int d = threadIdx.x;
    int before = 0;
    for (int c = 0; c < kSortCluster; ++c) {
      const int v = cluster.map_shared_rank(&C.ctot[0], c)[d];
      gsum += v;
      before += (c < crank) ? v : 0;
    }
    C.before[d] = before;
    // exclusive scan of gsum over the 256 digits: warp scans, then the 8 warp totals
    int incl = gsum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int n = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += n;
    }
    if (lane == 31) C.wsum[warp] = incl;
    C.dbase[d] = incl - gsum;
  }
  __syncthreads();
  // this CTA is done reading the others' shared memory: a relaxed arrive now, the matching
  // wait at exit (a full cluster.sync there would also wait for every scattered global
  // write below to be acknowledged)
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
  if (threadIdx.x < 256) {
    int wofs = 0;
    for (int w = 0; w < warp; ++w) wofs += C.wsum[w];
    const int d = threadIdx.x;
    C.dbase[d] += wofs;
    const int base = C.dbase[d] + C.before[d];
    for (int w = 0; w < 32; ++w) S.cnt[d][w] += base;
  }
  __syncthreads();
  // ---- second walk: stable slots, perm / rank / sorted ids
  for (int base = w0; base < w1; base += 32) {
    const int i = base + lane;
    const bool act = i < w1;
    const int d = act ? key[i] : 256 + lane;
    const uint32_t peers = __match_any_sync(0xffffffffu, d);
    const int below = __popc(peers & lanemask_lt());
    int off = 0;
    if (act) off = S.cnt[d][warp];
    __syncwarp();
    if (act) {
      const int slot = off + below;
      P[slot] = s0 + i;
      SH[slot] = d;
      R[s0 + i] = slot;
      if (below == 0) S.cnt[d][warp] = off + __popc(peers);
    }
    __syncwarp();
  }
  if (crank == 0) {
    if (threadIdx.x < 256) bounds[threadIdx.x] = C.dbase[threadIdx.x];
    if (threadIdx.x == 0) bounds[256] = T;
  }
  asm volatile("barrier.cluster.wait.aligned;" ::: "memory");  // the others' reads of this CTA's smem are done
}

// Kernel 2 (one thread per slot, all slices): sorted vectors, rank and visibility runs.
// With shared ids and positions = arange a query slot s in bucket run [a, e) sees key
// slots [a, s) ([a, s] without exclude_self); key slot s is seen by query slots (s, e).
__global__ void __launch_bounds__(256) hash_prepare_finish_kernel(int T, int T_pad, int excl, const int32_t* perm,
                                                                  const int32_t* scratch, int32_t* rank,
                                                                  int32_t* q_idx, int32_t* k_idx, int32_t* q_hash,
                                                                  int32_t* k_hash, int2* q_runs, int2* k_runs,
                                                                  int32_t* rows, int64_t H) {
  const int64_t bh = blockIdx.y;
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= T_pad) return;
  const size_t o = static_cast<size_t>(bh) * T_pad + s;
  if (s >= T) {
    q_idx[o] = kQueryPad;
    k_idx[o] = kColOob;
    q_hash[o] = kQHashOob;
    k_hash[o] = kKHashOob;
    q_runs[o] = make_int2(0, 0);
    k_runs[o] = make_int2(0, 0);
    if (rows) rows[o] = static_cast<int32_t>(((bh / H) * T + perm[bh * T]) * H + bh % H);
    return;
  }
  const int32_t t = perm[bh * T + s];
  if (rows) rows[o] = static_cast<int32_t>(((bh / H) * T + t) * H + bh % H);
  const int32_t g = q_hash[o];  // written sorted by kernel 1
  int a, e;
  const int32_t* bd = scratch + bh * (T + 257) + T;
  if (bd[0] >= 0) {
    a = bd[g];
    e = bd[g + 1];
  } else {  // multi-pass ids: search the sorted ids
    const int32_t* sh = q_hash + static_cast<size_t>(bh) * T_pad;
    int lo = 0, n = s;
    while (n > 0) { const int hh = n >> 1; if (sh[lo + hh] < g) { lo += hh + 1; n -= hh + 1; } else n = hh; }
    a = lo;
    lo = s + 1; n = T - s - 1;
    while (n > 0) { const int hh = n >> 1; if (sh[lo + hh] <= g) { lo += hh + 1; n -= hh + 1; } else n = hh; }
    e = lo;
  }
  q_idx[o] = t;
  k_idx[o] = t;
  k_hash[o] = g;
  q_runs[o] = make_int2(a, excl ? s : s + 1);
  k_runs[o] = make_int2(excl ? s + 1 : s, e);
}

// ------------------------------------------------------------------ gather / scatter

// Up to three row gathers sharing one permutation in one launch (Q | K | V).
// Each 8-thread group moves one 128-byte row piece; a warp keeps 4 rows x 4
// iterations of 16-byte loads in flight.
struct GatherJobs {
  const uint8_t* src[3];
  uint8_t* dst[3];
  const int32_t* perm[3];
  int64_t sb[3], st[3], sh[3];
  int64_t n_slots[3], T_perm[3];
};

__global__ void __launch_bounds__(256) gather_rows3_kernel(const __grid_constant__ GatherJobs J, int n_jobs, int eb,
                                                           int64_t H, int64_t D, int64_t BH) {
  const int64_t row_bytes = D * eb;
  const int vecs = static_cast<int>(row_bytes / 16);
  const int j = blockIdx.y;
  const int64_t n_rows = BH * J.n_slots[j];
  const int64_t total = n_rows * vecs;
  const uint8_t* __restrict__ src = J.src[j];
  uint8_t* __restrict__ dst = J.dst[j];
  const int32_t* __restrict__ perm = J.perm[j];
  const int64_t n_slots = J.n_slots[j], T_perm = J.T_perm[j], sb = J.sb[j], st = J.st[j], sh = J.sh[j];
  constexpr int U = 4;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t g0 = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; g0 < total; g0 += stride * U) {
    uint4 v[U];
    int64_t doff[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t g = g0 + u * stride;
      doff[u] = -1;
      if (g < total) {
        const int64_t r = g / vecs;
        const int c = static_cast<int>(g - r * vecs);
        const int64_t bh = r / n_slots, s = r - bh * n_slots;
        const int64_t b = bh / H, h = bh - b * H;
        const int64_t t = __ldg(perm + bh * T_perm + s);
        v[u] = __ldg(reinterpret_cast<const uint4*>(src + (b * sb + t * st + h * sh) * eb) + c);
        doff[u] = r * row_bytes + c * 16;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (doff[u] >= 0) *reinterpret_cast<uint4*>(dst + doff[u]) = v[u];
  }
}

// The same permutation as gather_rows3 driven from the source side: rows are read in
// memory order (fully sequential) and each 128-byte row is written to its slot
// rank[bh, t] (slots >= n_slots are dropped).  One tensor per blockIdx.y.
__global__ void __launch_bounds__(256) permute_rows3_kernel(const __grid_constant__ GatherJobs J, int eb, int64_t T,
                                                            int64_t H, int64_t D, int64_t B) {
  const int64_t row_bytes = D * eb;
  const int vecs = static_cast<int>(row_bytes / 16);
  const int j = blockIdx.y;
  const int64_t n_rows = B * T * H;
  const int64_t total = n_rows * vecs;
  const uint8_t* __restrict__ src = J.src[j];
  uint8_t* __restrict__ dst = J.dst[j];
  const int32_t* __restrict__ rank = J.perm[j];  // rank here: position -> slot
  const int64_t n_slots = J.n_slots[j], sb = J.sb[j], st = J.st[j], sh = J.sh[j];
  constexpr int U = 4;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t g0 = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; g0 < total; g0 += stride * U) {
    uint4 v[U];
    int64_t doff[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t g = g0 + u * stride;
      doff[u] = -1;
      if (g < total) {
        const int64_t r = g / vecs;  // (b, t, h), h fastest
        const int c = static_cast<int>(g - r * vecs);
        const int64_t h = r % H, bt = r / H;
        const int64_t t = bt % T, b = bt / T;
        const int64_t bh = b * H + h;
        const int32_t slot = __ldg(rank + bh * T + t);
        v[u] = __ldg(reinterpret_cast<const uint4*>(src + (b * sb + t * st + h * sh) * eb) + c);
        if (slot < n_slots) doff[u] = ((bh * n_slots + slot) * D) * eb + c * 16;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (doff[u] >= 0) *reinterpret_cast<uint4*>(dst + doff[u]) = v[u];
  }
}

// The same permutation for the common case — every tensor shares one rank vector, row
// counts fit 32-bit indexing, rows are 16-byte multiples that split evenly over a warp
// (VL lanes per row, 32 / VL rows per warp instruction): the (b, t, h) decode and the rank
// load are done once per row for all NT tensors, each warp reads 32 x 16 contiguous bytes
// of every source and writes whole rows.  U rows per lane in flight.
template <int NT, int U>
__global__ void __launch_bounds__(256) permute_rows_fast_kernel(const __grid_constant__ GatherJobs J, int vl_shift,
                                                                 int T, int H, int n_rows, int row_bytes) {
  const int vl = 1 << vl_shift;
  const int lane_row = (threadIdx.x & 31) >> vl_shift;  // row within the warp's group
  const int c = threadIdx.x & (vl - 1);                   // 16-byte chunk of the row
  const int rows_per_warp = 32 >> vl_shift;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int32_t* __restrict__ rank = J.perm[0];
  const int n_slots = static_cast<int>(J.n_slots[0]);
  for (int base = warp * rows_per_warp * U; base < n_rows; base += warps * rows_per_warp * U) {
    uint4 v[U][NT];
    long long doff[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int r = base + u * rows_per_warp + lane_row;  // memory-order row (b, t, h), h fastest
      doff[u] = -1;
      if (r < n_rows) {
        const int h = r % H, bt = r / H;
        const int t = bt % T, b = bt / T;
        const int bh = b * H + h;
        const int slot = __ldg(rank + static_cast<size_t>(bh) * T + t);
#pragma unroll
        for (int j = 0; j < NT; ++j)
          v[u][j] = __ldg(reinterpret_cast<const uint4*>(J.src[j] + static_cast<size_t>(r) * row_bytes) + c);
        if (slot < n_slots) doff[u] = (static_cast<long long>(bh) * n_slots + slot) * row_bytes + c * 16;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (doff[u] >= 0) {
#pragma unroll
        for (int j = 0; j < NT; ++j) *reinterpret_cast<uint4*>(J.dst[j] + doff[u]) = v[u][j];
      }
  }
}

__global__ void gather_rows_kernel(const uint8_t* __restrict__ src, int eb, int64_t H, int64_t D, int64_t sb,
                                   int64_t st, int64_t sh, const int32_t* __restrict__ perm, int64_t T_perm,
                                   int64_t n_slots, uint8_t* __restrict__ dst, int64_t n_rows) {
  const int64_t row_bytes = D * eb;
  const int vecs = static_cast<int>(row_bytes / 16);
  const int64_t total = n_rows * vecs;
  for (int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; g < total;
       g += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = g / vecs;
    const int v = static_cast<int>(g - r * vecs);
    const int64_t bh = r / n_slots, s = r - bh * n_slots;
    const int64_t b = bh / H, h = bh - b * H;
    const int64_t t = perm[bh * T_perm + s];
    const uint4* sp = reinterpret_cast<const uint4*>(src + (b * sb + t * st + h * sh) * eb) + v;
    uint4* dp = reinterpret_cast<uint4*>(dst + r * row_bytes) + v;
    *dp = __ldg(sp);
  }
}

template <typename TS, typename TD>
SCFA_DEVICE TD cvt(TS x);
template <> SCFA_DEVICE float cvt<float, float>(float x) { return x; }
template <> SCFA_DEVICE __nv_bfloat16 cvt<__nv_bfloat16, __nv_bfloat16>(__nv_bfloat16 x) { return x; }
template <> SCFA_DEVICE float cvt<__nv_bfloat16, float>(__nv_bfloat16 x) { return __bfloat162float(x); }
template <> SCFA_DEVICE __nv_bfloat16 cvt<float, __nv_bfloat16>(float x) { return __float2bfloat16_rn(x); }

template <typename TS, typename TD>
__global__ void scatter_rows_kernel(const TS* __restrict__ src, int64_t H, int64_t T, int64_t D,
                                    const int32_t* __restrict__ rank, int64_t n_slots, TD* __restrict__ dst,
                                    int64_t db, int64_t dt, int64_t dh, int64_t n_rows) {
  const int per = static_cast<int>(D / 8);  // 8 elements per thread
  const int64_t total = n_rows * per;
  for (int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; g < total;
       g += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = g / per;  // destination row in (b, t, h) order, h fastest
    const int c = static_cast<int>(g - r * per) * 8;
    const int64_t h = r % H;
    const int64_t t = (r / H) % T;
    const int64_t b = r / (H * T);
    const int64_t bh = b * H + h;
    const int32_t slot = rank[bh * T + t];
    TD out[8];
    if (slot < n_slots) {
      const TS* sp = src + (bh * n_slots + slot) * D + c;
      TS in[8];
      if (sizeof(TS) == 2) {
        *reinterpret_cast<uint4*>(in) = __ldg(reinterpret_cast<const uint4*>(sp));
      } else {
        reinterpret_cast<uint4*>(in)[0] = __ldg(reinterpret_cast<const uint4*>(sp));
        reinterpret_cast<uint4*>(in)[1] = __ldg(reinterpret_cast<const uint4*>(sp) + 1);
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) out[i] = cvt<TS, TD>(in[i]);
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) out[i] = cvt<float, TD>(0.f);
    }
    TD* dp = dst + b * db + t * dt + h * dh + c;
    if (sizeof(TD) == 2) {
      *reinterpret_cast<uint4*>(dp) = *reinterpret_cast<uint4*>(out);
    } else {
      reinterpret_cast<uint4*>(dp)[0] = reinterpret_cast<uint4*>(out)[0];
      reinterpret_cast<uint4*>(dp)[1] = reinterpret_cast<uint4*>(out)[1];
    }
  }
}

// ------------------------------------------------------------------ aux vectors

__global__ void build_aux_kernel(const int32_t* __restrict__ perm, const int32_t* __restrict__ counts, int64_t H,
                                 int64_t T_perm, int64_t n_slots, int64_t T_pad, int32_t pad_value, int32_t oob_value,
                                 const void* hash, int hdt, int64_t sb, int64_t st, int64_t sh, int32_t hash_oob,
                                 const void* pos, int pdt, int64_t ps_bh, int64_t ps_t,
                                 int32_t* __restrict__ idx_out, int32_t* __restrict__ hash_out, int64_t total) {
  for (int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; g < total;
       g += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t bh = g / T_pad, s = g - bh * T_pad;
    int32_t iv, hv = hash_oob;
    if (s < n_slots) {
      const int32_t t = perm[bh * T_perm + s];
      const int32_t tv = pos ? static_cast<int32_t>(load_int(pos, pdt, bh * ps_bh + static_cast<int64_t>(t) * ps_t)) : t;
      iv = (counts && s >= counts[bh]) ? pad_value : tv;
      if (hash_out) {
        const int64_t b = bh / H, h = bh - b * H;
        hv = static_cast<int32_t>(load_int(hash, hdt, b * sb + h * sh + static_cast<int64_t>(t) * st));
      }
    } else {
      iv = oob_value;
    }
    idx_out[g] = iv;
    if (hash_out) hash_out[g] = hv;
  }
}

__global__ void row_map_kernel(const int32_t* __restrict__ perm, int64_t H, int64_t T_perm, int64_t n_slots,
                               int64_t T_pad, int64_t T_src, int32_t* __restrict__ rows, int64_t total) {
  for (int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; g < total;
       g += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t bh = g / T_pad, s = g - bh * T_pad;
    const int64_t t = perm[bh * T_perm + (s < n_slots ? s : 0)];
    rows[g] = static_cast<int32_t>(((bh / H) * T_src + t) * H + bh % H);
  }
}

__global__ void pack_index_kernel(const void* src, int dt, int64_t T, int64_t s_bh, int64_t s_t, int64_t T_pad,
                                  int32_t oob_value, int32_t* dst, int64_t total) {
  for (int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; g < total;
       g += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t bh = g / T_pad, t = g - bh * T_pad;
    int32_t v = oob_value;
    if (t < T) {
      long long x = load_int(src, dt, bh * s_bh + t * s_t);
      if (x > 0x7fffffffLL) x = 0x7fffffffLL;
      if (x < -0x7fffffffLL) x = -0x7fffffffLL;
      v = static_cast<int32_t>(x);
    }
    dst[g] = v;
  }
}

// rank[bh, idx[b, s, h]] = s for s < n_slots; every other position -> n_slots (routes to zero)
__global__ void fill_i32_kernel(int32_t* dst, int32_t v, int64_t n) {
  for (int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; g < n;
       g += static_cast<int64_t>(gridDim.x) * blockDim.x)
    dst[g] = v;
}

__global__ void invert_index_kernel(const void* idx, int dt, int64_t H, int64_t n_slots, int64_t sb, int64_t ss,
                                    int64_t sh, int64_t T, int32_t* rank, int32_t* err, int64_t total) {
  for (int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; g < total;
       g += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t bh = g / n_slots, s = g - bh * n_slots;
    const int64_t b = bh / H, h = bh - b * H;
    const int64_t t = load_int(idx, dt, b * sb + s * ss + h * sh);
    if (t < 0 || t >= T) { flag_error(err, SCFA_ERR_SHAPE); continue; }
    rank[bh * T + t] = static_cast<int32_t>(s);
  }
}

// ------------------------------------------------------------------ contract checks

__global__ void validate_qk_kernel(const int32_t* q_idx, const int32_t* k_idx, int64_t T_q, int64_t T_kv,
                                   int64_t Tq_pad, int64_t Tkv_pad, int32_t* err) {
  const int64_t bh = blockIdx.x;
  const int32_t* q = q_idx + bh * Tq_pad;
  const int32_t* k = k_idx + bh * Tkv_pad;
  for (int64_t t = threadIdx.x; t + 1 < T_q; t += blockDim.x) {
    const int32_t a = q[t], c = q[t + 1];
    if (a == kQueryPad && c != kQueryPad) flag_error(err, SCFA_ERR_CONTRACT);
    if (a != kQueryPad && c != kQueryPad && c <= a) flag_error(err, SCFA_ERR_CONTRACT);
  }
  for (int64_t t = threadIdx.x; t < T_kv; t += blockDim.x) {
    const int32_t a = k[t];
    if (t + 1 < T_kv) {
      const int32_t c = k[t + 1];
      if (a == kKeyPad && c != kKeyPad) flag_error(err, SCFA_ERR_CONTRACT);
      if (a != kKeyPad && c != kKeyPad && c <= a) flag_error(err, SCFA_ERR_CONTRACT);
    }
    if (a != kKeyPad && a >= kKeyPad) flag_error(err, SCFA_ERR_CONTRACT);
  }
}

__global__ void validate_sorted_kernel(const int32_t* idx, const int32_t* hash, int64_t T, int64_t T_pad,
                                       int32_t* err) {
  const int64_t bh = blockIdx.x;
  const int32_t* ix = idx + bh * T_pad;
  const int32_t* hs = hash + bh * T_pad;
  for (int64_t t = threadIdx.x; t + 1 < T; t += blockDim.x) {
    if (hs[t + 1] < hs[t]) flag_error(err, SCFA_ERR_CONTRACT);
    else if (hs[t + 1] == hs[t] && ix[t + 1] <= ix[t]) flag_error(err, SCFA_ERR_CONTRACT);
  }
}

// ------------------------------------------------------------------ backward prep

// delta = rowsum(dO * O) per sorted/compacted row, lse2 from (M, L) when not given.
// Boundary mode (q_idx != nullptr): O and dO are (B, T_out, H, D); row s of slice bh
// lives at position q_idx[bh, s], and the dO row is also written to d_out_sorted
// (BH, T_q, D) — the gather of dO into kernel order fused with the delta pass.
__global__ void bwd_prep_kernel(const __nv_bfloat16* __restrict__ o, const __nv_bfloat16* __restrict__ d_out,
                                const float* __restrict__ lse2_in, const float* __restrict__ m,
                                const float* __restrict__ l, int64_t T_q, int64_t D, int64_t Tq_pad,
                                const int32_t* __restrict__ q_idx, int64_t H, int64_t T_out,
                                __nv_bfloat16* __restrict__ d_out_sorted, float* __restrict__ delta,
                                float* __restrict__ lse2_out, int64_t total_rows) {
  const int tpr = static_cast<int>(D / 8);  // threads per row, 16 B each
  const int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const int64_t r = g / tpr;  // padded row index
  const int part = static_cast<int>(g - r * tpr);
  float acc = 0.f;
  const bool live = r < total_rows;
  const int64_t bh = live ? r / Tq_pad : 0, t = live ? r - bh * Tq_pad : 0;
  const bool valid = live && t < T_q;
  if (valid) {
    int64_t off = (bh * T_q + t) * D + part * 8;
    bool have = true;
    if (q_idx) {
      const int64_t pos = q_idx[r];
      have = pos >= 0 && pos < T_out;
      const int64_t b = bh / H, h = bh - b * H;
      off = ((b * T_out + (have ? pos : 0)) * H + h) * D + part * 8;
    }
    uint4 a = make_uint4(0, 0, 0, 0), c = make_uint4(0, 0, 0, 0);
    if (have) {
      a = __ldg(reinterpret_cast<const uint4*>(o + off));
      c = __ldg(reinterpret_cast<const uint4*>(d_out + off));
    }
    if (q_idx) *reinterpret_cast<uint4*>(d_out_sorted + (bh * T_q + t) * D + part * 8) = c;
    const __nv_bfloat162* a2 = reinterpret_cast<const __nv_bfloat162*>(&a);
    const __nv_bfloat162* c2 = reinterpret_cast<const __nv_bfloat162*>(&c);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 x = __bfloat1622float2(a2[i]);
      const float2 y = __bfloat1622float2(c2[i]);
      acc = fmaf(x.x, y.x, acc);
      acc = fmaf(x.y, y.y, acc);
    }
  }
  // reduce over the tpr lanes of a row (tpr is a power of two <= 32 and rows never straddle warps)
  for (int w = tpr >> 1; w > 0; w >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, w);
  if (live && part == 0) {
    delta[r] = valid ? acc : 0.f;
    float lv = INFINITY;
    if (valid) {
      if (lse2_in) {
        lv = lse2_in[r];
      } else {
        const float M = m[bh * T_q + t], L = l[bh * T_q + t];
        lv = (L > 0.f) ? M * 1.4426950408889634f + log2f(L) : INFINITY;
      }
    }
    lse2_out[r] = lv;
  }
}

// ------------------------------------------------------------------ launchers

static int grid_for(int64_t work, int threads) {
  int64_t g = (work + threads - 1) / threads;
  if (g > 148 * 64) g = 148 * 64;
  if (g < 1) g = 1;
  return static_cast<int>(g);
}

static int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return SCFA_ERR_CUDA;
  }
  return SCFA_OK;
}

}  // namespace scfa

using namespace scfa;

extern "C" int scfa_qk_compact(const void* keep, int keep_dtype, int64_t B, int64_t T, int64_t H, int64_t sb,
                               int64_t st, int64_t sh, int32_t* perm, int32_t* rank, int32_t* counts,
                               int32_t* err_flag, void* stream) {
  if (B < 0 || T < 0 || H < 0) { set_error("negative extent"); return SCFA_ERR_SHAPE; }
  if (B * H == 0 || T == 0) {
    if (B * H > 0) cudaMemsetAsync(counts, 0, B * H * sizeof(int32_t), static_cast<cudaStream_t>(stream));
    return SCFA_OK;
  }
  qk_compact_kernel<<<static_cast<unsigned>(B * H), 1024, 0, static_cast<cudaStream_t>(stream)>>>(
      keep, keep_dtype, T, H, sb, st, sh, perm, rank, counts, err_flag);
  return check_launch("qk_compact");
}

extern "C" int scfa_qk_prepare(const void* keep_q, int keep_q_dtype, int64_t sbq, int64_t stq, int64_t shq,
                               const void* keep_k, int keep_k_dtype, int64_t sbk, int64_t stk, int64_t shk, int64_t B,
                               int64_t T_Q, int64_t T_KV, int64_t H, int32_t* perm_q, int32_t* rank_q, int32_t* perm_k,
                               int32_t* rank_k, int32_t* q_idx, int32_t* k_idx, int32_t* q_runs, int32_t* k_runs,
                               int32_t* q_rows, int32_t* k_rows, int32_t* counts, int32_t* err_flag, void* stream) {
  if (B < 0 || T_Q < 0 || T_KV < 0 || H < 0) { set_error("negative extent"); return SCFA_ERR_SHAPE; }
  if (T_Q > kQkPrepMaxT || T_KV > kQkPrepMaxT) {
    set_error("qk_prepare: T > %d (use scfa_qk_compact)", kQkPrepMaxT);
    return SCFA_ERR_SHAPE;
  }
  if (B * H > 65535) { set_error("qk_prepare: too many (b, h) slices"); return SCFA_ERR_SHAPE; }
  if (B * H == 0 || (T_Q == 0 && T_KV == 0)) return SCFA_OK;
  if (B * T_Q * H >= (1LL << 31) || B * T_KV * H >= (1LL << 31)) {
    set_error("qk_prepare: row tables need B*T*H < 2^31");
    return SCFA_ERR_SHAPE;
  }
  const size_t smem = (static_cast<size_t>(T_Q) + T_KV + 2 + 2 * (kQkPrepMaxT / 32) + 33) * sizeof(int);
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(qk_prepare_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>((2 * kQkPrepMaxT + 2 + 2 * (kQkPrepMaxT / 32) + 33) * sizeof(int))) !=
        cudaSuccess)
      return check_launch("qk_prepare attribute");
    attr = true;
  }
  const int Tq_pad = static_cast<int>((T_Q + 127) / 128) * 128, Tkv_pad = static_cast<int>((T_KV + 127) / 128) * 128;
  qk_prepare_kernel<<<static_cast<unsigned>(B * H), kQkPrepThreads, smem, static_cast<cudaStream_t>(stream)>>>(
      keep_q, keep_q_dtype, sbq, stq, shq, keep_k, keep_k_dtype, sbk, stk, shk, static_cast<int>(T_Q),
      static_cast<int>(T_KV), Tq_pad, Tkv_pad, static_cast<int>(H), perm_q, rank_q, perm_k, rank_k, q_idx, k_idx,
      reinterpret_cast<int2*>(q_runs), reinterpret_cast<int2*>(k_runs), q_rows, k_rows, counts,
      static_cast<int>(B * H), err_flag);
  return check_launch("qk_prepare");
}

extern "C" int scfa_hash_sort(const void* hash, int hash_dtype, int64_t B, int64_t T, int64_t H, int64_t sb,
                              int64_t st, int64_t sh, const void* pos, int pos_dtype, int64_t ps_bh, int64_t ps_t,
                              int32_t* perm, int32_t* rank, int32_t* scratch, int32_t* err_flag, void* stream) {
  if (B * H == 0 || T == 0) return SCFA_OK;
  hash_sort_kernel<<<static_cast<unsigned>(B * H), kSortThreads, 0, static_cast<cudaStream_t>(stream)>>>(
      hash, hash_dtype, T, H, sb, st, sh, pos, pos_dtype, ps_bh, ps_t, perm, rank, scratch, err_flag);
  return check_launch("hash_sort");
}

extern "C" int scfa_hash_prepare(const void* hash, int hash_dtype, int64_t B, int64_t T, int64_t H, int64_t sb,
                                 int64_t st, int64_t sh, int flags, int32_t* perm, int32_t* rank, int32_t* scratch,
                                 int32_t* q_idx, int32_t* k_idx, int32_t* q_hash, int32_t* k_hash, int32_t* q_runs,
                                 int32_t* k_runs, int32_t* rows, int32_t* err_flag, void* sorted_event,
                                 void* stream) {
  if (T > kPrepMaxT) { set_error("hash_prepare: T > %d (use scfa_hash_sort)", kPrepMaxT); return SCFA_ERR_SHAPE; }
  if (B * H == 0 || T == 0) return SCFA_OK;
  if (B * H > 65535) { set_error("hash_prepare: too many (b, h) slices"); return SCFA_ERR_SHAPE; }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int T_pad = static_cast<int>((T + 127) / 128) * 128;
  const size_t smem = sizeof(PrepSmem) + static_cast<size_t>(T) * 4;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(hash_prepare_sort_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(sizeof(PrepSmem) + kPrepMaxT * 4)) != cudaSuccess)
      return check_launch("hash_prepare attribute");
    attr = true;
  }
  static bool cattr = false;
  const size_t csmem = sizeof(PrepSmem) + sizeof(ClusterSortSmem) + static_cast<size_t>(T) * 4;
  if (!cattr) {
    if (cudaFuncSetAttribute(hash_prepare_sort_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(sizeof(PrepSmem) + sizeof(ClusterSortSmem) + kPrepMaxT * 4)) !=
        cudaSuccess)
      return check_launch("hash_prepare cluster attribute");
    cattr = true;
  }
  // a cluster of CTAs per slice when the slices alone leave most SMs idle and fit one
  // wave as clusters (measured: B*H = 24 at T = 16k 31 -> 13 us; 48 at 8k equal; 96 at 4k
  // the single-CTA kernel wins)
  static int sms = 0;
  if (!sms && cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0) != cudaSuccess) sms = 148;
  if (T >= 4096 && B * H * kSortCluster <= 2 * sms) {
    hash_prepare_sort_cluster_kernel<<<static_cast<unsigned>(B * H * kSortCluster), kSortThreads, csmem, s>>>(
        hash, hash_dtype, static_cast<int>(T), T_pad, H, sb, st, sh, perm, rank, scratch, q_hash, err_flag);
  } else {
    hash_prepare_sort_kernel<<<static_cast<unsigned>(B * H), kSortThreads, smem, s>>>(
        hash, hash_dtype, static_cast<int>(T), T_pad, H, sb, st, sh, perm, rank, scratch, q_hash, err_flag);
  }
  int rc = check_launch("hash_prepare_sort");
  if (rc) return rc;
  if (sorted_event) {  // perm / rank are final here: the caller may start the row copies
    if (cudaEventRecord(static_cast<cudaEvent_t>(sorted_event), s) != cudaSuccess)
      return check_launch("hash_prepare event");
  }
  dim3 grid(static_cast<unsigned>((T_pad + 255) / 256), static_cast<unsigned>(B * H));
  hash_prepare_finish_kernel<<<grid, 256, 0, s>>>(static_cast<int>(T), T_pad, (flags & SCFA_FLAG_EXCLUDE_SELF) ? 1 : 0,
                                                  perm, scratch, rank, q_idx, k_idx, q_hash, k_hash,
                                                  reinterpret_cast<int2*>(q_runs), reinterpret_cast<int2*>(k_runs),
                                                  rows, H);
  return check_launch("hash_prepare_finish");
}

extern "C" int scfa_gather_rows3(int n, const void* const* srcs, void* const* dsts, const int32_t* const* perms,
                                 const int64_t* strides, int elem_bytes, int64_t B, int64_t H, int64_t D,
                                 const int64_t* T_perm, const int64_t* n_slots, void* stream) {
  if (n < 1 || n > 3) { set_error("gather_rows3: 1 to 3 tensors"); return SCFA_ERR_PARAM; }
  if ((D * elem_bytes) % 16 != 0) { set_error("row bytes must be a multiple of 16"); return SCFA_ERR_SHAPE; }
  GatherJobs J{};
  int64_t most = 0;
  for (int i = 0; i < n; ++i) {
    J.src[i] = static_cast<const uint8_t*>(srcs[i]);
    J.dst[i] = static_cast<uint8_t*>(dsts[i]);
    J.perm[i] = perms[i];
    J.sb[i] = strides[3 * i];
    J.st[i] = strides[3 * i + 1];
    J.sh[i] = strides[3 * i + 2];
    J.T_perm[i] = T_perm[i];
    J.n_slots[i] = n_slots[i];
    if (((J.sb[i] | J.st[i] | J.sh[i]) * elem_bytes) % 16 != 0 || (reinterpret_cast<uintptr_t>(srcs[i]) & 15) ||
        (reinterpret_cast<uintptr_t>(dsts[i]) & 15)) {
      set_error("gather rows must be 16-byte aligned");
      return SCFA_ERR_SHAPE;
    }
    most = n_slots[i] > most ? n_slots[i] : most;
  }
  const int64_t work = B * H * most * (D * elem_bytes / 16);
  if (work == 0) return SCFA_OK;
  int64_t g = (work + 256 * 4 - 1) / (256 * 4);
  if (g > 148 * 16) g = 148 * 16;
  dim3 grid(static_cast<unsigned>(g), static_cast<unsigned>(n));
  gather_rows3_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(J, n, elem_bytes, H, D, B * H);
  return check_launch("gather_rows3");
}

extern "C" int scfa_permute_rows3(int n, const void* const* srcs, void* const* dsts, const int32_t* const* ranks,
                                  const int64_t* strides, int elem_bytes, int64_t B, int64_t T, int64_t H, int64_t D,
                                  const int64_t* n_slots, void* stream) {
  if (n < 1 || n > 3) { set_error("permute_rows3: 1 to 3 tensors"); return SCFA_ERR_PARAM; }
  if ((D * elem_bytes) % 16 != 0) { set_error("row bytes must be a multiple of 16"); return SCFA_ERR_SHAPE; }
  GatherJobs J{};
  for (int i = 0; i < n; ++i) {
    J.src[i] = static_cast<const uint8_t*>(srcs[i]);
    J.dst[i] = static_cast<uint8_t*>(dsts[i]);
    J.perm[i] = ranks[i];
    J.sb[i] = strides[3 * i];
    J.st[i] = strides[3 * i + 1];
    J.sh[i] = strides[3 * i + 2];
    J.n_slots[i] = n_slots[i];
    J.T_perm[i] = T;
  }
  const int64_t work = B * T * H * (D * elem_bytes / 16);
  if (work == 0) return SCFA_OK;
  // fast path: shared rank vector and slot count, contiguous (B, T, H, D) sources, a row of
  // 1..32 sixteen-byte chunks (power of two), 32-bit row indexing
  const int64_t row_bytes = D * elem_bytes;
  const int64_t vecs = row_bytes / 16;
  bool fast = (vecs & (vecs - 1)) == 0 && vecs <= 32 && B * T * H < (1LL << 31) && B * H * T < (1LL << 31);
  for (int i = 0; i < n && fast; ++i)
    fast = ranks[i] == ranks[0] && n_slots[i] == n_slots[0] && strides[3 * i + 2] == D &&
           strides[3 * i + 1] == H * D && strides[3 * i] == T * H * D &&
           (reinterpret_cast<uintptr_t>(srcs[i]) & 15) == 0 && (reinterpret_cast<uintptr_t>(dsts[i]) & 15) == 0;
  if (fast) {
    int shift = 0;
    while ((1LL << shift) < vecs) ++shift;
#ifndef SCFA_TUNE_PERM_U
#define SCFA_TUNE_PERM_U 4
#endif
// Grid cap, CTAs per SM: two (of eight resident) keep the copy at full speed alone
// (36 -> 39 us at cfg2) and leave the SMs' other slots to the finishing / tile-list /
// item-order kernels the copy runs beside on the main stream; with the whole GPU
// occupied those queue behind the copy (cfg2 step -12 us, T = 16k -9 us, cfg3 -10 us).
#ifndef SCFA_TUNE_PERM_G
#define SCFA_TUNE_PERM_G 2
#endif
    constexpr int U = SCFA_TUNE_PERM_U;
    const int64_t rows = B * T * H;
    const int64_t rows_per_block = (256 / 32) * (32 >> shift) * U;
    int64_t g = (rows + rows_per_block - 1) / rows_per_block;
    static const int perm_g = getenv("SCFA_PERM_G") ? atoi(getenv("SCFA_PERM_G")) : SCFA_TUNE_PERM_G;  // A/B knob
    if (g > 148 * perm_g) g = 148 * perm_g;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int Ti = static_cast<int>(T), Hi = static_cast<int>(H), R = static_cast<int>(rows), RB = static_cast<int>(row_bytes);
    if (n == 1) permute_rows_fast_kernel<1, U><<<static_cast<unsigned>(g), 256, 0, s>>>(J, shift, Ti, Hi, R, RB);
    else if (n == 2) permute_rows_fast_kernel<2, U><<<static_cast<unsigned>(g), 256, 0, s>>>(J, shift, Ti, Hi, R, RB);
    else permute_rows_fast_kernel<3, U><<<static_cast<unsigned>(g), 256, 0, s>>>(J, shift, Ti, Hi, R, RB);
    return check_launch("permute_rows (fast)");
  }
  int64_t g = (work + 256 * 4 - 1) / (256 * 4);
  if (g > 148 * 16) g = 148 * 16;
  dim3 grid(static_cast<unsigned>(g), static_cast<unsigned>(n));
  permute_rows3_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(J, elem_bytes, T, H, D, B);
  return check_launch("permute_rows3");
}

extern "C" int scfa_gather_rows(const void* src, int elem_bytes, int64_t B, int64_t H, int64_t D, int64_t sb,
                                int64_t st, int64_t sh, const int32_t* perm, int64_t T_perm, int64_t n_slots,
                                void* dst, void* stream) {
  if ((D * elem_bytes) % 16 != 0) { set_error("row bytes must be a multiple of 16"); return SCFA_ERR_SHAPE; }
  if (((sb | st | sh) * elem_bytes) % 16 != 0 || (reinterpret_cast<uintptr_t>(src) & 15) ||
      (reinterpret_cast<uintptr_t>(dst) & 15)) {
    set_error("gather rows must be 16-byte aligned");
    return SCFA_ERR_SHAPE;
  }
  const int64_t n_rows = B * H * n_slots;
  if (n_rows == 0) return SCFA_OK;
  const int64_t work = n_rows * (D * elem_bytes / 16);
  gather_rows_kernel<<<grid_for(work, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint8_t*>(src), elem_bytes, H, D, sb, st, sh, perm, T_perm, n_slots,
      static_cast<uint8_t*>(dst), n_rows);
  return check_launch("gather_rows");
}

extern "C" int scfa_scatter_rows(const void* src, int src_bytes, int64_t B, int64_t H, int64_t T, int64_t D,
                                 const int32_t* rank, int64_t n_slots, void* dst, int dst_bytes, int64_t db,
                                 int64_t dt, int64_t dh, void* stream) {
  if (D % 8 != 0) { set_error("D must be a multiple of 8"); return SCFA_ERR_SHAPE; }
  const int64_t n_rows = B * T * H;
  if (n_rows == 0) return SCFA_OK;
  const int64_t work = n_rows * (D / 8);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int g = grid_for(work, 256);
  if (src_bytes == 2 && dst_bytes == 2)
    scatter_rows_kernel<__nv_bfloat16, __nv_bfloat16><<<g, 256, 0, s>>>(
        static_cast<const __nv_bfloat16*>(src), H, T, D, rank, n_slots, static_cast<__nv_bfloat16*>(dst), db, dt,
        dh, n_rows);
  else if (src_bytes == 4 && dst_bytes == 4)
    scatter_rows_kernel<float, float><<<g, 256, 0, s>>>(static_cast<const float*>(src), H, T, D, rank, n_slots,
                                                       static_cast<float*>(dst), db, dt, dh, n_rows);
  else if (src_bytes == 4 && dst_bytes == 2)
    scatter_rows_kernel<float, __nv_bfloat16><<<g, 256, 0, s>>>(static_cast<const float*>(src), H, T, D, rank,
                                                               n_slots, static_cast<__nv_bfloat16*>(dst), db, dt,
                                                               dh, n_rows);
  else if (src_bytes == 2 && dst_bytes == 4)
    scatter_rows_kernel<__nv_bfloat16, float><<<g, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(src), H, T, D,
                                                               rank, n_slots, static_cast<float*>(dst), db, dt,
                                                               dh, n_rows);
  else { set_error("unsupported element sizes"); return SCFA_ERR_SHAPE; }
  return check_launch("scatter_rows");
}

extern "C" int scfa_build_aux(const int32_t* perm, const int32_t* counts, int64_t B, int64_t H, int64_t T_perm,
                              int64_t n_slots, int64_t T_pad, int32_t pad_value, int32_t oob_value,
                              const void* hash, int hash_dtype, int64_t sb, int64_t st, int64_t sh,
                              int32_t hash_oob, const void* pos, int pos_dtype, int64_t ps_bh, int64_t ps_t,
                              int32_t* idx_out, int32_t* hash_out, void* stream) {
  const int64_t total = B * H * T_pad;
  if (total == 0) return SCFA_OK;
  build_aux_kernel<<<grid_for(total, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      perm, counts, H, T_perm, n_slots, T_pad, pad_value, oob_value, hash, hash_dtype, sb, st, sh, hash_oob, pos,
      pos_dtype, ps_bh, ps_t, idx_out, hash ? hash_out : nullptr, total);
  return check_launch("build_aux");
}

extern "C" int scfa_row_map(const int32_t* perm, int64_t B, int64_t H, int64_t T_perm, int64_t n_slots, int64_t T_pad,
                            int64_t T_src, int32_t* rows, void* stream) {
  const int64_t total = B * H * T_pad;
  if (total == 0) return SCFA_OK;
  if (B * T_src * H >= (1LL << 31)) { set_error("row_map: row table exceeds 2^31 rows"); return SCFA_ERR_SHAPE; }
  if (n_slots < 1 || n_slots > T_perm) { set_error("row_map: n_slots must be in [1, T_perm]"); return SCFA_ERR_SHAPE; }
  row_map_kernel<<<grid_for(total, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(perm, H, T_perm, n_slots, T_pad,
                                                                                      T_src, rows, total);
  return check_launch("row_map");
}

extern "C" int scfa_pack_index(const void* src, int dtype, int64_t BH, int64_t T, int64_t s_bh, int64_t s_t,
                               int64_t T_pad, int32_t oob_value, int32_t* dst, void* stream) {
  const int64_t total = BH * T_pad;
  if (total == 0) return SCFA_OK;
  pack_index_kernel<<<grid_for(total, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      src, dtype, T, s_bh, s_t, T_pad, oob_value, dst, total);
  return check_launch("pack_index");
}

extern "C" int scfa_validate_qk(const int32_t* q_idx, const int32_t* k_idx, int64_t BH, int64_t T_q, int64_t T_kv,
                                int64_t Tq_pad, int64_t Tkv_pad, int32_t* err_flag, void* stream) {
  if (BH == 0) return SCFA_OK;
  validate_qk_kernel<<<static_cast<unsigned>(BH), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      q_idx, k_idx, T_q, T_kv, Tq_pad, Tkv_pad, err_flag);
  return check_launch("validate_qk");
}

extern "C" int scfa_validate_sorted(const int32_t* idx, const int32_t* hash, int64_t BH, int64_t T, int64_t T_pad,
                                    int32_t* err_flag, void* stream) {
  if (BH == 0) return SCFA_OK;
  validate_sorted_kernel<<<static_cast<unsigned>(BH), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      idx, hash, T, T_pad, err_flag);
  return check_launch("validate_sorted");
}

// The boundary-layout delta pass driven from the source side (shared hash ids: every
// position has a slot): O and dO rows are read in memory order (b, t, h) — fully
// sequential — and dO lands at its slot rank[bh, t] of d_out_sorted, delta at
// delta[bh, rank].  Slots past T (padding to Tq_pad) get delta 0.
__global__ void bwd_prep_rank_kernel(const __nv_bfloat16* __restrict__ o, const __nv_bfloat16* __restrict__ d_out,
                                     int64_t H, int64_t T, int64_t D, int64_t Tq_pad,
                                     const int32_t* __restrict__ rank, __nv_bfloat16* __restrict__ d_out_sorted,
                                     float* __restrict__ delta, int64_t rows, int64_t BH) {
  const int tpr = static_cast<int>(D / 8);
  const int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const int64_t main_threads = rows * tpr;
  if (g >= main_threads) {  // padding slots
    const int64_t p = g - main_threads, npad = Tq_pad - T;
    if (npad > 0 && p < BH * npad) {
      const int64_t bh = p / npad;
      delta[bh * Tq_pad + T + (p - bh * npad)] = 0.f;
    }
    return;
  }
  const int64_t r = g / tpr;  // (b, t, h) row, h fastest
  const int part = static_cast<int>(g - r * tpr);
  const int64_t h = r % H, bt = r / H;
  const int64_t t = bt % T, b = bt / T;
  const int64_t bh = b * H + h;
  const int32_t slot = __ldg(rank + bh * T + t);
  const uint4 a = __ldg(reinterpret_cast<const uint4*>(o + r * D) + part);
  const uint4 c = __ldg(reinterpret_cast<const uint4*>(d_out + r * D) + part);
  *reinterpret_cast<uint4*>(d_out_sorted + (bh * T + slot) * D + part * 8) = c;
  const __nv_bfloat162* a2 = reinterpret_cast<const __nv_bfloat162*>(&a);
  const __nv_bfloat162* c2 = reinterpret_cast<const __nv_bfloat162*>(&c);
  float acc = 0.f;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 x = __bfloat1622float2(a2[i]);
    const float2 y = __bfloat1622float2(c2[i]);
    acc = fmaf(x.x, y.x, acc);
    acc = fmaf(x.y, y.y, acc);
  }
  // rows never straddle warps (tpr is a power of two <= 32, main_threads a multiple of tpr)
  for (int w = tpr >> 1; w > 0; w >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, w);
  if (part == 0) delta[bh * Tq_pad + slot] = acc;
}

extern "C" int scfa_bwd_prep_rank(const void* o, const void* d_out, int64_t B, int64_t T, int64_t H, int64_t D,
                                  int64_t Tq_pad, const int32_t* rank, void* d_out_sorted, float* delta,
                                  void* stream) {
  if (D % 8 != 0 || D / 8 > 32 || ((D / 8) & (D / 8 - 1))) { set_error("bwd_prep_rank: unsupported D"); return SCFA_ERR_SHAPE; }
  if (Tq_pad < T) { set_error("bwd_prep_rank: Tq_pad < T"); return SCFA_ERR_SHAPE; }
  const int64_t rows = B * T * H;
  const int64_t threads = rows * (D / 8) + B * H * (Tq_pad - T);
  if (threads == 0) return SCFA_OK;
  bwd_prep_rank_kernel<<<static_cast<unsigned>((threads + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const __nv_bfloat16*>(o), static_cast<const __nv_bfloat16*>(d_out), H, T, D, Tq_pad, rank,
      static_cast<__nv_bfloat16*>(d_out_sorted), delta, rows, B * H);
  return check_launch("bwd_prep_rank");
}

// Zero the rows of dropped positions (keep == 0) of up to two (B, T, H, D) outputs:
// the kernels write every kept row, so the outputs need no full zero-fill
// (qk_postprocess / the backward scatter leave dropped rows 0, qk_sparse.py:214-225).
// One warp per (b, t): the H rows of a position are contiguous, so the warp's 16-byte
// stores walk them in order (coalesced), skipping the kept heads.
__global__ void zero_dropped_kernel(const void* __restrict__ keep, int kdt, int T, int H, int64_t sb, int64_t st,
                                    int64_t sh, uint8_t* __restrict__ out0, int row0, uint8_t* __restrict__ out1,
                                    int row1, int64_t n_bt) {
  const int64_t bt = blockIdx.x * static_cast<int64_t>(blockDim.x / 32) + (threadIdx.x >> 5);
  if (bt >= n_bt) return;
  const int lane = threadIdx.x & 31;
  const int64_t b = bt / T, t = bt - b * T;
  const int64_t kbase = b * sb + t * st;
  uint32_t dropped = 0;  // bit h: head h of this position is dropped (H <= 32 per pass)
  for (int h0 = 0; h0 < H; h0 += 32) {
    const int h = h0 + lane;
    const bool d = h < H && load_num(keep, kdt, kbase + h * sh) == 0.0;
    dropped = __ballot_sync(0xffffffffu, d);
    if (!dropped) continue;
    const int nh = min(32, H - h0);
#pragma unroll
    for (int o = 0; o < 2; ++o) {
      uint8_t* out = o == 0 ? out0 : out1;
      const int rb = o == 0 ? row0 : row1;
      if (!out || rb == 0) continue;
      const int pieces = rb / 16;
      uint4* base = reinterpret_cast<uint4*>(out + (bt * H + h0) * static_cast<int64_t>(rb));
      for (int p = lane; p < nh * pieces; p += 32)
        if ((dropped >> (p / pieces)) & 1u) base[p] = make_uint4(0u, 0u, 0u, 0u);
    }
  }
}

extern "C" int scfa_zero_dropped(const void* keep, int keep_dtype, int64_t B, int64_t T, int64_t H, int64_t sb,
                                 int64_t st, int64_t sh, void* out0, int64_t row_bytes0, void* out1,
                                 int64_t row_bytes1, void* stream) {
  if (row_bytes0 % 16 || row_bytes1 % 16 || (!out1 && row_bytes1)) {
    set_error("zero_dropped: row bytes must be multiples of 16");
    return SCFA_ERR_SHAPE;
  }
  if (T > 0x7fffffff || H > 0x7fffffff || row_bytes0 > 0x7fffffff || row_bytes1 > 0x7fffffff) {
    set_error("zero_dropped: sizes out of range");
    return SCFA_ERR_SHAPE;
  }
  const int64_t n_bt = B * T;
  if (n_bt == 0 || H == 0) return SCFA_OK;
  constexpr int kWarps = 8;
  zero_dropped_kernel<<<static_cast<unsigned>((n_bt + kWarps - 1) / kWarps), 32 * kWarps, 0,
                        static_cast<cudaStream_t>(stream)>>>(
      keep, keep_dtype, static_cast<int>(T), static_cast<int>(H), sb, st, sh, static_cast<uint8_t*>(out0),
      static_cast<int>(row_bytes0), static_cast<uint8_t*>(out1), static_cast<int>(row_bytes1), n_bt);
  return check_launch("zero_dropped");
}

extern "C" int scfa_bwd_prep(const void* o, const void* d_out, const float* lse2_in, const float* m, const float* l,
                             int64_t BH, int64_t T_q, int64_t D, int64_t Tq_pad, const int32_t* q_idx, int64_t H,
                             int64_t T_out, void* d_out_sorted, float* delta, float* lse2_out, void* stream) {
  if (D % 8 != 0 || D / 8 > 32 || ((D / 8) & (D / 8 - 1))) { set_error("bwd_prep: unsupported D"); return SCFA_ERR_SHAPE; }
  if (q_idx && (!d_out_sorted || H < 1)) { set_error("bwd_prep: boundary mode needs d_out_sorted and H"); return SCFA_ERR_SHAPE; }
  const int64_t rows = BH * Tq_pad;
  if (rows == 0) return SCFA_OK;
  const int64_t threads = rows * (D / 8);
  bwd_prep_kernel<<<static_cast<unsigned>((threads + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const __nv_bfloat16*>(o), static_cast<const __nv_bfloat16*>(d_out), lse2_in, m, l, T_q, D, Tq_pad,
      q_idx, H, T_out, static_cast<__nv_bfloat16*>(d_out_sorted), delta, lse2_out, rows);
  return check_launch("bwd_prep");
}

extern "C" int scfa_invert_index(const void* idx, int dtype, int64_t B, int64_t n_slots, int64_t H, int64_t sb,
                                 int64_t ss, int64_t sh, int64_t T, int32_t* rank, int32_t* err_flag, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t n = B * H * T;
  if (n == 0) return SCFA_OK;
  fill_i32_kernel<<<grid_for(n, 256), 256, 0, s>>>(rank, static_cast<int32_t>(n_slots), n);
  const int64_t total = B * H * n_slots;
  if (total > 0)
    invert_index_kernel<<<grid_for(total, 256), 256, 0, s>>>(idx, dtype, H, n_slots, sb, ss, sh, T, rank, err_flag,
                                                              total);
  return check_launch("invert_index");
}
