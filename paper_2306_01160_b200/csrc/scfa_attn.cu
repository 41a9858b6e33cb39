// scfa_attn.cu — tcgen05/TMEM/TMA tile engine for Sparse Causal Flash Attention.
//
// One kernel template runs all three passes of the reference tile loop
// (pkg/src/scfa/_kernel.py:92-193):
//
//   FWD      rows = queries, streamed cols = keys.   S = Q K^T ; P = softmax ; O += P V
//   BWD_DQ   rows = queries, streamed cols = keys.   S, dP = dO V^T ; dS ; dQ += dS K
//   BWD_DKDV rows = keys,    streamed cols = queries. S^T, dP^T ; dV += P^T dO ; dK += dS^T Q
//
// Each CTA owns one 128-row stationary block of one (b, h) slice and walks a
// per-block tile list built by scfa_sched.cu.  The list holds only tiles
// that contain at least one visible (query, key) pair — fully masked tiles
// are skipped, not masked — and flags the tiles whose pairs are all visible
// so that the per-element causal/bucket mask runs only in boundary tiles.
//
// Roles (192 threads):
//   warps 0-3  : one thread per stationary row == TMEM lane.  Online softmax
//                (fwd) or P / dS recompute (bwd), epilogue.
//   warp 4     : TMA producer (stationary tiles once, streamed tiles in an
//                NS-stage mbarrier ring, plus the per-column index/bucket
//                (and lse/delta) vectors via cp.async.bulk).
//   warp 5     : TMEM allocator + single-thread tcgen05.mma issuer.
//
// TMEM (per CTA, 256 columns for D=64 so that two CTAs share an SM):
//   FWD      S fp32 [0,128) (P bf16 aliases [0,64)), O fp32 [128,128+D)
//   BWD_DQ   S [0,64) (dS bf16 aliases [0,32)), dP [64,128), dQ [128,128+D)
//   BWD_DKDV S^T [0,64) (P^T aliases [0,32)), dP^T [64,128) (dS^T aliases
//            [64,96)), dV [128,128+D), dK [128+D,128+2D)
#include "scfa_common.cuh"
#include "scfa_internal.h"

namespace scfa {

enum Mode : int { MODE_FWD = 0, MODE_DQ = 1, MODE_DKDV = 2 };

template <int kMode, int kD>
struct Cfg {
  static constexpr int BM = 128;                             // stationary rows per work item
  static constexpr int BN = (kMode == MODE_FWD) ? 128 : 64;  // streamed rows per tile
  static constexpr int NS = 2;                               // streamed-tile pipeline stages
  static constexpr int NXS = 2;                              // stationary-tile slots (next item prefetch)
  static constexpr int DCH = kD / 64;                        // 128-byte column chunks
  static constexpr int NX = (kMode == MODE_FWD) ? 1 : 2;     // stationary tensors
  static constexpr int NAUX = (kMode == MODE_DKDV) ? 4 : 2;  // per-column vectors
  static constexpr int X_BYTES = BM * kD * 2;
  static constexpr int XSLOT_BYTES = NX * X_BYTES;
  static constexpr int Y_BYTES = BN * kD * 2;
  static constexpr int AUX_BYTES = BN * 4;
  static constexpr int STAGE_BYTES = 2 * Y_BYTES + NAUX * AUX_BYTES;
  // TMEM columns: S (and dP) then accumulators; two accumulator buffers when they fit
  static constexpr int TM_S = 0;
  static constexpr int TM_DP = (kMode == MODE_FWD) ? 0 : BN;
  static constexpr int TM_ACC = 128;
  static constexpr int ACC_COLS = (kMode == MODE_DKDV) ? 2 * kD : kD;  // one buffer (dK/dV: dV then dK)
  static constexpr int NACC = (kMode == MODE_DKDV) ? 1 : 2;
  static constexpr int TM_USED = TM_ACC + NACC * ACC_COLS;
  static constexpr uint32_t TM_COLS = TM_USED <= 256 ? 256 : 512;
  // shared memory carve-up (offsets from a 1024-aligned base)
  static constexpr int OFF_X = 0;
  static constexpr int OFF_STAGE = OFF_X + NXS * XSLOT_BYTES;
  static constexpr int OFF_BAR = OFF_STAGE + NS * STAGE_BYTES;
  static constexpr int N_BARS = 2 + 2 * NXS + 2 * NS + 2 * NACC;
  static constexpr int SMEM_BYTES = OFF_BAR + 8 * N_BARS + 16 + 1024 /*align slack*/;
};

struct AttnArgs {
  int BH, H;
  int T_rows, T_cols;          // true lengths of the stationary / streamed side
  int T_rows_pad, T_cols_pad;  // padded lengths of the aux vectors
  int T_out;                   // boundary-layout output length (out_boundary)
  int out_boundary;            // 1: write rows to (B, T_out, H, D) at their original position
  const int* row_idx;
  const int* row_hash;
  const int* col_idx;
  const int* col_hash;
  const float* lse2;   // (BH, Tq_pad), log2-domain; +inf where no key is visible
  const float* delta;  // (BH, Tq_pad)
  const uint16_t* list;
  const int* list_count;
  int list_stride;
  int n_row_blocks;
  int n_items;
  __nv_bfloat16* out_o;  // FWD
  float* out0;           // FWD: M      DQ: dQ   DKDV: dK
  float* out1;           // FWD: L      DKDV: dV
  float* out_lse2;       // FWD
  float scale_log2;
  float scale;
  int exclude_self;
  int use_hash;
  long long* dbg;   // optional per-tile timestamps (diagnostics)
  int dbg_tiles;
};

// Diagnostics: per-CTA, per-tile clock64 stamps (row thread 0: slots 0-2, MMA lane: 3-7).
#define SCFA_STAMP(k)                                                                         \
  if (args.dbg && threadIdx.x == 0 && tg < args.dbg_tiles)                                   \
    args.dbg[(static_cast<size_t>(blockIdx.x) * args.dbg_tiles + tg) * 8 + (k)] = clock64();
#define SCFA_MSTAMP(k) SCFA_STAMP_MMA(k)
#define SCFA_STAMP_MMA(k)                                                                     \
  if (args.dbg && tg < args.dbg_tiles)                                                       \
    args.dbg[(static_cast<size_t>(blockIdx.x) * args.dbg_tiles + tg) * 8 + (k)] = clock64();

// Work item -> (bh, row block).  Items run heaviest row block first (largest causal
// reach), cycling over heads, and CTAs take items round-robin.
SCFA_DEVICE void decode_item(const AttnArgs& a, int w, int& bh, int& rb) {
  rb = a.n_row_blocks - 1 - w / a.BH;
  bh = w - (w / a.BH) * a.BH;
}

// Output row of stationary row `row` (original position `pos`): engine layout
// (bh, row) or boundary layout (b, pos, h) — the fused inverse scatter.
SCFA_DEVICE bool out_row(const AttnArgs& a, int bh, int row, int pos, size_t& off) {
  if (row >= a.T_rows) return false;
  if (!a.out_boundary) {
    off = static_cast<size_t>(bh) * a.T_rows + row;
    return true;
  }
  if (pos < 0 || pos >= a.T_out) return false;  // pad slots (QUERY_PAD / KEY_PAD)
  const int b = bh / a.H, h = bh - b * a.H;
  off = (static_cast<size_t>(b) * a.T_out + pos) * a.H + h;
  return true;
}

// ---- per-row visibility interval -------------------------------------------------
// Inside one tile the streamed columns are sorted by (bucket, position) (hash) or by
// position (QK / dense), with pads and out-of-range slots at the tail.  The columns a
// stationary row can see therefore form ONE contiguous run [lo, hi): the row's bucket
// run, cut at the causal boundary.  It is found with a few binary searches in shared
// memory per row and tile, and applied as a 32-bit mask per 32 columns (R2P + FSEL).

// first i in [0, n) with a[i] >= x  (a ascending on [0, n))
SCFA_DEVICE int lower_bound(const int* a, int n, int x) {
  int lo = 0;
  while (n > 0) {
    const int h = n >> 1;
    if (a[lo + h] < x) { lo += h + 1; n -= h + 1; } else { n = h; }
  }
  return lo;
}
// first i in [0, n) with a[i] > x
SCFA_DEVICE int upper_bound(const int* a, int n, int x) {
  int lo = 0;
  while (n > 0) {
    const int h = n >> 1;
    if (a[lo + h] <= x) { lo += h + 1; n -= h + 1; } else { n = h; }
  }
  return lo;
}

// rows are queries (fwd, dQ): columns are keys.  visible <=> k_idx <(=) q_idx [and same bucket]
template <int BN>
SCFA_DEVICE void interval_q_rows(const int* kidx, const int* khash, int nv, int qi, int qh, bool excl, bool use_hash,
                                 int& lo, int& hi) {
  if (!use_hash) {  // keys ascending over all BN slots (pads 10^9, out-of-range INT_MAX)
    lo = 0;
    hi = excl ? lower_bound(kidx, BN, qi) : upper_bound(kidx, BN, qi);
  } else {          // valid slots [0, nv) sorted by (bucket, position)
    const int a = lower_bound(khash, nv, qh);
    const int e = a + upper_bound(khash + a, nv - a, qh);
    lo = a;
    hi = a + (excl ? lower_bound(kidx + a, e - a, qi) : upper_bound(kidx + a, e - a, qi));
  }
}

// rows are keys (dK/dV): columns are queries.  visible <=> q_idx >(=) k_idx [and same bucket]
template <int BN>
SCFA_DEVICE void interval_k_rows(const int* qidx, const int* qhash, int nv, int ki, int kh, bool excl, bool use_hash,
                                 int& lo, int& hi) {
  if (!use_hash) {  // real queries ascending, then pads / out-of-range (-1) at the tail
    int nreal = 0, n = BN;
    while (n > 0) {
      const int h = n >> 1;
      if (qidx[nreal + h] >= 0) { nreal += h + 1; n -= h + 1; } else { n = h; }
    }
    lo = excl ? upper_bound(qidx, nreal, ki) : lower_bound(qidx, nreal, ki);
    hi = nreal;
  } else {
    const int a = lower_bound(qhash, nv, kh);
    const int e = a + upper_bound(qhash + a, nv - a, kh);
    lo = a + (excl ? upper_bound(qidx + a, e - a, ki) : lower_bound(qidx + a, e - a, ki));
    hi = e;
  }
}

SCFA_DEVICE uint32_t bits_below(int n) { return n <= 0 ? 0u : (n >= 32 ? 0xffffffffu : ((1u << n) - 1u)); }

// 32-column visibility words of the run [lo, hi)
template <int NW>
SCFA_DEVICE void run_mask(int lo, int hi, uint32_t (&w)[NW]) {
#pragma unroll
  for (int i = 0; i < NW; ++i) w[i] = bits_below(hi - 32 * i) & ~bits_below(lo - 32 * i);
}

template <int kMode, int kD>
__global__ void __launch_bounds__(192, (kD == 64) ? 2 : 1)
    scfa_attn_kernel(const __grid_constant__ CUtensorMap tm_x0, const __grid_constant__ CUtensorMap tm_x1,
                     const __grid_constant__ CUtensorMap tm_y0, const __grid_constant__ CUtensorMap tm_y1,
                     const AttnArgs args) {
  using C = Cfg<kMode, kD>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* bar_s_full = bars + 0;
  uint64_t* bar_p_full = bars + 1;
  uint64_t* bar_x_full = bars + 2;
  uint64_t* bar_x_empty = bar_x_full + C::NXS;
  uint64_t* bar_y_full = bar_x_empty + C::NXS;
  uint64_t* bar_y_empty = bar_y_full + C::NS;
  uint64_t* bar_acc_full = bar_y_empty + C::NS;
  uint64_t* bar_acc_free = bar_acc_full + C::NACC;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + C::OFF_BAR + 8 * C::N_BARS);

  if (threadIdx.x == 0) {
    mbar_init(bar_s_full, 1);
    mbar_init(bar_p_full, 128);
    for (int i = 0; i < C::NXS; ++i) {
      mbar_init(bar_x_full + i, 1);
      mbar_init(bar_x_empty + i, 1);
    }
    for (int i = 0; i < C::NS; ++i) {
      mbar_init(bar_y_full + i, 1);
      mbar_init(bar_y_empty + i, 1);
    }
    for (int i = 0; i < C::NACC; ++i) {
      mbar_init(bar_acc_full + i, 1);
      mbar_init(bar_acc_free + i, 128);
    }
    fence_barrier_init();
  }
  if (warp == 5) tmem_alloc<C::TM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 4) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      tma_prefetch_desc(&tm_x0);
      tma_prefetch_desc(&tm_y0);
      tma_prefetch_desc(&tm_y1);
      if (C::NX == 2) tma_prefetch_desc(&tm_x1);
      int tg = 0, ia = 0;  // global tile counter, non-empty item counter
      for (int w = blockIdx.x; w < args.n_items; w += gridDim.x) {
        int bh, rb;
        decode_item(args, w, bh, rb);
        const int lb = bh * args.n_row_blocks + rb;
        const int n = args.list_count[lb];
        if (n == 0) continue;
        const uint16_t* lst = args.list + static_cast<size_t>(lb) * args.list_stride;
        const int xs = ia % C::NXS;
        if (ia >= C::NXS) mbar_wait(bar_x_empty + xs, ((ia / C::NXS) - 1) & 1);
        uint8_t* xb = smem + C::OFF_X + xs * C::XSLOT_BYTES;
        mbar_arrive_expect_tx(bar_x_full + xs, C::XSLOT_BYTES);
        for (int c = 0; c < C::DCH; ++c) {
          tma_load_3d(xb + c * C::BM * 128, &tm_x0, bar_x_full + xs, c * 64, rb * C::BM, bh);
          if (C::NX == 2) tma_load_3d(xb + C::X_BYTES + c * C::BM * 128, &tm_x1, bar_x_full + xs, c * 64, rb * C::BM, bh);
        }
        for (int t = 0; t < n; ++t, ++tg) {
          const int st = tg % C::NS;
          if (tg >= C::NS) mbar_wait(bar_y_empty + st, ((tg / C::NS) - 1) & 1);
          const int col0 = (lst[t] & 0x7fff) * C::BN;
          uint8_t* stage = smem + C::OFF_STAGE + st * C::STAGE_BYTES;
          mbar_arrive_expect_tx(bar_y_full + st, C::STAGE_BYTES);
          for (int c = 0; c < C::DCH; ++c) {
            tma_load_3d(stage + c * C::BN * 128, &tm_y0, bar_y_full + st, c * 64, col0, bh);
            tma_load_3d(stage + C::Y_BYTES + c * C::BN * 128, &tm_y1, bar_y_full + st, c * 64, col0, bh);
          }
          uint8_t* aux = stage + 2 * C::Y_BYTES;
          const size_t coff = static_cast<size_t>(bh) * args.T_cols_pad + col0;
          bulk_load(aux, args.col_idx + coff, C::AUX_BYTES, bar_y_full + st);
          bulk_load(aux + C::AUX_BYTES, args.col_hash + coff, C::AUX_BYTES, bar_y_full + st);
          if (kMode == MODE_DKDV) {
            bulk_load(aux + 2 * C::AUX_BYTES, args.lse2 + coff, C::AUX_BYTES, bar_y_full + st);
            bulk_load(aux + 3 * C::AUX_BYTES, args.delta + coff, C::AUX_BYTES, bar_y_full + st);
          }
        }
        ++ia;
      }
    }
  } else if (warp == 5) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc_s = make_idesc_bf16(128, C::BN, false, false);
      constexpr uint32_t idesc_acc = make_idesc_bf16(128, kD, false, true);
      int tg = 0, ia = 0;
      for (int w = blockIdx.x; w < args.n_items; w += gridDim.x) {
        int bh, rb;
        decode_item(args, w, bh, rb);
        const int n = args.list_count[bh * args.n_row_blocks + rb];
        if (n == 0) continue;
        const int xs = ia % C::NXS;
        const int ab = ia % C::NACC;
        const uint32_t acc = tmem + C::TM_ACC + ab * C::ACC_COLS;
        const uint32_t x0_addr = smem_u32(smem + C::OFF_X + xs * C::XSLOT_BYTES);
        const uint32_t x1_addr = x0_addr + C::X_BYTES;
        mbar_wait(bar_x_full + xs, (ia / C::NXS) & 1);
        tc_fence_after();
        for (int t = 0; t < n; ++t, ++tg) {
          const int st = tg % C::NS;
          SCFA_MSTAMP(6);
          mbar_wait(bar_y_full + st, (tg / C::NS) & 1);
          SCFA_MSTAMP(7);
          tc_fence_after();
          const uint32_t y0_addr = smem_u32(smem + C::OFF_STAGE + st * C::STAGE_BYTES);
          const uint32_t y1_addr = y0_addr + C::Y_BYTES;
          // S = X0 . Y0^T  (and dP = X1 . Y1^T), K = head dim, both operands K-major.
#pragma unroll
          for (int k = 0; k < kD / 16; ++k) {
            const uint32_t koff = (k & 3) * 32;
            const uint32_t a = x0_addr + (k >> 2) * (C::BM * 128) + koff;
            const uint32_t b = y0_addr + (k >> 2) * (C::BN * 128) + koff;
            umma_ss(tmem + C::TM_S, make_sdesc_sw128(a, 16, 1024), make_sdesc_sw128(b, 16, 1024), idesc_s, k > 0);
          }
          if (kMode != MODE_FWD) {
#pragma unroll
            for (int k = 0; k < kD / 16; ++k) {
              const uint32_t koff = (k & 3) * 32;
              const uint32_t a = x1_addr + (k >> 2) * (C::BM * 128) + koff;
              const uint32_t b = y1_addr + (k >> 2) * (C::BN * 128) + koff;
              umma_ss(tmem + C::TM_DP, make_sdesc_sw128(a, 16, 1024), make_sdesc_sw128(b, 16, 1024), idesc_s, k > 0);
            }
          }
          umma_commit(bar_s_full);
          if (t == n - 1) umma_commit(bar_x_empty + xs);  // last read of this stationary slot issued
          SCFA_MSTAMP(3);
          mbar_wait(bar_p_full, tg & 1);
          SCFA_MSTAMP(4);
          if (t == 0 && ia >= C::NACC) mbar_wait(bar_acc_free + ab, ((ia / C::NACC) - 1) & 1);
          tc_fence_after();
          // Accumulate: A (bf16) from TMEM, B = streamed tile read MN-major, K = BN streamed rows.
#pragma unroll
          for (int k = 0; k < C::BN / 16; ++k) {
            const uint32_t on = (t > 0 || k > 0);
            if (kMode == MODE_FWD) {  // O += P V
              umma_ts(acc, tmem + C::TM_S + k * 8, make_sdesc_sw128(y1_addr + k * 2048, C::BN * 128, 1024),
                      idesc_acc, on);
            } else if (kMode == MODE_DQ) {  // dQ += dS K
              umma_ts(acc, tmem + C::TM_S + k * 8, make_sdesc_sw128(y0_addr + k * 2048, C::BN * 128, 1024),
                      idesc_acc, on);
            } else {  // dV += P^T dO ; dK += dS^T Q
              umma_ts(acc, tmem + C::TM_S + k * 8, make_sdesc_sw128(y1_addr + k * 2048, C::BN * 128, 1024),
                      idesc_acc, on);
              umma_ts(acc + kD, tmem + C::TM_DP + k * 8, make_sdesc_sw128(y0_addr + k * 2048, C::BN * 128, 1024),
                      idesc_acc, on);
            }
          }
          umma_commit(bar_y_empty + st);
          SCFA_MSTAMP(5);
        }
        umma_commit(bar_acc_full + ab);
        ++ia;
      }
    }
  } else {
    // ------------------------------------------------------------ row threads
    const int r = threadIdx.x;  // 0..127 == TMEM lane
    const uint32_t lane_off = static_cast<uint32_t>(warp * 32) << 16;
    const uint32_t t_s = tmem + lane_off + C::TM_S;
    const uint32_t t_dp = tmem + lane_off + C::TM_DP;
    const float sl = args.scale_log2;
    const bool excl = args.exclude_self != 0;
    const bool use_hash = args.use_hash != 0;
    const float NEG_INF = -INFINITY;
    int tg = 0, ia = 0;
    for (int w = blockIdx.x; w < args.n_items; w += gridDim.x) {
      int bh, rb;
      decode_item(args, w, bh, rb);
      const int lb = bh * args.n_row_blocks + rb;
      const int n = args.list_count[lb];
      const uint16_t* lst = args.list + static_cast<size_t>(lb) * args.list_stride;
      const int row = rb * C::BM + r;
      const size_t roff = static_cast<size_t>(bh) * args.T_rows_pad + row;
      const int my_idx = args.row_idx[roff];
      const int my_hash = args.row_hash[roff];
      const int ab = ia % C::NACC;
      const uint32_t t_acc = tmem + lane_off + C::TM_ACC + ab * C::ACC_COLS;
      size_t orow = 0;
      const bool live = out_row(args, bh, row, my_idx, orow);

      if (kMode == MODE_FWD) {
        const float mask_val = sl >= 0.f ? NEG_INF : INFINITY;
        float m_run = NEG_INF;   // log2-domain max used for exponentiation (lags by < 8)
        float m_true = NEG_INF;  // exact running max of scaled logits (log2 domain)
        float l_run = 0.f;
        for (int t = 0; t < n; ++t, ++tg) {
          const int entry = lst[t];
          const bool full = (entry & 0x8000) != 0;
          const int st = tg % C::NS;
          const int* kidx = reinterpret_cast<const int*>(smem + C::OFF_STAGE + st * C::STAGE_BYTES + 2 * C::Y_BYTES);
          const int* khash = kidx + C::BN;
          constexpr int NW = C::BN / 32;
          uint32_t vis[NW];
          SCFA_STAMP(0);
          mbar_wait(bar_s_full, tg & 1);
          SCFA_STAMP(1);
          tc_fence_after();
          uint32_t raw[C::BN];
#pragma unroll
          for (int c = 0; c < C::BN; c += 32) tmem_ld32(t_s + c, *reinterpret_cast<uint32_t(*)[32]>(&raw[c]));
          if (full) {
#pragma unroll
            for (int i = 0; i < NW; ++i) vis[i] = 0xffffffffu;
          } else {
            const int nv = min(C::BN, args.T_cols - (entry & 0x7fff) * C::BN);
            int lo, hi;
            interval_q_rows<C::BN>(kidx, khash, nv, my_idx, my_hash, excl, use_hash, lo, hi);
            run_mask<NW>(lo, hi, vis);
          }
          tmem_wait_ld();
          float s[C::BN];
#pragma unroll
          for (int c = 0; c < C::BN; ++c) s[c] = ((vis[c >> 5] >> (c & 31)) & 1u) ? __uint_as_float(raw[c]) : mask_val;
          float mq[4] = {mask_val, mask_val, mask_val, mask_val};
          if (sl >= 0.f) {
#pragma unroll
            for (int c = 0; c < C::BN; ++c) mq[c & 3] = fmaxf(mq[c & 3], s[c]);
          } else {
#pragma unroll
            for (int c = 0; c < C::BN; ++c) mq[c & 3] = fminf(mq[c & 3], s[c]);
          }
          const float mx = (sl >= 0.f) ? fmaxf(fmaxf(mq[0], mq[1]), fmaxf(mq[2], mq[3]))
                                       : fminf(fminf(mq[0], mq[1]), fminf(mq[2], mq[3]));
          const float m_tile = mx * sl;  // -inf when the whole row is masked in this tile
          m_true = fmaxf(m_true, m_tile);
          // Rebase to a new max (log2 units) only when the max grows by >= 2^8: P stays
          // <= 256 and the final normalisation by l keeps the result exact.
          float alpha = 1.f;
          const bool rebase = m_tile > m_run + 8.0f || (m_run == NEG_INF && m_tile != NEG_INF);
          if (rebase) {
            alpha = (m_run == NEG_INF) ? 0.f : ex2(m_run - m_tile);
            l_run *= alpha;
            m_run = m_tile;
          }
          const float m_use = (m_run == NEG_INF) ? 0.f : m_run;
          float ls[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
          for (int c = 0; c < C::BN; c += 32) {
            uint32_t pk[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const float p0 = ex2(fmaf(s[c + 2 * i], sl, -m_use));
              const float p1 = ex2(fmaf(s[c + 2 * i + 1], sl, -m_use));
              ls[(2 * i) & 3] += p0;
              ls[(2 * i + 1) & 3] += p1;
              pk[i] = pack_bf16(p0, p1);
            }
            tmem_st16(t_s + c / 2, pk);
          }
          l_run += (ls[0] + ls[1]) + (ls[2] + ls[3]);
          // tcgen05.ld/st are warp-collective: the whole warp rescales when any row must
          // (alpha == 1 for the others, an exact no-op).  The previous P.V into this
          // accumulator has completed: s_full of this tile was committed after it.
          if (__any_sync(0xffffffffu, rebase && t > 0)) {
#pragma unroll 1
            for (int c = 0; c < kD; c += 32) {
              uint32_t v[32];
              tmem_ld32(t_acc + c, v);
              tmem_wait_ld();
#pragma unroll
              for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) * alpha);
              tmem_st32(t_acc + c, v);
            }
          }
          tmem_wait_st();
          tc_fence_before();
          mbar_arrive(bar_p_full);
          SCFA_STAMP(2);
        }
        // ---------------- epilogue: O / l (fused scatter), M, L, lse2
        if (n > 0) {
          mbar_wait(bar_acc_full + ab, (ia / C::NACC) & 1);
          tc_fence_after();
        }
        const float inv_l = (l_run > 0.f) ? 1.f / l_run : 0.f;
        __nv_bfloat16* op = args.out_o + orow * kD;
#pragma unroll
        for (int c = 0; c < kD; c += 32) {
          uint32_t v[32];
          if (n > 0) {  // warp-uniform; every thread of the warp loads (warp-collective)
            tmem_ld32(t_acc + c, v);
            tmem_wait_ld();
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = 0u;
          }
          uint4 o4[4];
          uint32_t* ow = reinterpret_cast<uint32_t*>(o4);
#pragma unroll
          for (int i = 0; i < 16; ++i)
            ow[i] = pack_bf16(__uint_as_float(v[2 * i]) * inv_l, __uint_as_float(v[2 * i + 1]) * inv_l);
          if (live) {
            uint4* dst = reinterpret_cast<uint4*>(op + c);
#pragma unroll
            for (int i = 0; i < 4; ++i) dst[i] = o4[i];
          }
        }
        if (n > 0) {
          tc_fence_before();
          mbar_arrive(bar_acc_free + ab);
          ++ia;
        }
        if (row < args.T_rows) {
          const size_t so = static_cast<size_t>(bh) * args.T_rows + row;
          const float LN2 = 0.6931471805599453f;
          const bool dead = !(l_run > 0.f);
          const float m_use = (m_run == NEG_INF) ? 0.f : m_run;
          args.out0[so] = dead ? NEG_INF : m_true * LN2;           // M
          args.out1[so] = dead ? 0.f : l_run * ex2(m_use - m_true);  // L relative to M
          args.out_lse2[roff] = dead ? INFINITY : (m_use + __log2f(l_run));
        }
      } else {
        // ---------------- backward passes: P and dS recomputed from (lse2, delta)
        float my_lse = 0.f, my_delta = 0.f;
        if (kMode == MODE_DQ) {
          my_lse = args.lse2[roff];
          my_delta = args.delta[roff];
        }
        for (int t = 0; t < n; ++t, ++tg) {
          const int entry = lst[t];
          const bool full = (entry & 0x8000) != 0;
          const int st = tg % C::NS;
          const int* cidx = reinterpret_cast<const int*>(smem + C::OFF_STAGE + st * C::STAGE_BYTES + 2 * C::Y_BYTES);
          const int* chash = cidx + C::BN;
          const float* clse = reinterpret_cast<const float*>(chash + C::BN);
          const float* cdelta = clse + C::BN;
          constexpr int NW = C::BN / 32;
          uint32_t vis[NW];
          SCFA_STAMP(0);
          mbar_wait(bar_s_full, tg & 1);
          SCFA_STAMP(1);
          tc_fence_after();
          if (full) {
#pragma unroll
            for (int i = 0; i < NW; ++i) vis[i] = 0xffffffffu;
          } else {
            const int nv = min(C::BN, args.T_cols - (entry & 0x7fff) * C::BN);
            int lo, hi;
            if (kMode == MODE_DQ)
              interval_q_rows<C::BN>(cidx, chash, nv, my_idx, my_hash, excl, use_hash, lo, hi);
            else
              interval_k_rows<C::BN>(cidx, chash, nv, my_idx, my_hash, excl, use_hash, lo, hi);
            run_mask<NW>(lo, hi, vis);
          }
#pragma unroll
          for (int c = 0; c < C::BN; c += 32) {
            uint32_t sv[32], dv[32];
            tmem_ld32(t_s + c, sv);
            tmem_ld32(t_dp + c, dv);
            tmem_wait_ld();
            const uint32_t wv = vis[c >> 5];
            uint32_t pk_p[16], pk_ds[16];
#pragma unroll
            for (int i = 0; i < 32; i += 4) {
              float lse4[4], del4[4];
              if (kMode == MODE_DQ) {
#pragma unroll
                for (int e = 0; e < 4; ++e) { lse4[e] = my_lse; del4[e] = my_delta; }
              } else {
                const float4 a = *reinterpret_cast<const float4*>(clse + c + i);
                const float4 b = *reinterpret_cast<const float4*>(cdelta + c + i);
                lse4[0] = a.x; lse4[1] = a.y; lse4[2] = a.z; lse4[3] = a.w;
                del4[0] = b.x; del4[1] = b.y; del4[2] = b.z; del4[3] = b.w;
              }
              float pp[4], dd[4];
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                float p = ex2(fmaf(__uint_as_float(sv[i + e]), sl, -lse4[e]));
                p = ((wv >> (i + e)) & 1u) ? p : 0.f;
                pp[e] = p;
                dd[e] = p * (__uint_as_float(dv[i + e]) - del4[e]);
              }
              pk_p[i / 2] = pack_bf16(pp[0], pp[1]);
              pk_p[i / 2 + 1] = pack_bf16(pp[2], pp[3]);
              pk_ds[i / 2] = pack_bf16(dd[0], dd[1]);
              pk_ds[i / 2 + 1] = pack_bf16(dd[2], dd[3]);
            }
            if (kMode == MODE_DQ) {
              tmem_st16(t_s + c / 2, pk_ds);
            } else {
              tmem_st16(t_s + c / 2, pk_p);
              tmem_st16(t_dp + c / 2, pk_ds);
            }
          }
          tmem_wait_st();
          tc_fence_before();
          mbar_arrive(bar_p_full);
          SCFA_STAMP(2);
        }
        if (n > 0) {
          mbar_wait(bar_acc_full + ab, (ia / C::NACC) & 1);
          tc_fence_after();
        }
        const int n_out = (kMode == MODE_DKDV) ? 2 : 1;
#pragma unroll
        for (int o = 0; o < n_out; ++o) {
          // DQ: out0 = scale * dQ.  DKDV: out0 = scale * dK (acc + D), out1 = dV (acc).
          const int col = (kMode == MODE_DKDV && o == 0) ? kD : 0;
          const float mul = (o == 0) ? args.scale : 1.f;
          float* dst = ((o == 0) ? args.out0 : args.out1) + orow * kD;
#pragma unroll
          for (int c = 0; c < kD; c += 32) {
            uint32_t v[32];
            if (n > 0) {
              tmem_ld32(t_acc + col + c, v);
              tmem_wait_ld();
            } else {
#pragma unroll
              for (int i = 0; i < 32; ++i) v[i] = 0u;
            }
            if (live) {
              float4* d4 = reinterpret_cast<float4*>(dst + c);
#pragma unroll
              for (int i = 0; i < 8; ++i)
                d4[i] = make_float4(__uint_as_float(v[4 * i]) * mul, __uint_as_float(v[4 * i + 1]) * mul,
                                    __uint_as_float(v[4 * i + 2]) * mul, __uint_as_float(v[4 * i + 3]) * mul);
            }
          }
        }
        if (n > 0) {
          tc_fence_before();
          mbar_arrive(bar_acc_free + ab);
          ++ia;
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 5) {
    tc_fence_after();
    tmem_dealloc<C::TM_COLS>(tmem);
  }
}

// ------------------------------------------------------------------ host side

static int make_map(CUtensorMap* map, const void* base, int BH, int T, int D, int box_rows) {
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(D), static_cast<cuuint64_t>(T), static_cast<cuuint64_t>(BH)};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(D) * 2, static_cast<cuuint64_t>(T) * D * 2};
  cuuint32_t box[3] = {64, static_cast<cuuint32_t>(box_rows), 1};
  cuuint32_t estr[3] = {1, 1, 1};
  return encode_tensor_map_bf16_3d(map, base, dims, strides, box, estr);
}

static long long* g_dbg_buf = nullptr;
static int g_dbg_tiles = 0;

static int sm_count() {
  int dev = 0, n = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n > 0 ? n : 148;
}

template <int kMode, int kD>
static int launch_mode(const AttnLaunch& L, cudaStream_t stream) {
  using C = Cfg<kMode, kD>;
  CUtensorMap mx0, mx1, my0, my1;
  int rc = 0;
  rc |= make_map(&mx0, L.x0, L.BH, L.T_rows, kD, C::BM);
  rc |= make_map(&mx1, L.x1 ? L.x1 : L.x0, L.BH, L.T_rows, kD, C::BM);
  rc |= make_map(&my0, L.y0, L.BH, L.T_cols, kD, C::BN);
  rc |= make_map(&my1, L.y1, L.BH, L.T_cols, kD, C::BN);
  if (rc) return SCFA_ERR_CUDA;
  AttnArgs a;
  a.BH = L.BH;
  a.H = L.H > 0 ? L.H : 1;
  a.T_rows = L.T_rows;
  a.T_cols = L.T_cols;
  a.T_rows_pad = L.T_rows_pad;
  a.T_cols_pad = L.T_cols_pad;
  a.T_out = L.T_out;
  a.out_boundary = L.out_boundary;
  a.row_idx = L.row_idx;
  a.row_hash = L.row_hash;
  a.col_idx = L.col_idx;
  a.col_hash = L.col_hash;
  a.lse2 = L.lse2;
  a.delta = L.delta;
  a.list = L.list;
  a.list_count = L.list_count;
  a.list_stride = L.list_stride;
  a.n_row_blocks = L.n_row_blocks;
  a.n_items = L.n_row_blocks * L.BH;
  a.out_o = L.out_o;
  a.out0 = L.out0;
  a.out1 = L.out1;
  a.out_lse2 = L.out_lse2;
  a.scale_log2 = L.scale * 1.4426950408889634f;
  a.scale = L.scale;
  a.exclude_self = L.exclude_self;
  a.use_hash = L.use_hash;
  a.dbg = g_dbg_buf;
  a.dbg_tiles = g_dbg_tiles;
  auto kern = scfa_attn_kernel<kMode, kD>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM_BYTES) != cudaSuccess)
    return SCFA_ERR_CUDA;
  if (a.n_items == 0) return SCFA_OK;
  // persistent: as many CTAs as fit (2 per SM when smem and TMEM allow)
  const int per_sm = (2 * C::SMEM_BYTES <= 227 * 1024 && C::TM_COLS <= 256) ? 2 : 1;
  int grid = sm_count() * per_sm;
  if (grid > a.n_items) grid = a.n_items;
  kern<<<grid, 192, C::SMEM_BYTES, stream>>>(mx0, mx1, my0, my1, a);
  return cudaGetLastError() == cudaSuccess ? SCFA_OK : SCFA_ERR_CUDA;
}

int launch_attention(const AttnLaunch& L, cudaStream_t stream) {
  if (L.D == 64) {
    if (L.mode == MODE_FWD) return launch_mode<MODE_FWD, 64>(L, stream);
    if (L.mode == MODE_DQ) return launch_mode<MODE_DQ, 64>(L, stream);
    if (L.mode == MODE_DKDV) return launch_mode<MODE_DKDV, 64>(L, stream);
  } else if (L.D == 128) {
    if (L.mode == MODE_FWD) return launch_mode<MODE_FWD, 128>(L, stream);
    if (L.mode == MODE_DQ) return launch_mode<MODE_DQ, 128>(L, stream);
    if (L.mode == MODE_DKDV) return launch_mode<MODE_DKDV, 128>(L, stream);
  }
  return SCFA_ERR_SHAPE;
}

void set_debug_buffer(long long* p, int tiles) {
  g_dbg_buf = p;
  g_dbg_tiles = tiles;
}

}  // namespace scfa

extern "C" int scfa_debug_timing(void* buf, int64_t tiles_per_cta) {
  scfa::set_debug_buffer(static_cast<long long*>(buf), static_cast<int>(tiles_per_cta));
  return 0;
}
