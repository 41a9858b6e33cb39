// scfa_attn.cu — tcgen05/TMEM/TMA tile engine for Sparse Causal Flash Attention.
//
// One kernel template runs all three passes of the reference tile loop
// (pkg/src/scfa/_kernel.py:92-193):
//
//   FWD      rows = queries, streamed cols = keys.   S = Q K^T ; P = softmax ; O += P V
//   BWD_DQ   rows = queries, streamed cols = keys.   S, dP = dO V^T ; dS ; dQ += dS K
//   BWD_DKDV rows = keys,    streamed cols = queries. S^T, dP^T ; dV += P^T dO ; dK += dS^T Q
//
// Each CTA owns one 128-row stationary block of one (b, h) slice at a time
// (persistent, items handed out round-robin) and walks that block's tile list
// (scfa_sched.cu): only tiles holding at least one visible (query, key) pair are
// listed, so fully masked tiles are skipped, not masked, and tiles whose pairs
// are all visible carry a flag that removes the per-element mask.  Inside a
// boundary tile a row's visible columns are one contiguous run [lo, hi) of slots
// (its bucket run cut at the causal boundary), precomputed per row, so the mask
// costs two subtractions per tile.
//
// One persistent CTA per SM (148 x 512 threads), items (slice, 128-row block) handed
// out dynamically through an atomic counter and published in a shared-memory ring one
// item ahead.  Roles (warpgroups):
//   WG0, WG1  : row threads, one per stationary row == TMEM lane: online softmax (fwd)
//               or P / dS recompute (bwd) with packed fp32x2 math.  FWD and dQ run two
//               independent item streams per CTA (WG0 / WG1, each with its own producer,
//               MMA issuer, smem slots and 256 TMEM columns); dK/dV runs one stream whose
//               tiles alternate between WG0 and WG1 ("ALT") over two S / dP buffers.
//   WG2       : epilogue: reads finished accumulators out of TMEM, releases them
//               (o_free), stages the rows in the item's stationary slot and copies them
//               out so each warp store covers whole rows, each row going straight to its
//               original position (the inverse scatter fused in).
//   WG3       : warps 12 / 14 TMA producers (tiled 128-B-swizzle boxes, or tile::gather4
//               from the caller's (B, T, H, D) tensors through row tables), warps 13 / 15
//               warp-uniform MMA issuers (one elected lane issues tcgen05.mma / .cp /
//               .commit).  setmaxnreg gives the row warpgroups the register file.
//
// TMEM (512 columns per CTA; per stream at D = 64 with two streams):
//   FWD   S fp32 [0,128)  O [128,128+D)  P bf16 [128+D, 192+D)
//   DQ    S [0,64)  dP [64,128)  dQ [128,128+D)  dS bf16 [128+D, 160+D)
//   DKDV  buffers j = 0, 1 at 128 j: S^T [0,64) dP^T [64,128) with P^T / dS^T bf16 written
//         over them; dV, dK accumulators at 256; at D = 64 the stationary K / V rows
//         (tcgen05.cp) at 384 in two buffers, read by the S^T / dP^T MMAs (TS mode).
// With P (dS) in its own columns the S buffer is free as soon as the row threads
// have loaded it, so the MMA warp issues the next tile's S while they work on
// this one ("overlap"); an item's last tile accumulates behind the next item's
// first S when that item is already staged.
#include "scfa_common.cuh"
#include "scfa_internal.h"

namespace scfa {

// MODE_BWD: the single-pass backward — key-stationary like MODE_DKDV, and each pair of
// streamed 64-query tiles also issues dQ = scale * dS K into TMEM, drained by the epilogue
// warpgroup with fp32 reductions into the caller's zero-filled dQ (not bitwise
// deterministic: the add order varies; MODE_DQ + MODE_DKDV remain the deterministic path).
enum Mode : int { MODE_FWD = 0, MODE_DQ = 1, MODE_DKDV = 2, MODE_BWD = 3 };

#ifndef SCFA_TUNE_NS0_FWD
#define SCFA_TUNE_NS0_FWD 2
#endif
#ifndef SCFA_TUNE_NS1_FWD
#define SCFA_TUNE_NS1_FWD 3
#endif
#ifndef SCFA_TUNE_NS0_DQ
#define SCFA_TUNE_NS0_DQ 4
#endif
#ifndef SCFA_TUNE_NS1_DQ
#define SCFA_TUNE_NS1_DQ 2
#endif
#ifndef SCFA_TUNE_NS0_ALT
#define SCFA_TUNE_NS0_ALT 6
#endif
#ifndef SCFA_TUNE_NS1_ALT
#define SCFA_TUNE_NS1_ALT 5
#endif
#ifndef SCFA_TUNE_ROW_REGS_DQ
#define SCFA_TUNE_ROW_REGS_DQ 184
#endif
#ifndef SCFA_TUNE_KV_TMEM
#define SCFA_TUNE_KV_TMEM 1
#endif
#ifndef SCFA_TUNE_QE
#define SCFA_TUNE_QE 3
#endif
#ifndef SCFA_TUNE_DKDV_PFREE
#define SCFA_TUNE_DKDV_PFREE 1
#endif
#ifndef SCFA_TUNE_DQ_SPLIT_SDP
#define SCFA_TUNE_DQ_SPLIT_SDP 1
#endif
#ifndef SCFA_TUNE_DKDV_SPLIT_SDP
#define SCFA_TUNE_DKDV_SPLIT_SDP 0
#endif

template <int kMode, int kD>
struct Cfg {
  // One CTA per SM runs NSTREAM independent item streams (two at D = 64: each has its
  // own row warpgroup, producer warp, MMA warp, smem slots and 256 TMEM columns), and a
  // shared epilogue warpgroup drains finished accumulators for both.
  // Backward ("ALT"): one stream per CTA whose tiles alternate between the two row
  // warpgroups (a tile's P / dS depend only on that tile), each with its own S / dP TMEM
  // buffer, so S(t+1) runs while P(t) is computed and both warpgroups work at once.
  // measured: dK/dV gains; dQ loses at D = 64 (two streams beat one MMA issuer) but gains at
  // D = 128, where TMEM holds only one dQ stream anyway
  static constexpr bool FUSED = (kMode == MODE_BWD);
  // FWD at D = 128 (one item stream: TMEM holds one S + O set): the two row warpgroups split
  // each 128-column S tile by columns, each with its own running max / sum and its own O
  // accumulator (O0 += P[:, :64] V[:64], O1 += P[:, 64:] V[64:]); the epilogue combines
  // O = (2^(m0-m) O0 + 2^(m1-m) O1) / (2^(m0-m) l0 + 2^(m1-m) l1).
  static constexpr bool SPLIT = (kMode == MODE_FWD && kD == 128);
  static constexpr bool KEYS = (kMode == MODE_DKDV || kMode == MODE_BWD);  // key-stationary
#ifndef SCFA_TUNE_DQ_ALT64
#define SCFA_TUNE_DQ_ALT64 0
#endif
  static constexpr bool ALT = KEYS || (kMode == MODE_DQ && (kD == 128 || SCFA_TUNE_DQ_ALT64));
  static constexpr int NSTREAM = ALT ? 1 : ((kD == 64) ? 2 : 1);
  static constexpr int THREADS = 512;
  static constexpr int BM = 128;                             // stationary rows per work item
  static constexpr int BN = (kMode == MODE_FWD) ? 128 : 64;  // streamed rows per tile
  static constexpr int DCH = kD / 64;                        // 128-byte column chunks
  static constexpr int NX = (kMode == MODE_FWD) ? 1 : 2;     // stationary tensors
  static constexpr int NXS = 2;                              // stationary slots (next item prefetch)
  static constexpr bool AUX = KEYS;                          // per-column lse2 / delta with y0
  static constexpr int X_BYTES = BM * kD * 2;
  static constexpr int XSLOT_BYTES = NX * X_BYTES;
  static constexpr int Y_BYTES = BN * kD * 2;
  static constexpr int AUX_BYTES = AUX ? 2 * BN * 4 : 0;
  // y0 / y1 ring slots are released after the S-phase MMAs ("early") or after the
  // accumulate MMAs: K feeds only S in the forward, V feeds only dP in dQ.
  static constexpr bool Y0_EARLY = (kMode == MODE_FWD);
  static constexpr bool Y1_EARLY = (kMode == MODE_DQ);
  // ring depths (SCFA_TUNE_* build-time overrides for tuning sweeps, scripts/tune.py)
  static constexpr int NS0 = FUSED ? 5 : (kMode == MODE_FWD)   ? ((kD == 64) ? SCFA_TUNE_NS0_FWD : 2)
                             : (ALT && kD == 64)   ? SCFA_TUNE_NS0_ALT
                             : (kMode == MODE_DQ && kD == 64) ? SCFA_TUNE_NS0_DQ
                                                   : 3;
  static constexpr int NS1 = FUSED ? 5 : (kMode == MODE_FWD)   ? ((kD == 64) ? SCFA_TUNE_NS1_FWD : 2)
                             : (ALT && kD == 64)   ? SCFA_TUNE_NS1_ALT
                             : (kMode == MODE_DQ && kD == 64) ? SCFA_TUNE_NS1_DQ
                                                   : 2;
  // TMEM (per stream)
  static constexpr int TM_COLS = 512;  // allocated once per CTA
  static constexpr int TM_STREAM = TM_COLS / NSTREAM;
  // FWD: S [0,128) O [128,128+D) P bf16 [128+D, 192+D).  ALT: buffer j at j*128 holds
  // S [0,64) and dP [64,128), with P / dS (bf16) written over them; accumulators at 256.
  static constexpr int TM_BUF = 128;
  // ALT: S / dP buffers in TMEM (tile t uses buffer t % NBUF, row warpgroup t % 2)
  // dK/dV at D = 64: the stationary K and V also live in TMEM (32 columns each, two
  // buffers: item i uses buffer i % 2), so the S^T / dP^T MMAs read A from TMEM (TS mode:
  // 32 instead of 48 clk per N = 64 MMA, scripts/mma_issue.cu) — which leaves room for
  // two S / dP buffers, not three
  static constexpr bool KV_TMEM = SCFA_TUNE_KV_TMEM && (kMode == MODE_DKDV && kD == 64);
  // S and dP committed separately, so the rows compute a tile's first P chunk from S while
  // the dP MMAs still run: dQ (two streams; dP completes on s_full + 1) and dK/dV at D = 64
  // (Sᵀ / dPᵀ from TMEM-resident K / V; dPᵀ of buffer j completes on dq_full + j, a barrier
  // the dK/dV pass does not otherwise use)
  static constexpr bool SDP_SPLIT = (SCFA_TUNE_DQ_SPLIT_SDP && kMode == MODE_DQ && !ALT) ||
                                    (SCFA_TUNE_DKDV_SPLIT_SDP && kMode == MODE_DKDV && KV_TMEM);
  static constexpr int NBUF = (KV_TMEM || FUSED) ? 2 : ((ALT && 3 * TM_BUF + (KEYS ? 2 * kD : kD) <= 512) ? 3 : 2);
  static constexpr int TM_S = 0;
  static constexpr int TM_DP = (kMode == MODE_FWD) ? 0 : BN;
  static constexpr int TM_ACC = ALT ? NBUF * TM_BUF : 128;
  static constexpr int ACC_COLS = (KEYS || SPLIT) ? 2 * kD : kD;
  static constexpr int P_COLS = KEYS ? BN : BN / 2;
  static constexpr bool OVERLAP = !ALT && (TM_ACC + ACC_COLS + P_COLS <= TM_STREAM);
  static constexpr int TM_P = OVERLAP ? TM_ACC + ACC_COLS : TM_S;                 // P | dS | P^T
  static constexpr int TM_P2 = OVERLAP ? TM_ACC + ACC_COLS + BN / 2 : TM_DP;      // dS^T (DKDV)
  static_assert(TM_ACC + ACC_COLS <= TM_STREAM, "TMEM budget");
  static constexpr int TM_KV = TM_ACC + ACC_COLS;  // KV_TMEM buffer b: K [TM_KV + b*kD, +kD/2), V next
  static_assert(!KV_TMEM || TM_KV + 2 * kD <= TM_STREAM, "TMEM budget (K / V)");
  // FUSED: two dQ accumulators (M = 128 rows = the 2 x 64 queries of a tile pair, N = kD)
  static constexpr int TM_DQ = TM_ACC + ACC_COLS;
  static_assert(!FUSED || TM_DQ + 2 * kD <= TM_STREAM, "TMEM budget (dQ)");
  // shared memory per stream (all TMA destinations 1024-aligned)
  static constexpr int OFF_X = 0;
  static constexpr int OFF_Y0 = OFF_X + NXS * XSLOT_BYTES;
  static constexpr int OFF_Y1 = OFF_Y0 + NS0 * Y_BYTES;
  static constexpr int OFF_AUX = OFF_Y1 + NS1 * Y_BYTES;
  // FUSED: dS of a tile pair as the dQ MMA's A operand (M = 128 queries, K = 128 keys,
  // MN-major: two 64-query atoms of 128 key rows x 128 B), double-buffered by pair
  static constexpr int DS_ATOM = BM * 128;
  static constexpr int DS_PAIR = 2 * DS_ATOM;
  static constexpr int OFF_DS = ((OFF_AUX + NS0 * AUX_BYTES + 1023) / 1024) * 1024;
  static constexpr int STREAM_BYTES = OFF_DS + (FUSED ? 2 * DS_PAIR : 0);
  // per-stream control block after all streams' tiles: s_full, s_free, p_full, p_free,
  // acc_full, o_free, x_full/empty[NXS], y0_full/empty[NS0], y1_full/empty[NS1],
  // q_full/empty[NQ] (work ring); the ring
  static constexpr int NQ = 4;
  static constexpr int N_BARS = 12 + 2 * NXS + 2 * NS0 + 2 * NS1 + 2 * NQ + 6;
  static constexpr int OFF_BAR = 0;
  static constexpr int OFF_RING = OFF_BAR + 8 * N_BARS;  // int2 {item, tiles} x NQ
  static constexpr int CTRL_BYTES = ((OFF_RING + 8 * NQ + 15) / 16) * 16;
  static constexpr int OFF_CTRL = NSTREAM * STREAM_BYTES;
  // epilogue queues, one per TMEM lane quadrant (row warp q of either stream -> epilogue
  // warp q), entries taken in ticket order: per quadrant eq_full[QE], eq_empty[QE], a
  // ticket, entries {int4 info, float inv_l[32]}
  static constexpr int QE = SCFA_TUNE_QE;
  static constexpr int OFF_EQ = OFF_CTRL + NSTREAM * CTRL_BYTES;
  static constexpr int EQ_ENTRY = 16 + 4 * 32 + (SPLIT ? 4 * 32 : 0);  // info, inv_l[32] (SPLIT: + a1[32])
  // SPLIT: the second warpgroup's (m_run, l_run, m_true) per row for the item's combine, by item parity
  static constexpr int XCH_BYTES = SPLIT ? 2 * 3 * BM * 4 : 0;
  static constexpr int EQQ_BYTES = 16 * QE + 16 + QE * EQ_ENTRY;  // one quadrant
  static constexpr int EQ_BYTES = 4 * EQQ_BYTES;
  static constexpr int OFF_XCH = OFF_EQ + EQ_BYTES;
  static constexpr int SMEM_BYTES = OFF_XCH + XCH_BYTES + 16;
  static_assert(X_BYTES % 1024 == 0 && Y_BYTES % 1024 == 0, "TMA tiles must stay 1024-aligned");
  static_assert(SMEM_BYTES <= 227 * 1024, "shared memory budget");
  // epilogue staging reuses the item's stationary slot
  static_assert((kMode == MODE_FWD ? BM * kD * 2 : BM * kD * 4) <= XSLOT_BYTES, "staging fits the slot");
};

struct AttnArgs {
  int BH, H;
  int T_rows, T_cols;          // true lengths of the stationary / streamed side
  int T_rows_pad, T_cols_pad;  // padded lengths of the per-slot vectors
  int T_out;                   // boundary-layout output length (out_boundary)
  int out_boundary;            // 1: write rows to (B, T_out, H, D) at their original position
  const int* row_idx;          // original position of each stationary row (output routing)
  const int2* row_runs;        // visible streamed-slot run [lo, hi) of each stationary row
  const float* lse2;           // (BH, Tq_pad), log2 domain; +inf where no key is visible
  const float* delta;          // (BH, Tq_pad)
  const int* x_rows;  // gather mode: global row per stationary slot (BH, T_rows_pad); null = tiled loads
  const int* out_rows;  // optional output routing: global row of each stationary slot (BH, T_rows_pad), pad
                        // slots included (every row of the [R, D] output is written; tiled loads)
  const int* y_rows;  // gather mode: global row per streamed slot (BH, T_cols_pad)
  int x0_tiled;                // gather mode: the first stationary tensor comes tiled (kernel order)
  int x_writeout;              // gather mode: write a gathered stationary tile out through tm_xo (kernel
                               // order): FWD its Q, DQ its dO (the tensors dK/dV streams)
  const __nv_bfloat16* o_src;  // DQ: O rows (addressed like dO) for the fused delta
  float* delta_out;            // DQ: delta = rowsum(dO * O) per query slot (BH, T_rows_pad)
  const uint16_t* list;
  const int* list_count;
  int list_stride;
  int n_row_blocks;
  int n_items;
  const int* col_idx;  // BWD: original position of each streamed (query) slot (BH, T_cols_pad)
  float* out2;         // BWD: dQ, zero-filled by the caller, reduced into
  int T_out_cols;      // BWD: boundary-layout length of the dQ rows
  __nv_bfloat16* out_o;  // FWD
  float* out0;           // FWD: M      DQ: dQ   DKDV: dK
  float* out1;           // FWD: L      DKDV: dV
  float* out_lse2;       // FWD
  float scale_log2;
  float scale;
  int* err_flag;  // FWD: SCFA_ERR_NUMERIC on a non-finite output (update_stats, softmax.py:63-64)
  long long* dbg;  // optional per-tile timestamps (diagnostics)
  int dbg_tiles;
};

// Diagnostics: per-CTA, per-tile clock64 stamps, 16 slots per tile (see scripts/timing.py).
#define SCFA_STAMP_AT(i, k)                                                                   \
  if (args.dbg && (i) >= 0 && (i) < args.dbg_tiles)                                          \
    args.dbg[(static_cast<size_t>(dbg_cta) * args.dbg_tiles + (i)) * 16 + (k)] = clock64();
#define SCFA_STAMP(k) \
  if (r == 0) { SCFA_STAMP_AT(tg, k) }
#define SCFA_MSTAMP(k) SCFA_STAMP_AT(tg, k)

// Work index -> item (bh * n_row_blocks + rb).  Items are handed out dynamically
// (one atomic counter per launch, next to the tile counts) in the order: heaviest row
// block first (largest causal reach), cycling over heads.
SCFA_DEVICE int item_of(const AttnArgs& a, int w) {
  const int rb = a.n_row_blocks - 1 - w / a.BH;
  const int bh = w - (w / a.BH) * a.BH;
  return bh * a.n_row_blocks + rb;
}

// Output row of stationary row `row` (original position `pos`): engine layout
// (bh, row) or boundary layout (b, pos, h) — the fused inverse scatter.
SCFA_DEVICE bool out_row(const AttnArgs& a, int bh, int row, int pos, size_t& off) {
  if (row >= a.T_rows) return false;
  if (a.out_rows) {  // routing table: pad slots map to the positions they stand for (zero rows)
    off = static_cast<size_t>(a.out_rows[static_cast<size_t>(bh) * a.T_rows_pad + row]);
    return true;
  }
  if (a.x_rows) {  // row tables: `pos` is the global row the stationary operand came from
    off = static_cast<size_t>(pos);
    return true;
  }
  if (!a.out_boundary) {
    off = static_cast<size_t>(bh) * a.T_rows + row;
    return true;
  }
  if (pos < 0 || pos >= a.T_out) return false;  // pad slots (QUERY_PAD / KEY_PAD)
  const int b = bh / a.H, h = bh - b * a.H;
  off = (static_cast<size_t>(b) * a.T_out + pos) * a.H + h;
  return true;
}

// BWD: output row of streamed (query) slot `slot` with original position `pos` — the dQ
// row, engine layout (bh, slot) or boundary layout (b, pos, h).
SCFA_DEVICE bool out_col(const AttnArgs& a, int bh, int slot, int pos, size_t& off) {
  if (slot >= a.T_cols) return false;
  if (!a.out_boundary) {
    off = static_cast<size_t>(bh) * a.T_cols + slot;
    return true;
  }
  if (pos < 0 || pos >= a.T_out_cols) return false;  // pad slots
  const int b = bh / a.H, h = bh - b * a.H;
  off = (static_cast<size_t>(b) * a.T_out_cols + pos) * a.H + h;
  return true;
}

SCFA_DEVICE void red_add_v4(float* p, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
}

// Which element pairs of a 32-column chunk take the polynomial exp2 (FMA pipe) instead of
// MUFU.  Measured: none — the loops are issue / latency bound rather than MUFU bound, and
// the polynomial's extra instructions cost more than the MUFU time they free.
#ifndef SCFA_TUNE_POLY
#define SCFA_TUNE_POLY 0
#endif
// every SCFA_TUNE_POLY-th exponential pair on the FMA pipe (0: none)
SCFA_DEVICE constexpr bool kPolyPair(int pair) { return SCFA_TUNE_POLY > 0 && (pair % (SCFA_TUNE_POLY > 0 ? SCFA_TUNE_POLY : 1)) == SCFA_TUNE_POLY - 1; }

SCFA_DEVICE uint32_t bits_below(int n) { return n <= 0 ? 0u : (n >= 32 ? 0xffffffffu : ((1u << n) - 1u)); }

// 32-column visibility words of the run [lo, hi) (tile-local columns)
template <int NW>
SCFA_DEVICE void run_mask(int lo, int hi, uint32_t (&w)[NW]) {
#pragma unroll
  for (int i = 0; i < NW; ++i) w[i] = bits_below(hi - 32 * i) & ~bits_below(lo - 32 * i);
}

// ---- coalesced epilogue ------------------------------------------------------------
// Each row thread holds one output row; written directly, every 16-byte piece of a
// warp store lands in a different row (32 partial-line writes per instruction).  The
// rows are instead staged in the item's stationary smem slot — free once the last
// S MMA has run — and copied out so that each warp store covers whole rows.
// Staging layout: row r at r * RB bytes, 16-byte chunk c at position c ^ (r & 7).
template <int RB>
SCFA_DEVICE void stage_put(uint8_t* stage, int r, int c, uint32_t a, uint32_t b, uint32_t cc, uint32_t d) {
  const uint32_t addr = smem_u32(stage + r * RB + ((c ^ (r & 7)) << 4));
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(cc), "r"(d) : "memory");
}

// Copy this warp's 32 staged rows to global: row (warp*32 + i) goes to gbase +
// off[i] bytes where off/live are held by lane i.
template <int RB>
SCFA_DEVICE void stage_copy_out(const uint8_t* stage, int warp, int lane, uint8_t* gbase, long long my_off,
                                bool my_live) {
  constexpr int CPR = RB / 16;  // 16-byte chunks per row
  constexpr int R = 32 / CPR;   // rows per warp instruction
  __syncwarp();
#pragma unroll
  for (int j = 0; j < CPR; ++j) {
    const int i = j * R + lane / CPR;
    const int c = lane % CPR;
    const long long off = __shfl_sync(0xffffffffu, my_off, i);
    const int lv = __shfl_sync(0xffffffffu, my_live ? 1 : 0, i);
    const int row = warp * 32 + i;
    const uint32_t addr = smem_u32(stage + row * RB + ((c ^ (row & 7)) << 4));
    uint4 v;
    asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
    if (lv) *reinterpret_cast<uint4*>(gbase + off + c * 16) = v;
  }
  __syncwarp();
}

template <int N>
SCFA_DEVICE void tmem_ld_cols(uint32_t taddr, uint32_t* r) {
#pragma unroll
  for (int c = 0; c < N; c += 32) tmem_ld32(taddr + c, *reinterpret_cast<uint32_t(*)[32]>(r + c));
}

// Per-role stream context, declared inside each role after the register rebalancing so
// that nothing is live across setmaxnreg.
#define SCFA_STREAM_SETUP                                                                        \
  uint8_t* smem = smem_base + s * C::STREAM_BYTES;                                               \
  uint8_t* ctrl = smem_base + C::OFF_CTRL + s * C::CTRL_BYTES;                                   \
  const int dbg_cta = blockIdx.x * C::NSTREAM + s;                                               \
  (void)dbg_cta;                                                                                 \
  const Bars B = bars_of<C>(ctrl);                                                               \
  const MBar bar_s_full = B.s_full, bar_s_free = B.s_free, bar_p_full = B.p_full;                \
  const MBar bar_p_free = B.p_free, bar_acc_full = B.acc_full, bar_x_full = B.x_full;            \
  const MBar bar_x_empty = B.x_empty, bar_y0_full = B.y0_full, bar_y0_empty = B.y0_empty;        \
  const MBar bar_y1_full = B.y1_full, bar_y1_empty = B.y1_empty, bar_q_full = B.q_full;          \
  const MBar bar_q_empty = B.q_empty;                                                            \
  (void)bar_s_full; (void)bar_s_free; (void)bar_p_full; (void)bar_p_free; (void)bar_acc_full;    \
  (void)bar_x_full; (void)bar_x_empty; (void)bar_y0_full; (void)bar_y0_empty; (void)bar_y1_full; \
  (void)bar_y1_empty; (void)bar_q_full; (void)bar_q_empty;                                       \
  int2* ring = reinterpret_cast<int2*>(ctrl + C::OFF_RING);                                      \
  int* work_ctr = const_cast<int*>(args.list_count) + args.n_items;                              \
  const uint32_t tmem = *tmem_slot + static_cast<uint32_t>(s * C::TM_STREAM);                    \
  (void)ring; (void)work_ctr; (void)tmem; (void)smem;

struct Bars {
  MBar s_full, s_free, p_full, p_free, acc_full, o_free, x_full, x_empty, y0_full, y0_empty, y1_full, y1_empty, q_full,
      q_empty;  // s_full / p_full / p_free: three consecutive barriers (TMEM buffers in ALT)
  MBar ds_free, dq_full, dq_free;  // BWD, two each (by tile pair parity)
};

template <class C>
SCFA_DEVICE Bars bars_of(uint8_t* base) {
  Bars b;
  const MBar p0(smem_u32(base + C::OFF_BAR));
  int i = 0;
  b.s_full = p0 + i;
  i += 3;
  b.s_free = p0 + i++;
  b.p_full = p0 + i;
  i += 3;
  b.p_free = p0 + i;
  i += 3;
  b.acc_full = p0 + i++;
  b.o_free = p0 + i++;
  b.x_full = p0 + i;
  i += C::NXS;
  b.x_empty = p0 + i;
  i += C::NXS;
  b.y0_full = p0 + i;
  i += C::NS0;
  b.y0_empty = p0 + i;
  i += C::NS0;
  b.y1_full = p0 + i;
  i += C::NS1;
  b.y1_empty = p0 + i;
  i += C::NS1;
  b.q_full = p0 + i;
  i += C::NQ;
  b.q_empty = p0 + i;
  i += C::NQ;
  b.ds_free = p0 + i;
  i += 2;
  b.dq_full = p0 + i;
  i += 2;
  b.dq_free = p0 + i;
  return b;
}

// One bounded wait: suspends the warp (no issue slots) until the phase completes or
// about `ns` nanoseconds pass; returns whether it completed.
SCFA_DEVICE bool mbar_try(MBar bar, uint32_t parity, uint32_t ns) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2, %3;\n\t"
      "selp.b32 %0, 1, 0, P1;\n\t}"
      : "=r"(ok)
      : "r"(bar.a), "r"(parity), "r"(ns)
      : "memory");
  return ok != 0;
}

// ------------------------------------------------------------------ epilogue warpgroup
// Drains finished items of both streams: waits for an item handed over by the row
// threads (mailbox) and its accumulators (acc_full), reads them out of TMEM, releases
// them (o_free: the stream's next item may accumulate), stages the rows in the item's
// stationary slot and copies them out — each row to its original position — then hands
// the slot back to the producer (x_empty).  The row threads never wait for any of it.
template <int kMode, int kD>
SCFA_DEVICE void epilogue_wg(const AttnArgs& args, uint8_t* smem_base, uint32_t tmem0, int warp, int lane,
                             int dbg_cta0) {
  using C = Cfg<kMode, kD>;
  const int r = threadIdx.x & 127;
  const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
  int cnt[2] = {0, 0};
  int pce = 0;  // BWD: tile pairs drained
  int live_streams = C::NSTREAM;
  uint8_t* eqb = smem_base + C::OFF_EQ + (warp & 3) * C::EQQ_BYTES;
  const MBar eq(smem_u32(eqb));
  for (int k = 0; live_streams > 0; ++k) {
    {
      int s;
      int2 item;
      float inv_l = 0.f, a1 = 0.f;  // SPLIT: O = inv_l * O0 + a1 * O1
      if (C::ALT) {  // one stream: follow its work ring (items finish in ring order)
        s = 0;
        const Bars B0 = bars_of<C>(smem_base + C::OFF_CTRL);
        const int qs = k % C::NQ;
        mbar_wait_lazy(B0.q_full + qs, (k / C::NQ) & 1);
        item = reinterpret_cast<const int2*>(smem_base + C::OFF_CTRL + C::OFF_RING)[qs];
        mbar_arrive(B0.q_empty + qs);
        if (item.x < 0) {
          --live_streams;
          continue;
        }
        if (item.y == 0) {  // no visible pair in the block: zero gradients (and delta)
          const int bh = item.x / args.n_row_blocks, rb = item.x - bh * args.n_row_blocks;
          const int row = rb * C::BM + r;
          const size_t foff = static_cast<size_t>(bh) * args.T_rows_pad + row;
          const int pos = args.x_rows ? args.x_rows[foff] : args.row_idx[foff];
          size_t orow = 0;
          if (kMode == MODE_DQ && args.delta_out) args.delta_out[foff] = 0.f;
          if (out_row(args, bh, row, pos, orow)) {
#pragma unroll
            for (int o = 0; o < (C::KEYS ? 2 : 1); ++o) {
              float4* d4 = reinterpret_cast<float4*>(((o == 0) ? args.out0 : args.out1) + orow * kD);
#pragma unroll
              for (int i = 0; i < kD / 4; ++i) d4[i] = make_float4(0.f, 0.f, 0.f, 0.f);
            }
          }
          continue;
        }
      } else {
        const int slot = k % C::QE;
        mbar_wait_lazy(eq + slot, (k / C::QE) & 1);
        const uint8_t* ent = eqb + 16 * C::QE + 16 + slot * C::EQ_ENTRY;
        const int4 info = *reinterpret_cast<const int4*>(ent);
        inv_l = reinterpret_cast<const float*>(ent + 16)[lane];
        if (C::SPLIT) a1 = reinterpret_cast<const float*>(ent + 16 + 128)[lane];
        mbar_arrive(eq + C::QE + slot);
        if (info.y < 0) {  // a stream's end
          --live_streams;
          continue;
        }
        s = info.x;
        item = make_int2(info.y, info.z);
      }
      uint8_t* smem = smem_base + s * C::STREAM_BYTES;
      uint8_t* ctrl = smem_base + C::OFF_CTRL + s * C::CTRL_BYTES;
      const Bars B = bars_of<C>(ctrl);
      const int ia = cnt[s]++;
      const int bh = item.x / args.n_row_blocks, rb = item.x - bh * args.n_row_blocks;
      const int row = rb * C::BM + r;
      const size_t foff = static_cast<size_t>(bh) * args.T_rows_pad + row;
      const int pos = args.x_rows ? args.x_rows[foff] : args.row_idx[foff];
      size_t orow = 0;
      const bool live = out_row(args, bh, row, pos, orow);
      const uint32_t t_acc = tmem0 + static_cast<uint32_t>(s * C::TM_STREAM) + lane_off + C::TM_ACC;
      uint8_t* stage = smem + C::OFF_X + (ia % C::NXS) * C::XSLOT_BYTES;
      if (C::FUSED) {
        // dQ of each tile pair of the item, as its MMAs finish: TMEM lane r holds query
        // (r & 63) of tile 2m + (r >> 6).  The buffer is released as soon as it is read,
        // then each row is reduced (fp32 red.v4) into the query's dQ row at its original
        // position.  (Coalescing the reductions through shared memory, or issuing them from
        // the row warpgroups, measured no faster: DESIGN.md §6.)
        const uint32_t t_dq = tmem0 + lane_off + C::TM_DQ;
        const uint16_t* lst = args.list + static_cast<size_t>(item.x) * args.list_stride;
        for (int t0 = 0; t0 < item.y; t0 += 2, ++pce) {
          const int pb = pce & 1;
          mbar_wait_lazy(B.dq_full + pb, (pce >> 1) & 1);
          tc_fence_after();
          uint32_t v0[32], v1[32];
          tmem_ld32(t_dq + pb * kD, v0);
          tmem_ld32(t_dq + pb * kD + 32, v1);
          tmem_wait_ld();
          tc_fence_before();
          mbar_arrive_relaxed(B.dq_free + pb);
          const int t = t0 + (r >> 6);
          if (t < item.y) {
            const int slot = (lst[t] & 0x7fff) * C::BN + (r & 63);
            size_t qoff = 0;
            if (slot < args.T_cols) {
              const int pos = args.col_idx[static_cast<size_t>(bh) * args.T_cols_pad + slot];
              if (out_col(args, bh, slot, pos, qoff)) {
                float* dst = args.out2 + qoff * kD;
                const float sc = args.scale;
#pragma unroll
                for (int i = 0; i < 8; ++i)
                  red_add_v4(dst + 4 * i, __uint_as_float(v0[4 * i]) * sc, __uint_as_float(v0[4 * i + 1]) * sc,
                             __uint_as_float(v0[4 * i + 2]) * sc, __uint_as_float(v0[4 * i + 3]) * sc);
#pragma unroll
                for (int i = 0; i < 8; ++i)
                  red_add_v4(dst + 32 + 4 * i, __uint_as_float(v1[4 * i]) * sc, __uint_as_float(v1[4 * i + 1]) * sc,
                             __uint_as_float(v1[4 * i + 2]) * sc, __uint_as_float(v1[4 * i + 3]) * sc);
              }
            }
          }
        }
      }
      mbar_wait_lazy(B.acc_full, ia & 1);
      tc_fence_after();
      if (kMode == MODE_FWD) {
        constexpr int RB = kD * 2;  // bf16 output row
        bool finite_ok = true;
#pragma unroll
        for (int c = 0; c < kD; c += 32) {
          uint32_t v[32];
          tmem_ld32(t_acc + c, v);
          if (C::SPLIT) {
            uint32_t u[32];
            tmem_ld32(t_acc + kD + c, u);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 32; ++i)
              v[i] = __float_as_uint(fmaf(__uint_as_float(v[i]), inv_l, __uint_as_float(u[i]) * a1));
          } else {
            tmem_wait_ld();
          }
          uint32_t w[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const float o0 = C::SPLIT ? __uint_as_float(v[2 * i]) : __uint_as_float(v[2 * i]) * inv_l;
            const float o1 = C::SPLIT ? __uint_as_float(v[2 * i + 1]) : __uint_as_float(v[2 * i + 1]) * inv_l;
            finite_ok &= (fabsf(o0) <= FLT_MAX) & (fabsf(o1) <= FLT_MAX);
            w[i] = pack_bf16(o0, o1);
          }
#pragma unroll
          for (int i = 0; i < 4; ++i) stage_put<RB>(stage, r, c / 8 + i, w[4 * i], w[4 * i + 1], w[4 * i + 2], w[4 * i + 3]);
        }
        tc_fence_before();
        mbar_arrive_relaxed(B.o_free);
        // the reference raises NumericError when o turns non-finite (softmax.py:63-64)
        if (__any_sync(0xffffffffu, live && !finite_ok) && args.err_flag && lane == 0)
          atomicCAS(args.err_flag, 0, SCFA_ERR_NUMERIC);
        stage_copy_out<RB>(stage, warp & 3, lane, reinterpret_cast<uint8_t*>(args.out_o), static_cast<long long>(orow) * RB,
                           live);
      } else if (kMode == MODE_DQ) {
        constexpr int RB = kD * 4;
#pragma unroll
        for (int c = 0; c < kD; c += 32) {
          uint32_t v[32];
          tmem_ld32(t_acc + c, v);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) * args.scale);
#pragma unroll
          for (int i = 0; i < 8; ++i) stage_put<RB>(stage, r, c / 4 + i, v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
        }
        tc_fence_before();
        mbar_arrive_relaxed(B.o_free);
        stage_copy_out<RB>(stage, warp & 3, lane, reinterpret_cast<uint8_t*>(args.out0), static_cast<long long>(orow) * RB,
                           live);
      } else {
        // dK (scale * acc[kD:2kD]) staged; at D = 64 dV (acc[0:kD]) is held in registers so
        // the accumulators are released before either copy-out
        constexpr int RB = kD * 4;
#pragma unroll
        for (int c = 0; c < kD; c += 32) {
          uint32_t v[32];
          tmem_ld32(t_acc + kD + c, v);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) * args.scale);
#pragma unroll
          for (int i = 0; i < 8; ++i) stage_put<RB>(stage, r, c / 4 + i, v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
        }
        if (kD == 64) {
          uint32_t dv[kD];
          tmem_ld32(t_acc, *reinterpret_cast<uint32_t(*)[32]>(dv));
          tmem_ld32(t_acc + 32, *reinterpret_cast<uint32_t(*)[32]>(dv + 32));
          tmem_wait_ld();
          tc_fence_before();
          mbar_arrive_relaxed(B.o_free);
          stage_copy_out<RB>(stage, warp & 3, lane, reinterpret_cast<uint8_t*>(args.out0),
                             static_cast<long long>(orow) * RB, live);
#pragma unroll
          for (int i = 0; i < kD / 4; ++i) stage_put<RB>(stage, r, i, dv[4 * i], dv[4 * i + 1], dv[4 * i + 2], dv[4 * i + 3]);
          stage_copy_out<RB>(stage, warp & 3, lane, reinterpret_cast<uint8_t*>(args.out1),
                             static_cast<long long>(orow) * RB, live);
        } else {
          stage_copy_out<RB>(stage, warp & 3, lane, reinterpret_cast<uint8_t*>(args.out0),
                             static_cast<long long>(orow) * RB, live);
#pragma unroll
          for (int c = 0; c < kD; c += 32) {
            uint32_t v[32];
            tmem_ld32(t_acc + c, v);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 8; ++i) stage_put<RB>(stage, r, c / 4 + i, v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
          }
          tc_fence_before();
          mbar_arrive_relaxed(B.o_free);
          stage_copy_out<RB>(stage, warp & 3, lane, reinterpret_cast<uint8_t*>(args.out1),
                             static_cast<long long>(orow) * RB, live);
        }
      }
      fence_proxy_async_smem();  // the next TMA load into this slot comes after these accesses
      mbar_arrive(B.x_empty + (ia % C::NXS));
    }
  }
}

template <int kMode, int kD>
__global__ void __launch_bounds__(512, 1)
    scfa_attn_kernel(const __grid_constant__ CUtensorMap tm_x0, const __grid_constant__ CUtensorMap tm_x1,
                     const __grid_constant__ CUtensorMap tm_y0, const __grid_constant__ CUtensorMap tm_y1,
                     const __grid_constant__ CUtensorMap tm_xo, const AttnArgs args) {
  using C = Cfg<kMode, kD>;
  extern __shared__ __align__(1024) uint8_t smem_base[];

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int wg = warp >> 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem_base + C::OFF_XCH + C::XCH_BYTES);

  if (threadIdx.x == 0) {
    if (smem_u32(smem_base) & 1023) __trap();  // TMA SWIZZLE_128B destinations need 1024-byte alignment
    for (int st = 0; st < C::NSTREAM; ++st) {
      const Bars b = bars_of<C>(smem_base + C::OFF_CTRL + st * C::CTRL_BYTES);
      for (int j = 0; j < 3; ++j) {
        mbar_init(b.s_full + j, 1);
        mbar_init(b.p_full + j, C::SPLIT ? 256 : 128);
        mbar_init(b.p_free + j, 1);
      }
      mbar_init(b.s_free, C::SPLIT ? 256 : 128);
      mbar_init(b.acc_full, 1);
      mbar_init(b.o_free, 128);  // epilogue threads: accumulators read, the next item may overwrite
      for (int i = 0; i < C::NXS; ++i) {
        mbar_init(b.x_full + i, 1);
        mbar_init(b.x_empty + i, 128);  // released by the epilogue threads after staging
      }
      for (int i = 0; i < C::NS0; ++i) {
        mbar_init(b.y0_full + i, 1);
        mbar_init(b.y0_empty + i, 1);
      }
      for (int i = 0; i < C::NS1; ++i) {
        mbar_init(b.y1_full + i, 1);
        mbar_init(b.y1_empty + i, 1);
      }
      for (int i = 0; i < 2; ++i) {
        mbar_init(b.ds_free + i, 1);   // BWD: the pair's dQ MMAs have read its dS
        mbar_init(b.dq_full + i, 1);   // BWD: the pair's dQ is in TMEM
        mbar_init(b.dq_free + i, 128); // BWD: the epilogue has read it
      }
      for (int i = 0; i < C::NQ; ++i) {
        mbar_init(b.q_full + i, 1);
        // the MMA thread + the row threads (+ the second row warpgroup and the epilogue in ALT)
        mbar_init(b.q_empty + i, C::ALT ? 1 + 128 + 128 + 128 : (C::SPLIT ? 1 + 256 : 1 + 128));
      }
    }
    for (int q = 0; q < 4; ++q) {
      uint8_t* eqb = smem_base + C::OFF_EQ + q * C::EQQ_BYTES;
      const MBar eq(smem_u32(eqb));
      for (int i = 0; i < C::QE; ++i) {
        mbar_init(eq + i, 32);          // a row warp: its quadrant of an item handed over
        mbar_init(eq + C::QE + i, 32);  // the quadrant's epilogue warp: entry read
      }
      reinterpret_cast<int*>(eqb + 16 * C::QE)[0] = 0;  // ticket
    }
    fence_barrier_init();
  }
  if (warp == 13) tmem_alloc<C::TM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // roles: warps 0-3 rows of stream 0, 4-7 rows of stream 1, 8-11 epilogue (both
  // streams), 12 / 14 producer of stream 0 / 1, 13 / 15 MMA issuer of stream 0 / 1.
  // Register rebalancing happens first thing inside each warpgroup's branch (nothing
  // live across it, no merge after it): the row warpgroups take the file the epilogue /
  // producer / MMA warps do not need.
  // row / epilogue register split (the two row warpgroups take what the epilogue gives up);
  // SCFA_TUNE_ROW_REGS_DQ: the dQ pass's row code spills at 176 and not at 184, the
  // epilogue still fits 88 there (ptxas -v)
  constexpr int kRowSplit = (kMode == MODE_DQ && kD == 64) ? SCFA_TUNE_ROW_REGS_DQ : 176;
  constexpr int kRowRegs = (C::NSTREAM == 2 || C::ALT || C::SPLIT) ? kRowSplit : 240;
  constexpr int kEpiRegs = (C::NSTREAM == 2 || C::ALT || C::SPLIT) ? 104 - 2 * (kRowSplit - 176) : 104;
  const int s = (C::ALT || C::SPLIT) ? 0 : ((wg < 2) ? wg : ((warp >= 12) ? ((warp - 12) >> 1) : 0));
  const bool active = (C::ALT || C::SPLIT) ? (wg < 2 || ((warp - 12) >> 1) == 0) : (s < C::NSTREAM);
  if (wg == 3) {
   asm volatile("setmaxnreg.dec.sync.aligned.u32 56;" ::: "memory");
   if (((warp - 12) & 1) == 0 && active) {
    // ------------------------------------------------------------ TMA producer warp
    SCFA_STREAM_SETUP
    if (lane == 0) {
      tma_prefetch_desc(&tm_x0);
      tma_prefetch_desc(&tm_y0);
      tma_prefetch_desc(&tm_y1);
      if (C::NX == 2) tma_prefetch_desc(&tm_x1);
    }
    const bool gx = args.x_rows != nullptr, gy = args.y_rows != nullptr;
    int tg = 0, ia = 0;
    // Work ring: item k+1 is grabbed and published before item k's tiles are loaded, so
    // the consumers can always look one item ahead without waiting on the loads.
    auto grab = [&](int k) -> int2 {
      int2 e = make_int2(-1, 0);
      if (lane == 0) {
        const int w = atomicAdd(work_ctr, 1);
        if (w < args.n_items) {
          // the schedule's order: the longest items first (item_order_kernel)
          const int* ord = args.list_count + item_order_offset(args.n_items) + 2 * w;
          e.x = ord[0];
          e.y = ord[1];
        }
        const int qs = k % C::NQ;
        if (k >= C::NQ) mbar_wait_lazy(bar_q_empty + qs, ((k / C::NQ) - 1) & 1);
        ring[qs] = e;
        mbar_arrive(bar_q_full + qs);
      }
      e.x = __shfl_sync(0xffffffffu, e.x, 0);
      e.y = __shfl_sync(0xffffffffu, e.y, 0);
      return e;
    };
    int2 cur = grab(0);
    for (int k = 0; cur.x >= 0; ++k) {
      const int2 item = cur;
      cur = grab(k + 1);
      const int lb = item.x, n = item.y;
      if (n == 0) continue;
      const int bh = lb / args.n_row_blocks, rb = lb - bh * args.n_row_blocks;
      const uint16_t* lst = args.list + static_cast<size_t>(lb) * args.list_stride;
      const int xs = ia % C::NXS;
      if (ia >= C::NXS) mbar_wait_lazy(bar_x_empty + xs, ((ia / C::NXS) - 1) & 1);
      uint8_t* xb = smem + C::OFF_X + xs * C::XSLOT_BYTES;
      if (lane == 0) {
        mbar_arrive_expect_tx(bar_x_full + xs, C::XSLOT_BYTES);
      }
      __syncwarp();
      if (gx) {  // 128 stationary rows: 4 per lane
        const int4 r4 = __ldg(reinterpret_cast<const int4*>(args.x_rows + static_cast<size_t>(bh) * args.T_rows_pad +
                                                          rb * C::BM) + lane);
        if (args.x0_tiled && lane == 0) {  // Q already in kernel order: one tiled box per chunk
          for (int c = 0; c < C::DCH; ++c) tma_load_3d(xb + c * C::BM * 128, &tm_x0, bar_x_full + xs, c * 64, rb * C::BM, bh);
        }
#pragma unroll
        for (int c = 0; c < C::DCH; ++c) {
          if (!args.x0_tiled)
            tma_gather4(xb + c * C::BM * 128 + lane * 512, &tm_x0, bar_x_full + xs, c * 64, r4.x, r4.y, r4.z, r4.w);
          if (C::NX == 2)
            tma_gather4(xb + C::X_BYTES + c * C::BM * 128 + lane * 512, &tm_x1, bar_x_full + xs, c * 64, r4.x, r4.y,
                        r4.z, r4.w);
        }
      } else if (lane == 0) {
        for (int c = 0; c < C::DCH; ++c) {
          tma_load_3d(xb + c * C::BM * 128, &tm_x0, bar_x_full + xs, c * 64, rb * C::BM, bh);
          if (C::NX == 2) tma_load_3d(xb + C::X_BYTES + c * C::BM * 128, &tm_x1, bar_x_full + xs, c * 64, rb * C::BM, bh);
        }
      }
      // list entries one tile ahead: a dependent global load per tile would pace the
      // whole stream at one L2 round trip per tile
      int ent_next = lst[0];
      for (int t = 0; t < n; ++t, ++tg) {
        const int col0 = (ent_next & 0x7fff) * C::BN;
        if (t + 1 < n) ent_next = lst[t + 1];
        int4 r4 = make_int4(0, 0, 0, 0);
        if (gy && lane < C::BN / 4)
          r4 = __ldg(reinterpret_cast<const int4*>(args.y_rows + static_cast<size_t>(bh) * args.T_cols_pad + col0) + lane);
        // y0 ring (+ per-column lse2 / delta for dK/dV)
        const int st = tg % C::NS0;
        if (tg >= C::NS0) mbar_wait_lazy(bar_y0_empty + st, ((tg / C::NS0) - 1) & 1);
        uint8_t* yb = smem + C::OFF_Y0 + st * C::Y_BYTES;
        if (lane == 0) {
          SCFA_STAMP_AT(tg, 14);
          mbar_arrive_expect_tx(bar_y0_full + st, C::Y_BYTES + C::AUX_BYTES);
        }
        __syncwarp();
        if (gy) {
          if (lane < C::BN / 4) {
#pragma unroll
            for (int c = 0; c < C::DCH; ++c)
              tma_gather4(yb + c * C::BN * 128 + lane * 512, &tm_y0, bar_y0_full + st, c * 64, r4.x, r4.y, r4.z, r4.w);
          }
        } else if (lane == 0) {
          for (int c = 0; c < C::DCH; ++c) tma_load_3d(yb + c * C::BN * 128, &tm_y0, bar_y0_full + st, c * 64, col0, bh);
        }
        if (C::AUX && lane == 0) {
          uint8_t* aux = smem + C::OFF_AUX + st * C::AUX_BYTES;
          const size_t coff = static_cast<size_t>(bh) * args.T_cols_pad + col0;
          bulk_load(aux, args.lse2 + coff, C::BN * 4, bar_y0_full + st);
          bulk_load(aux + C::BN * 4, args.delta + coff, C::BN * 4, bar_y0_full + st);
        }
        // y1 ring
        const int st1 = tg % C::NS1;
        if (tg >= C::NS1) mbar_wait_lazy(bar_y1_empty + st1, ((tg / C::NS1) - 1) & 1);
        uint8_t* yb1 = smem + C::OFF_Y1 + st1 * C::Y_BYTES;
        if (lane == 0) {
          SCFA_STAMP_AT(tg, 15);
          mbar_arrive_expect_tx(bar_y1_full + st1, C::Y_BYTES);
        }
        __syncwarp();
        if (gy) {
          if (lane < C::BN / 4) {
#pragma unroll
            for (int c = 0; c < C::DCH; ++c)
              tma_gather4(yb1 + c * C::BN * 128 + lane * 512, &tm_y1, bar_y1_full + st1, c * 64, r4.x, r4.y, r4.z,
                          r4.w);
          }
        } else if (lane == 0) {
          for (int c = 0; c < C::DCH; ++c) tma_load_3d(yb1 + c * C::BN * 128, &tm_y1, bar_y1_full + st1, c * 64, col0, bh);
        }
      }
      ++ia;
    }
   } else if (((warp - 12) & 1) == 1 && active) {
    // ------------------------------------------------------------ MMA issuer
    // The whole warp runs the loop (warp-uniform control flow keeps the descriptors in
    // uniform registers); one elected lane issues the MMAs and their commits.
    SCFA_STREAM_SETUP
    {
      constexpr uint32_t idesc_s = make_idesc_bf16(128, C::BN, false, false);
      constexpr uint32_t idesc_acc = make_idesc_bf16(128, kD, false, true);
      // the accumulate MMAs of tile `p` (P V | dS K | P^T dO + dS^T Q)
      int tg = 0, ia = 0;
      int pc = 0;  // BWD: tile pairs whose dQ has been issued
      constexpr uint32_t idesc_dq = make_idesc_bf16(128, kD, true, true);  // A = dS, B = K: both MN-major
      auto flush = [&](int ptg, bool first, bool last, int pia, int pt) {
        const int s0 = ptg % C::NS0, s1 = ptg % C::NS1;
        if (kMode == MODE_FWD) mbar_wait_lazy(bar_y1_full + s1, (ptg / C::NS1) & 1);  // V not needed before
        if (lane == 0) { SCFA_STAMP_AT(ptg, 12); }
        const int jb = C::ALT ? (ptg % C::NBUF) : 0;  // TMEM buffer holding tile ptg's P / dS
        mbar_wait(bar_p_full + jb, C::ALT ? ((ptg / C::NBUF) & 1) : (ptg & 1));
        if (lane == 0) { SCFA_STAMP_AT(ptg, 13); }
        if (first && pia > 0) mbar_wait_lazy(B.o_free, (pia - 1) & 1);  // the epilogue has read the previous item
        // BWD: a pair of tiles (local 2m, 2m+1; or a last odd tile alone) is complete: its dQ
        // goes into TMEM buffer pc % 2 once the epilogue has drained that buffer's last pair
        const bool dq_now = C::FUSED && (((pt & 1) == 1) || last);
        if (dq_now && pc >= 2) mbar_wait_lazy(B.dq_free + (pc & 1), ((pc >> 1) - 1) & 1);
        if (lane == 0) { SCFA_STAMP_AT(ptg, 4); }
        tc_fence_after();
        // the epilogue reuses the stationary slot once acc_full fires: the write-out must
        // have read it by then
        if (!C::KEYS && last && args.x_writeout && lane == 0) bulk_wait_read0();
        __syncwarp();
        const uint32_t y0_addr = smem_u32(smem + C::OFF_Y0 + s0 * C::Y_BYTES);
        const uint32_t y1_addr = smem_u32(smem + C::OFF_Y1 + s1 * C::Y_BYTES);
        const uint32_t acc = tmem + C::TM_ACC;
        const uint32_t pb = tmem + jb * C::TM_BUF;
        if (elect_one()) {
#pragma unroll
        for (int k = 0; k < C::BN / 16; ++k) {
          const uint32_t on = (!first || k > 0);
          if (kMode == MODE_FWD) {  // O += P V  (SPLIT: keys [0, 64) into O0, [64, 128) into O1)
            const uint32_t acc_k = (C::SPLIT && k >= C::BN / 32) ? acc + kD : acc;
            const uint32_t on_k = C::SPLIT ? static_cast<uint32_t>(!first || (k % (C::BN / 32)) > 0) : on;
            umma_ts(acc_k, pb + C::TM_P + k * 8, make_sdesc_sw128(y1_addr + k * 2048, C::BN * 128, 1024), idesc_acc,
                    on_k);
          } else if (kMode == MODE_DQ) {  // dQ += dS K
            umma_ts(acc, pb + C::TM_P + k * 8, make_sdesc_sw128(y0_addr + k * 2048, C::BN * 128, 1024), idesc_acc,
                    on);
          } else {  // dV += P^T dO ; dK += dS^T Q
            umma_ts(acc, pb + C::TM_P + k * 8, make_sdesc_sw128(y1_addr + k * 2048, C::BN * 128, 1024), idesc_acc,
                    on);
            umma_ts(acc + kD, pb + C::TM_P2 + k * 8, make_sdesc_sw128(y0_addr + k * 2048, C::BN * 128, 1024),
                    idesc_acc, on);
          }
        }
        if (C::FUSED && dq_now) {
          // dQ[pair] = dS K over the item's 128 keys: A = the pair's dS (M = 128 queries,
          // MN-major, written by the row threads), B = the stationary K tile read MN-major
          // (N = head dim contiguous); 16 keys per MMA
          const uint32_t ds_addr = smem_u32(smem + C::OFF_DS + (pc & 1) * C::DS_PAIR);
          const uint32_t k_addr = smem_u32(smem + C::OFF_X + (pia % C::NXS) * C::XSLOT_BYTES);
          const uint32_t dq_acc = tmem + C::TM_DQ + (pc & 1) * kD;
#pragma unroll
          for (int k = 0; k < C::BM / 16; ++k)
            umma_ss(dq_acc, make_sdesc_sw128(ds_addr + k * 2048, C::DS_ATOM, 1024),
                    make_sdesc_sw128(k_addr + k * 2048, C::BM * 128, 1024), idesc_dq, k > 0);
          umma_commit(B.ds_free + (pc & 1));
          umma_commit(B.dq_full + (pc & 1));
        }
        if (!C::Y0_EARLY) umma_commit(bar_y0_empty + s0);
        if (!C::Y1_EARLY) umma_commit(bar_y1_empty + s1);
        umma_commit(bar_p_free + jb);
        if (last) umma_commit(bar_acc_full);
        }
        __syncwarp();
        if (dq_now) ++pc;
      };
      // The item's last tile accumulates behind the next item's first S, as inner tiles do,
      // when the next item is already staged; otherwise (the producer is behind, or no
      // item is left) it accumulates at once, since the epilogue waits for it.
      constexpr bool kDeferLast = true;
      int p_tg = -1, p_ia = 0, p_t = 0;
      bool p_first = false, p_last = false;
      for (int k = 0;; ++k) {
        const int qs = k % C::NQ;
        if (p_tg >= 0 && (!kDeferLast || !mbar_test(bar_q_full + qs, (k / C::NQ) & 1))) {
          flush(p_tg, p_first, p_last, p_ia, p_t);
          p_tg = -1;
        }
        mbar_wait_lazy(bar_q_full + qs, (k / C::NQ) & 1);
        // lane 0 reads the slot and releases it to the producer (one arrival for the MMA warp);
        // the other lanes take the item from it, so no lane reads a slot already released
        int2 item = make_int2(0, 0);
        if (lane == 0) {
          item = ring[qs];
          mbar_arrive(bar_q_empty + qs);
        }
        item.x = __shfl_sync(0xffffffffu, item.x, 0);
        item.y = __shfl_sync(0xffffffffu, item.y, 0);
        if (item.x < 0) break;
        const int n = item.y;
        if (n == 0) continue;
        const int xs = ia % C::NXS;
        const uint32_t x0_addr = smem_u32(smem + C::OFF_X + xs * C::XSLOT_BYTES);
        const uint32_t x1_addr = x0_addr + C::X_BYTES;
        if (p_tg >= 0 && !(mbar_test(bar_x_full + xs, (ia / C::NXS) & 1) &&
                           mbar_test(bar_y0_full + tg % C::NS0, (tg / C::NS0) & 1))) {
          flush(p_tg, p_first, p_last, p_ia, p_t);
          p_tg = -1;
        }
        mbar_wait_lazy(bar_x_full + xs, (ia / C::NXS) & 1);
        if (!C::KEYS && args.x_writeout && lane == 0) {
          // the gathered stationary rows (FWD: Q, DQ: dO), in kernel order, for the dK/dV
          // pass (the slot is read by TMA only, the proxy of its load; the wait is before
          // acc_full, after which the epilogue reuses the slot)
          const int wbh = item.x / args.n_row_blocks, wrb = item.x - wbh * args.n_row_blocks;
          const uint8_t* src = smem + C::OFF_X + xs * C::XSLOT_BYTES + ((kMode == MODE_DQ) ? C::X_BYTES : 0);
          for (int c = 0; c < C::DCH; ++c) tma_store_3d(&tm_xo, src + c * C::BM * 128, c * 64, wrb * C::BM, wbh);
          bulk_commit();
        }
        __syncwarp();
        if (C::KV_TMEM && elect_one()) {
          // stationary K / V -> TMEM buffer ia % 2 (tcgen05.cp, 128 rows x 16 bf16 per copy);
          // copies and MMAs execute in issue order, so the S^T / dP^T below see them
          tc_fence_after();
          const uint32_t kv = tmem + C::TM_KV + (ia & 1) * kD;
#pragma unroll
          for (int k = 0; k < kD / 16; ++k) {
            tmem_cp_128x256b(kv + k * 8, make_sdesc_sw128(x0_addr + k * 32, 16, 1024));
            tmem_cp_128x256b(kv + kD / 2 + k * 8, make_sdesc_sw128(x1_addr + k * 32, 16, 1024));
          }
        }
        __syncwarp();
        if (lane == 0) { SCFA_STAMP_AT(tg, 9); }
        for (int t = 0; t < n; ++t, ++tg) {
          const int s0 = tg % C::NS0, s1 = tg % C::NS1;
          if (lane == 0) { SCFA_MSTAMP(6); }
          mbar_wait_lazy(bar_y0_full + s0, (tg / C::NS0) & 1);
          if (kMode != MODE_FWD) mbar_wait_lazy(bar_y1_full + s1, (tg / C::NS1) & 1);
          const int j = C::ALT ? (tg % C::NBUF) : 0;  // TMEM buffer of this tile
          if (C::ALT) {
            // tile tg-NBUF accumulated (SCFA_TUNE_DKDV_PFREE=0, dK/dV: not waited for — the
            // accumulate MMAs were issued earlier by this thread, tcgen05.mma runs in issue order)
            if (tg >= C::NBUF && (kMode != MODE_DKDV || SCFA_TUNE_DKDV_PFREE))
              mbar_wait(bar_p_free + j, ((tg / C::NBUF) - 1) & 1);
          } else if (C::OVERLAP) {
            if (tg > 0) mbar_wait_lazy(bar_s_free, (tg - 1) & 1);
          } else if (p_tg >= 0) {
            flush(p_tg, p_first, p_last, p_ia, p_t);  // aliased P: the accumulate MMAs must read it first
            p_tg = -1;
          }
          if (lane == 0) { SCFA_MSTAMP(7); }
          tc_fence_after();
          const uint32_t y0_addr = smem_u32(smem + C::OFF_Y0 + s0 * C::Y_BYTES);
          const uint32_t y1_addr = smem_u32(smem + C::OFF_Y1 + s1 * C::Y_BYTES);
          // S = X0 . Y0^T  (and dP = X1 . Y1^T), K = head dim, both operands K-major.
          if (elect_one()) {
            // S and dP are independent accumulation chains: interleaving their K steps lets
            // the tensor pipe overlap one chain's dependent steps with the other's
#pragma unroll
            for (int k = 0; k < kD / 16; ++k) {
              const uint32_t koff = (k & 3) * 32;
              const uint32_t a = x0_addr + (k >> 2) * (C::BM * 128) + koff;
              const uint32_t b = y0_addr + (k >> 2) * (C::BN * 128) + koff;
              if (C::KV_TMEM) {  // A = K / V rows in TMEM (16 bf16 = 8 columns per K step)
                const uint32_t kv = tmem + C::TM_KV + (ia & 1) * kD;
                umma_ts(tmem + j * C::TM_BUF + C::TM_S, kv + k * 8, make_sdesc_sw128(b, 16, 1024), idesc_s, k > 0);
                if (!C::SDP_SPLIT) {
                  const uint32_t b1 = y1_addr + (k >> 2) * (C::BN * 128) + koff;
                  umma_ts(tmem + j * C::TM_BUF + C::TM_DP, kv + kD / 2 + k * 8, make_sdesc_sw128(b1, 16, 1024),
                          idesc_s, k > 0);
                }
              } else {
                umma_ss(tmem + j * C::TM_BUF + C::TM_S, make_sdesc_sw128(a, 16, 1024), make_sdesc_sw128(b, 16, 1024),
                        idesc_s, k > 0);
                if (kMode != MODE_FWD && !C::SDP_SPLIT) {
                  const uint32_t a1 = x1_addr + (k >> 2) * (C::BM * 128) + koff;
                  const uint32_t b1 = y1_addr + (k >> 2) * (C::BN * 128) + koff;
                  umma_ss(tmem + j * C::TM_BUF + C::TM_DP, make_sdesc_sw128(a1, 16, 1024),
                          make_sdesc_sw128(b1, 16, 1024), idesc_s, k > 0);
                }
              }
            }
          if constexpr (C::SDP_SPLIT) {
            umma_commit(bar_s_full + j);  // S complete: the rows start on P
#pragma unroll
            for (int k = 0; k < kD / 16; ++k) {
              const uint32_t koff = (k & 3) * 32;
              const uint32_t b1 = y1_addr + (k >> 2) * (C::BN * 128) + koff;
              if (C::KV_TMEM) {
                const uint32_t kv = tmem + C::TM_KV + (ia & 1) * kD;
                umma_ts(tmem + j * C::TM_BUF + C::TM_DP, kv + kD / 2 + k * 8, make_sdesc_sw128(b1, 16, 1024),
                        idesc_s, k > 0);
              } else {
                const uint32_t a1 = x1_addr + (k >> 2) * (C::BM * 128) + koff;
                umma_ss(tmem + C::TM_DP, make_sdesc_sw128(a1, 16, 1024), make_sdesc_sw128(b1, 16, 1024), idesc_s,
                        k > 0);
              }
            }
            umma_commit(C::KEYS ? B.dq_full + j : bar_s_full + 1);  // dP complete
          } else {
            umma_commit(bar_s_full + j);
          }
          if (C::Y0_EARLY) umma_commit(bar_y0_empty + s0);
          if (C::Y1_EARLY) umma_commit(bar_y1_empty + s1);
          }
          __syncwarp();
          if (lane == 0) { SCFA_MSTAMP(3); }
          if (p_tg >= 0) flush(p_tg, p_first, p_last, p_ia, p_t);  // overlap: tile t-1 accumulates behind S(t)
          p_tg = tg;
          p_ia = ia;
          p_t = t;
          p_first = (t == 0);
          p_last = (t == n - 1);
          if (lane == 0) { SCFA_MSTAMP(5); }
        }
        ++ia;
      }
      if (p_tg >= 0) flush(p_tg, p_first, p_last, p_ia, p_t);
      if (!C::KEYS && args.x_writeout && lane == 0) bulk_wait0();  // write-outs complete
      __syncwarp();
    }
   }
  } else if (wg == 2) {
    // ------------------------------------------------------------ epilogue warpgroup
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kEpiRegs) : "memory");
    epilogue_wg<kMode, kD>(args, smem_base, *tmem_slot, warp, lane, 0);
  } else if (!active) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 24;" ::: "memory");  // idle row warpgroup (one stream)
  } else {
    // ------------------------------------------------------------ row threads
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRowRegs) : "memory");
    SCFA_STREAM_SETUP
    const int r = threadIdx.x & 127;  // 0..127 == TMEM lane
    // hand an item (or the stream's end, lb = -1) to the epilogue queue: a ticket per
    // item keeps one queue for both streams in completion order
    int tg = 0, ia = 0;
    auto handoff = [&](int lb_, int n_, float inv_l_, float a1_ = 0.f) {
      // per row warp: quadrant (warp & 3) of the item goes to epilogue warp (warp & 3)
      uint8_t* eqb = smem_base + C::OFF_EQ + (warp & 3) * C::EQQ_BYTES;
      int tk = 0;
      if (lane == 0) tk = atomicAdd(reinterpret_cast<int*>(eqb + 16 * C::QE), 1);
      tk = __shfl_sync(0xffffffffu, tk, 0);
      const int slot = tk % C::QE;
      const MBar eq(smem_u32(eqb));
      if (tk >= C::QE) mbar_wait(eq + C::QE + slot, ((tk / C::QE) - 1) & 1);
      uint8_t* ent = eqb + 16 * C::QE + 16 + slot * C::EQ_ENTRY;
      reinterpret_cast<float*>(ent + 16)[lane] = inv_l_;
      if (C::SPLIT) reinterpret_cast<float*>(ent + 16 + 128)[lane] = a1_;
      if (lane == 0) *reinterpret_cast<int4*>(ent) = make_int4(s, lb_, n_, 0);
      mbar_arrive(eq + slot);
    };
    const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
    int pcr = 0;  // BWD: tile pairs of the items before this one
    const uint32_t t_s = tmem + lane_off + C::TM_S;
    const uint32_t t_dp = tmem + lane_off + C::TM_DP;
    const uint32_t t_p = tmem + lane_off + C::TM_P;
    const uint32_t t_p2 = tmem + lane_off + C::TM_P2;
    const uint32_t t_acc = tmem + lane_off + C::TM_ACC;
    const float sl = args.scale_log2;
    const float NEG_INF = -INFINITY;
    constexpr int NW = C::BN / 32;
    // per-item metadata is fetched one item ahead (its global-load latency hides behind
    // the current item), and each tile's list entry one tile ahead
    int nx_idx = 0, nx_e0 = 0;
    int2 nx_run = make_int2(0, 0);
    int2 nx_item = make_int2(-1, 0);
    // ring slot k: wait until published, read (the q_empty arrival comes when the item
    // is consumed), and prefetch its per-row metadata
    auto peek = [&](int k) {
      const int qs = k % C::NQ;
      mbar_wait(bar_q_full + qs, (k / C::NQ) & 1);
      nx_item = ring[qs];
      if (nx_item.x < 0) return;
      const int fbh = nx_item.x / args.n_row_blocks, frb = nx_item.x - fbh * args.n_row_blocks;
      const size_t foff = static_cast<size_t>(fbh) * args.T_rows_pad + frb * C::BM + r;
      nx_e0 = args.list[static_cast<size_t>(nx_item.x) * args.list_stride];  // (an empty item's entry is 0)
      nx_idx = args.x_rows ? args.x_rows[foff] : args.row_idx[foff];
      nx_run = args.row_runs[foff];
    };
    peek(0);
    for (int k = 0;; ++k) {
      const int2 item = nx_item;
      mbar_arrive(bar_q_empty + (k % C::NQ));
      if (item.x < 0) break;
      const int lb = item.x;
      const int bh = lb / args.n_row_blocks, rb = lb - bh * args.n_row_blocks;
      const int n = item.y;
      const int my_idx = nx_idx;
      const int2 run = nx_run;
      int entry_next = nx_e0;
      peek(k + 1);
      const uint16_t* lst = args.list + static_cast<size_t>(lb) * args.list_stride;
      const int row = rb * C::BM + r;
      const size_t roff = static_cast<size_t>(bh) * args.T_rows_pad + row;
      size_t orow = 0;
      const bool live = out_row(args, bh, row, my_idx, orow);

      if (kMode == MODE_FWD) {
        // One pass over S per tile, in 32-column chunks, with a lagging exponent base:
        // P = 2^(s*scale*log2e - m_run) where m_run is the row max as of the row's first
        // visible chunk, raised only when a chunk's max exceeds it by more than kLag
        // (P <= 2^kLag stays far inside fp32 / bf16 range; the final 1/l makes the
        // result exact).  A raise is free for a row that has seen nothing yet (l = 0,
        // O = 0) and otherwise rescales l, this tile's stored P chunks and O (rare).
        // Chunks no row of the warp can see are skipped (P = 0, no exponentials).
        constexpr float kLag = 64.f;
        constexpr int NCH = C::BN / 32;
        constexpr int NCH_W = C::SPLIT ? NCH / 2 : NCH;  // chunks of each tile this warpgroup owns
        const int ch0 = C::SPLIT ? wg * NCH_W : 0;
        const uint32_t t_accw = t_acc + (C::SPLIT ? static_cast<uint32_t>(wg * kD) : 0u);  // its O
        const bool neg = sl < 0.f;  // a negative scale turns the row max into a row min
        const float mask_val = neg ? INFINITY : NEG_INF;
        float m_run = NEG_INF;   // log2-domain exponent base (lags the max by < kLag)
        float m_true = NEG_INF;  // exact running max of scaled logits (log2 domain)
        float l_run = 0.f;
        for (int t = 0; t < n; ++t, ++tg) {
          const int entry = entry_next;
          if (t + 1 < n) entry_next = lst[t + 1];
          const bool full = (entry & 0x8000) != 0;
          const int col0 = (entry & 0x7fff) * C::BN;
          SCFA_STAMP(0);
          mbar_wait(bar_s_full, tg & 1);
          SCFA_STAMP(1);
          tc_fence_after();
          const int rlo = run.x - col0, rhi = run.y - col0;
          float la[4] = {0.f, 0.f, 0.f, 0.f};
          bool p_ready = (tg == 0);  // P columns free: the previous tile's PV has read them
#pragma unroll
          for (int chl = 0; chl < NCH_W; ++chl) {
            const int ch = ch0 + chl;
            const uint32_t wv = full ? 0xffffffffu : (bits_below(rhi - 32 * ch) & ~bits_below(rlo - 32 * ch));
            uint32_t pk[16];
            if (__any_sync(0xffffffffu, wv != 0u)) {
              float x[32];
              tmem_ld32(t_s + 32 * ch, *reinterpret_cast<uint32_t(*)[32]>(x));
              tmem_wait_ld();
              if (chl == NCH_W - 1) {
                tc_fence_before();
                mbar_arrive(bar_s_free);  // S fully read: the next tile's S may overwrite it
              }
              const bool partial = __any_sync(0xffffffffu, wv != 0xffffffffu);
              if (partial) {
#pragma unroll
                for (int c = 0; c < 32; ++c) x[c] = ((wv >> c) & 1u) ? x[c] : mask_val;
              }
              float e0 = mask_val, e1 = mask_val;
              if (!neg) {
#pragma unroll
                for (int c = 0; c < 32; c += 4) {
                  e0 = max3(e0, x[c], x[c + 1]);
                  e1 = max3(e1, x[c + 2], x[c + 3]);
                }
              } else {
#pragma unroll
                for (int c = 0; c < 32; c += 4) {
                  e0 = min3(e0, x[c], x[c + 1]);
                  e1 = min3(e1, x[c + 2], x[c + 3]);
                }
              }
              const float ms = (neg ? fminf(e0, e1) : fmaxf(e0, e1)) * sl;  // -inf: nothing visible
              m_true = fmaxf(m_true, ms);
              const bool raise = ms > m_run + kLag;  // includes the row's first visible chunk
              if (__any_sync(0xffffffffu, raise)) {
                const bool rescale = raise && (m_run != NEG_INF);
                float alpha = 1.f;
                if (raise) {
                  alpha = rescale ? ex2(m_run - ms) : 0.f;
                  m_run = ms;
                }
                if (__any_sync(0xffffffffu, rescale)) {  // rare: P chunks of this tile, l, O
                  if (!p_ready) {
                    mbar_wait(bar_p_free, (tg - 1) & 1);
                    tc_fence_after();
                    p_ready = true;
                  }
                  tmem_wait_st();
#pragma unroll 1
                  for (int j = ch0; j < ch; ++j) {
                    uint32_t q16[16];
                    tmem_ld16(t_p + 16 * j, q16);
                    tmem_wait_ld();
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                      const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&q16[i]));
                      q16[i] = pack_bf16(f.x * alpha, f.y * alpha);
                    }
                    tmem_st16(t_p + 16 * j, q16);
                  }
#pragma unroll 1
                  for (int c = 0; c < kD; c += 32) {
                    uint32_t v[32];
                    tmem_ld32(t_accw + c, v);
                    tmem_wait_ld();
#pragma unroll
                    for (int i = 0; i < 32; i += 2) {
                      float o0, o1;
                      mul2(o0, o1, __uint_as_float(v[i]), __uint_as_float(v[i + 1]), alpha, alpha);
                      v[i] = __float_as_uint(o0);
                      v[i + 1] = __float_as_uint(o1);
                    }
                    tmem_st32(t_accw + c, v);
                  }
                  tmem_wait_st();
                }
                l_run *= alpha;
#pragma unroll
                for (int i = 0; i < 4; ++i) la[i] *= alpha;
              }
              const float nm = (m_run == NEG_INF) ? 0.f : -m_run;
#pragma unroll
              for (int c = 0; c < 32; c += 2) {
                float a0, a1;
                fma2(a0, a1, x[c], x[c + 1], sl, sl, nm, nm);
                if (!partial && kPolyPair(c >> 1)) {  // no masked (-inf) inputs in this chunk
                  ex2_poly2(a0, a1, a0, a1);
                } else {
                  a0 = ex2(a0);
                  a1 = ex2(a1);
                }
                const int q = (c >> 1) & 1;
                add2(la[2 * q], la[2 * q + 1], la[2 * q], la[2 * q + 1], a0, a1);
                pk[c >> 1] = pack_bf16(a0, a1);
              }
            } else {
              if (chl == NCH_W - 1) {
                tc_fence_before();
                mbar_arrive(bar_s_free);
              }
#pragma unroll
              for (int i = 0; i < 16; ++i) pk[i] = 0u;
            }
            if (!p_ready) {  // P's columns are read by the previous tile's accumulate MMAs
              mbar_wait(bar_p_free, (tg - 1) & 1);
              tc_fence_after();
              p_ready = true;
            }
            tmem_st16(t_p + 16 * ch, pk);
          }
          l_run += (la[0] + la[1]) + (la[2] + la[3]);
          tmem_wait_st();
          tc_fence_before();
          mbar_arrive(bar_p_full);
          SCFA_STAMP(2);
        }
        // ---------------- hand O / l to the epilogue warpgroup; write M, L, lse2 here
        float inv_l, a1 = 0.f;
        if (C::SPLIT) {
          // the two warpgroups' statistics of each row meet here; the second one is done
          if (wg == 1) {
            if (n > 0) {
              float* xch = reinterpret_cast<float*>(smem_base + C::OFF_XCH) + (ia & 1) * 3 * C::BM;
              xch[r] = m_run;
              xch[C::BM + r] = l_run;
              xch[2 * C::BM + r] = m_true;
              named_bar_sync(1, 256);
              ++ia;
            }
            continue;
          }
          float e0 = 0.f, e1 = 0.f;
          if (n > 0) {
            named_bar_sync(1, 256);
            const float* xch = reinterpret_cast<const float*>(smem_base + C::OFF_XCH) + (ia & 1) * 3 * C::BM;
            const float m1 = xch[r], l1 = xch[C::BM + r], t1 = xch[2 * C::BM + r];
            const float mr = fmaxf(m_run, m1);
            e0 = (m_run == NEG_INF) ? 0.f : ex2(m_run - mr);
            e1 = (m1 == NEG_INF) ? 0.f : ex2(m1 - mr);
            l_run = l_run * e0 + l1 * e1;
            m_run = mr;
            m_true = fmaxf(m_true, t1);
          }
          const float inv = (l_run > 0.f) ? rcp_approx(l_run) : 0.f;
          inv_l = e0 * inv;  // O0's factor; O1's is a1
          a1 = e1 * inv;
        } else {
          inv_l = (l_run > 0.f) ? rcp_approx(l_run) : 0.f;
        }
        if (n > 0) {
          handoff(lb, n, inv_l, a1);
          ++ia;
        } else if (live) {
          uint4* dst = reinterpret_cast<uint4*>(args.out_o + orow * kD);
#pragma unroll
          for (int i = 0; i < kD / 8; ++i) dst[i] = make_uint4(0u, 0u, 0u, 0u);
        }
        if (row < args.T_rows) {
          const size_t so = static_cast<size_t>(bh) * args.T_rows + row;
          const float LN2 = 0.6931471805599453f;
          const bool dead = !(l_run > 0.f);
          if (!(l_run <= FLT_MAX) && args.err_flag) atomicCAS(args.err_flag, 0, SCFA_ERR_NUMERIC);  // inf / NaN
          const float m_use = (m_run == NEG_INF) ? 0.f : m_run;
          args.out0[so] = dead ? NEG_INF : m_true * LN2;             // M
          args.out1[so] = dead ? 0.f : l_run * ex2(m_use - m_true);  // L relative to M
          args.out_lse2[roff] = dead ? INFINITY : (m_use + __log2f(l_run));
        } else {
          args.out_lse2[roff] = INFINITY;  // pad slot: read (never used) by the dK/dV column loads
        }
      } else {
        // ---------------- backward passes: P and dS recomputed from (lse2, delta)
        float my_nlse = 0.f, my_ndelta = 0.f;
        const int pc0 = pcr;  // BWD: pair index of this item's tiles 0 / 1
        pcr += (n + 1) >> 1;
        if (kMode == MODE_DQ) {
          my_nlse = -args.lse2[roff];
          if (args.delta_out) {
            // fused delta = rowsum(dO * O) (qk_sparse.py:168): O row from global, dO row
            // from the stationary tile in shared memory.  Summed as the delta passes do
            // (scfa_bwd_prep*: one partial per 16-byte piece, then an xor-butterfly), so
            // every path gives the same bits.
            float dl = 0.f;
            float part[kD / 8];
            if (n > 0 && row < args.T_rows) {
              const size_t orow_o = args.x_rows ? static_cast<size_t>(my_idx)
                                                : static_cast<size_t>(bh) * args.T_rows + row;
              const uint4* op = reinterpret_cast<const uint4*>(args.o_src + orow_o * kD);
              uint4 ov[kD / 8];
#pragma unroll
              for (int j = 0; j < kD / 8; ++j) ov[j] = __ldg(op + j);
              mbar_wait(bar_x_full + (ia % C::NXS), (ia / C::NXS) & 1);
              const uint8_t* dob = smem + C::OFF_X + (ia % C::NXS) * C::XSLOT_BYTES + C::X_BYTES;
#pragma unroll
              for (int j = 0; j < kD / 8; ++j) {
                const uint32_t addr =
                    smem_u32(dob + (j >> 3) * C::BM * 128 + r * 128 + (((j & 7) ^ (r & 7)) << 4));
                uint4 dv4;
                asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                             : "=r"(dv4.x), "=r"(dv4.y), "=r"(dv4.z), "=r"(dv4.w)
                             : "r"(addr));
                const __nv_bfloat162* a2 = reinterpret_cast<const __nv_bfloat162*>(&ov[j]);
                const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&dv4);
                float acc = 0.f;
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  const float2 x = __bfloat1622float2(a2[e]);
                  const float2 y = __bfloat1622float2(b2[e]);
                  acc = fmaf(x.x, y.x, acc);
                  acc = fmaf(x.y, y.y, acc);
                }
                part[j] = acc;
              }
#pragma unroll
              for (int w = kD / 16; w >= 1; w >>= 1) {
#pragma unroll
                for (int i = 0; i < w; ++i) part[i] = part[i] + part[i + w];
              }
              dl = part[0];
            }
            args.delta_out[roff] = dl;
            my_ndelta = -dl;
          } else {
            my_ndelta = -args.delta[roff];
          }
        }
        // ALT: this warpgroup takes the stream's tiles with tg % 2 == wg, in TMEM buffer tg % NBUF
        for (int t = 0; t < n; ++t, ++tg) {
          const int entry = entry_next;
          if (t + 1 < n) entry_next = lst[t + 1];
          if (C::ALT && (tg & 1) != wg) continue;
          const int jb = C::ALT ? (tg % C::NBUF) : 0;
          const uint32_t t_sb = t_s + jb * C::TM_BUF, t_dpb = t_dp + jb * C::TM_BUF;
          const uint32_t t_pb = t_p + jb * C::TM_BUF, t_p2b = t_p2 + jb * C::TM_BUF;
          const bool full = (entry & 0x8000) != 0;
          const int col0 = (entry & 0x7fff) * C::BN;
          SCFA_STAMP(0);
          mbar_wait(bar_s_full + jb, C::ALT ? ((tg / C::NBUF) & 1) : (tg & 1));
          SCFA_STAMP(1);
          tc_fence_after();
          const float* clse = nullptr;
          const float* cdelta = nullptr;
          if (C::KEYS) {
            const int s0 = tg % C::NS0;
            mbar_wait(bar_y0_full + s0, (tg / C::NS0) & 1);  // acquire the per-column lse/delta
            clse = reinterpret_cast<const float*>(smem + C::OFF_AUX + s0 * C::AUX_BYTES);
            cdelta = clse + C::BN;
          }
          // BWD: this tile's dS goes to half (t & 1) of pair buffer pc % 2, free once the dQ
          // MMAs of the pair two before have read it
          const int pc = pc0 + (t >> 1);
          uint8_t* ds_row = smem + C::OFF_DS + (pc & 1) * C::DS_PAIR + (t & 1) * C::DS_ATOM + r * 128;
          if (C::FUSED && pc >= 2) mbar_wait(B.ds_free + (pc & 1), ((pc >> 1) - 1) & 1);
          SCFA_STAMP(10);
          uint32_t vis[NW];
          if (full) {
#pragma unroll
            for (int i = 0; i < NW; ++i) vis[i] = 0xffffffffu;
          } else {
            run_mask<NW>(run.x - col0, run.y - col0, vis);
          }
          bool dp_ok = false;  // SDP_SPLIT: this tile's dP commit waited for
          (void)dp_ok;
          // 32-column chunks: read S and dP, compute P (and dS), store them over the
          // columns already read (chunk k's P / dS land in columns [16k, 16k+16) of S / dP)
#pragma unroll
          for (int cc = 0; cc < C::BN; cc += 32) {
            uint32_t pk_p[16], pk_ds[16];
            // a chunk no row of this warp can see: P = dS = 0 without loading S / dP or any
            // exponential (bitwise the masked result)
            if (!full && !__any_sync(0xffffffffu, vis[cc >> 5] != 0u)) {
              if (!C::ALT && C::OVERLAP && cc + 32 == C::BN) {
                tc_fence_before();
                mbar_arrive(bar_s_free);
              }
#pragma unroll
              for (int i = 0; i < 16; ++i) {
                pk_p[i] = 0u;
                pk_ds[i] = 0u;
              }
            } else if constexpr (C::SDP_SPLIT) {
            // P from S first; dP (its own commit) is waited for once per tile, after the first
            // loaded chunk's exponentials
            float sv[32], dv[32];
            const MBar dp_full = C::KEYS ? B.dq_full + jb : bar_s_full + 1;
            const uint32_t dp_par = C::ALT ? ((tg / C::NBUF) & 1) : (tg & 1);
            auto p_in_place = [&]() {
#pragma unroll
              for (int c = 0; c < 32; c += 2) {
                float p0, p1, n0 = my_nlse, n1 = my_nlse;
                if (C::KEYS) {
                  n0 = -clse[cc + c];
                  n1 = -clse[cc + c + 1];
                }
                fma2(p0, p1, sv[c], sv[c + 1], sl, sl, n0, n1);
                p0 = ex2(p0);
                p1 = ex2(p1);
                const uint32_t wv = vis[(cc + c) >> 5];
                sv[c] = ((wv >> ((cc + c) & 31)) & 1u) ? p0 : 0.f;
                sv[c + 1] = ((wv >> ((cc + c + 1) & 31)) & 1u) ? p1 : 0.f;
              }
            };
            if (cc == 0) {
              tmem_ld32(t_sb + cc, *reinterpret_cast<uint32_t(*)[32]>(sv));
              tmem_wait_ld();
              p_in_place();
              mbar_wait(dp_full, dp_par);
              tc_fence_after();
              dp_ok = true;
              tmem_ld32(t_dpb + cc, *reinterpret_cast<uint32_t(*)[32]>(dv));
              tmem_wait_ld();
            } else {
              if (!dp_ok) {
                mbar_wait(dp_full, dp_par);
                tc_fence_after();
                dp_ok = true;
              }
              tmem_ld32(t_sb + cc, *reinterpret_cast<uint32_t(*)[32]>(sv));
              tmem_ld32(t_dpb + cc, *reinterpret_cast<uint32_t(*)[32]>(dv));
              tmem_wait_ld();
              p_in_place();
            }
            if (!C::ALT && C::OVERLAP && cc + 32 == C::BN) {
              tc_fence_before();
              mbar_arrive(bar_s_free);
            }
#pragma unroll
            for (int c = 0; c < 32; c += 2) {
              float d0, d1, n0 = my_ndelta, n1 = my_ndelta;
              if (C::KEYS) {
                n0 = -cdelta[cc + c];
                n1 = -cdelta[cc + c + 1];
              }
              add2(d0, d1, dv[c], dv[c + 1], n0, n1);
              mul2(d0, d1, d0, d1, sv[c], sv[c + 1]);
              pk_ds[c >> 1] = pack_bf16(d0, d1);
              if (C::KEYS) pk_p[c >> 1] = pack_bf16(sv[c], sv[c + 1]);
            }
            } else {
            float sv[32], dv[32];
            tmem_ld32(t_sb + cc, *reinterpret_cast<uint32_t(*)[32]>(sv));
            tmem_ld32(t_dpb + cc, *reinterpret_cast<uint32_t(*)[32]>(dv));
            tmem_wait_ld();
            if (!C::ALT && C::OVERLAP && cc + 32 == C::BN) {
              tc_fence_before();
              mbar_arrive(bar_s_free);
            }
#pragma unroll
            for (int c = cc; c < cc + 32; c += 4) {
              float nl[4], nd[4];
              if (kMode == MODE_DQ) {
#pragma unroll
                for (int e = 0; e < 4; ++e) { nl[e] = my_nlse; nd[e] = my_ndelta; }
              } else {
                const float4 a4 = *reinterpret_cast<const float4*>(clse + c);
                const float4 b4 = *reinterpret_cast<const float4*>(cdelta + c);
                nl[0] = -a4.x; nl[1] = -a4.y; nl[2] = -a4.z; nl[3] = -a4.w;
                nd[0] = -b4.x; nd[1] = -b4.y; nd[2] = -b4.z; nd[3] = -b4.w;
              }
#pragma unroll
              for (int e = 0; e < 4; e += 2) {
                float p0, p1, d0, d1;
                fma2(p0, p1, sv[c - cc + e], sv[c - cc + e + 1], sl, sl, nl[e], nl[e + 1]);
                if (kPolyPair((c - cc + e) >> 1)) {
                  ex2_poly2(p0, p1, p0, p1);  // part of the exponentials on the FMA pipe
                } else {
                  p0 = ex2(p0);
                  p1 = ex2(p1);
                }
                const uint32_t wv = vis[(c + e) >> 5];
                p0 = ((wv >> ((c + e) & 31)) & 1u) ? p0 : 0.f;
                p1 = ((wv >> ((c + e + 1) & 31)) & 1u) ? p1 : 0.f;
                add2(d0, d1, dv[c - cc + e], dv[c - cc + e + 1], nd[e], nd[e + 1]);
                mul2(d0, d1, d0, d1, p0, p1);
                pk_p[(c - cc + e) >> 1] = pack_bf16(p0, p1);
                pk_ds[(c - cc + e) >> 1] = pack_bf16(d0, d1);
              }
            }
            }
            if (!C::ALT && cc == 0) {  // the previous tile's accumulate MMAs read these columns
              if (tg > 0) mbar_wait(bar_p_free, (tg - 1) & 1);
              tc_fence_after();
            }
            if (kMode == MODE_DQ) {
              tmem_st16(t_pb + cc / 2, pk_ds);
            } else {
              tmem_st16(t_pb + cc / 2, pk_p);
              tmem_st16(t_p2b + cc / 2, pk_ds);
            }
            if (C::FUSED) {
              // dS row of this key: 32 queries = four 16-byte chunks, 128-byte swizzle (as TMA
              // writes an SW128 tile), the MN-major image the dQ MMA reads
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                const int c = cc / 8 + i;
                const uint32_t addr = smem_u32(ds_row + ((c ^ (r & 7)) << 4));
                asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(pk_ds[4 * i]),
                             "r"(pk_ds[4 * i + 1]), "r"(pk_ds[4 * i + 2]), "r"(pk_ds[4 * i + 3])
                             : "memory");
              }
            }
          }
          if (C::FUSED) fence_proxy_async_smem();  // dS visible to the tensor core before p_full
          tmem_wait_st();
          tc_fence_before();
          mbar_arrive(bar_p_full + jb);
          SCFA_STAMP(2);
        }
        if (n > 0) {  // accumulators to the epilogue (ALT: it follows the work ring itself)
          if (!C::ALT) handoff(lb, n, 0.f);
          ++ia;
        } else if (!C::ALT && live) {
#pragma unroll
          for (int o = 0; o < (C::KEYS ? 2 : 1); ++o) {
            float4* d4 = reinterpret_cast<float4*>(((o == 0) ? args.out0 : args.out1) + orow * kD);
#pragma unroll
            for (int i = 0; i < kD / 4; ++i) d4[i] = make_float4(0.f, 0.f, 0.f, 0.f);
          }
        }
      }
    }
    if (!C::ALT && (!C::SPLIT || wg == 0)) handoff(-1, 0, 0.f);  // end of the stream
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 13) {
    tc_fence_after();
    tmem_dealloc<C::TM_COLS>(*tmem_slot);
  }
  if (threadIdx.x == 0) {  // the last CTA to finish re-arms the work counter for the next launch
    int* work_ctr = const_cast<int*>(args.list_count) + args.n_items;  // [0] next item, [1] CTAs done
    __threadfence();
    if (atomicAdd(work_ctr + 1, 1) == static_cast<int>(gridDim.x) - 1) {
      work_ctr[0] = 0;
      work_ctr[1] = 0;
      __threadfence();
    }
  }
}

// ------------------------------------------------------------------ host side

// Row-table map for tile::gather4 / tile::scatter4: a [nrows, D] matrix of elem_bytes
// elements, one 128-byte column window (64 bf16 / 32 fp32) per box row.
static int make_row_map(CUtensorMap* map, const void* base, long long nrows, int D, int elem_bytes) {
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(D), static_cast<cuuint64_t>(nrows > 0 ? nrows : 1)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(D) * elem_bytes};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(128 / elem_bytes), 1};
  return encode_tensor_map(map, elem_bytes, 2, base, dims, strides, box);
}

static int make_map(CUtensorMap* map, const void* base, int BH, int T, int D, int box_rows) {
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(D), static_cast<cuuint64_t>(T), static_cast<cuuint64_t>(BH)};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(D) * 2, static_cast<cuuint64_t>(T) * D * 2};
  cuuint32_t box[3] = {64, static_cast<cuuint32_t>(box_rows), 1};
  cuuint32_t estr[3] = {1, 1, 1};
  return encode_tensor_map_bf16_3d(map, base, dims, strides, box, estr);
}

static long long* g_dbg_buf = nullptr;
static int g_dbg_tiles = 0;
static int g_per_sm[4][2] = {};  // resident CTAs per SM chosen per (mode, D); 0 = not launched yet

static int sm_count() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

template <int kMode, int kD>
static int launch_mode(const AttnLaunch& L, cudaStream_t stream) {
  using C = Cfg<kMode, kD>;
  CUtensorMap mx0, mx1, my0, my1, mxo;
  int rc = 0;
  if (L.x_rows) {
    if (L.x0_tiled) {
      rc |= make_map(&mx0, L.x0_tiled, L.BH, L.T_rows, kD, C::BM);
    } else {
      rc |= make_row_map(&mx0, L.x0, L.x_nrows, kD, 2);
    }
    rc |= make_row_map(&mx1, L.x1 ? L.x1 : L.x0, L.x_nrows, kD, 2);
  } else {
    rc |= make_map(&mx0, L.x0, L.BH, L.T_rows, kD, C::BM);
    rc |= make_map(&mx1, L.x1 ? L.x1 : L.x0, L.BH, L.T_rows, kD, C::BM);
  }
  if (L.y_rows) {
    rc |= make_row_map(&my0, L.y0, L.y_nrows, kD, 2);
    rc |= make_row_map(&my1, L.y1, L.y_nrows, kD, 2);
  } else {
    rc |= make_map(&my0, L.y0, L.BH, L.T_cols, kD, C::BN);
    rc |= make_map(&my1, L.y1, L.BH, L.T_cols, kD, C::BN);
  }
  const bool writeout = L.x_rows && L.x_out && (kMode == MODE_FWD || kMode == MODE_DQ);
  rc |= writeout ? make_map(&mxo, L.x_out, L.BH, L.T_rows, kD, C::BM) : make_map(&mxo, L.x0, 1, 1, kD, C::BM);
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
  a.row_runs = reinterpret_cast<const int2*>(L.row_runs);
  a.x_rows = L.x_rows;
  a.out_rows = L.out_rows;
  a.y_rows = L.y_rows;
  a.x_writeout = writeout ? 1 : 0;
  a.x0_tiled = (L.x_rows && L.x0_tiled && kMode == MODE_DQ) ? 1 : 0;
  a.o_src = static_cast<const __nv_bfloat16*>(L.o_src);
  a.delta_out = L.delta_out;
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
  a.col_idx = L.col_idx;
  a.out2 = L.out2;
  a.T_out_cols = L.T_out_cols;
  a.scale_log2 = L.scale * 1.4426950408889634f;
  a.scale = L.scale;
  a.err_flag = L.err_flag;
  a.dbg = g_dbg_buf;
  a.dbg_tiles = g_dbg_tiles;
  auto kern = scfa_attn_kernel<kMode, kD>;
  static bool attr = false;  // one persistent CTA per SM, C::NSTREAM item streams in it
  if (!attr) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM_BYTES) != cudaSuccess)
      return SCFA_ERR_CUDA;
    g_per_sm[kMode][kD == 64 ? 0 : 1] = C::NSTREAM;
    attr = true;
  }
  if (a.n_items == 0) return SCFA_OK;
  int grid = sm_count();
  if (grid * C::NSTREAM > a.n_items) grid = (a.n_items + C::NSTREAM - 1) / C::NSTREAM;
  kern<<<grid, C::THREADS, C::SMEM_BYTES, stream>>>(mx0, mx1, my0, my1, mxo, a);
  return cudaGetLastError() == cudaSuccess ? SCFA_OK : SCFA_ERR_CUDA;
}

#ifndef SCFA_ONLY
#define SCFA_ONLY(m, d) 1
#endif
int launch_attention(const AttnLaunch& L, cudaStream_t stream) {
#if SCFA_ONLY(0, 64)
  if (L.D == 64 && L.mode == MODE_FWD) return launch_mode<MODE_FWD, 64>(L, stream);
#endif
#if SCFA_ONLY(1, 64)
  if (L.D == 64 && L.mode == MODE_DQ) return launch_mode<MODE_DQ, 64>(L, stream);
#endif
#if SCFA_ONLY(2, 64)
  if (L.D == 64 && L.mode == MODE_DKDV) return launch_mode<MODE_DKDV, 64>(L, stream);
#endif
#if SCFA_ONLY(3, 64)
  if (L.D == 64 && L.mode == MODE_BWD) return launch_mode<MODE_BWD, 64>(L, stream);
#endif
#if SCFA_ONLY(0, 128)
  if (L.D == 128 && L.mode == MODE_FWD) return launch_mode<MODE_FWD, 128>(L, stream);
#endif
#if SCFA_ONLY(1, 128)
  if (L.D == 128 && L.mode == MODE_DQ) return launch_mode<MODE_DQ, 128>(L, stream);
#endif
#if SCFA_ONLY(2, 128)
  if (L.D == 128 && L.mode == MODE_DKDV) return launch_mode<MODE_DKDV, 128>(L, stream);
#endif
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

extern "C" int scfa_debug_ctas_per_sm(int mode, int64_t D) {
  if (mode < 0 || mode > 3 || (D != 64 && D != 128)) return -1;
  return scfa::g_per_sm[mode][D == 64 ? 0 : 1];
}
