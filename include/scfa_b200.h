/* scfa_b200.h — C ABI of the B200 Sparse Causal Flash Attention engine.
 *
 * Drop-in boundary for the QK-sparse and hash-sparse attention path of the
 * reference `scfa` package (a NumPy package; its "FFI" is the Python API it
 * exports from pkg/src/scfa/__init__.py:10-90).  Every entry point below
 * replaces one reference function, cited as file:line under /root/reference.
 *
 * Conventions
 *   - All pointers are DEVICE pointers; every call is stream-ordered on the
 *     caller's `stream` (cudaStream_t passed as void*) and never synchronises.
 *   - Caller owns every buffer (including workspace); the library allocates
 *     nothing persistent.  Buffer sizes are stated per function.
 *   - Return value: SCFA_OK or one of the SCFA_ERR_* codes, which map 1:1 to
 *     the reference exception taxonomy (pkg/src/scfa/errors.py:4-29).
 *     scfa_last_error() returns a thread-local message for the last failure.
 *   - Data-dependent contract violations found on the device (keep values
 *     outside {0,1}, negative bucket ids, unsorted batches ...) are reported
 *     through an int32 `err_flag` in device memory (0 = ok, else SCFA_ERR_*),
 *     so that the host decides when to synchronise.
 *   - Layouts: boundary (B, T, H, D) and engine (B, H, T, D) are both
 *     accepted through explicit element strides; attention operands are
 *     engine-layout, contiguous, bf16.  Index/bucket vectors consumed by the
 *     schedule are int32, one row of T_pad entries per (b, h)
 *     (T_pad = round_up(T, 128)), produced by scfa_build_aux / scfa_pack_index.
 */
#ifndef SCFA_B200_H
#define SCFA_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SCFA_OK 0
#define SCFA_ERR_SHAPE 1     /* ShapeError     (errors.py:8-9)   */
#define SCFA_ERR_FORMAT 2    /* FormatError    (errors.py:12-17) */
#define SCFA_ERR_PARAM 3     /* ParameterError (errors.py:20-21) */
#define SCFA_ERR_NUMERIC 4   /* NumericError   (errors.py:24-25) */
#define SCFA_ERR_CONTRACT 5  /* ContractError  (errors.py:28-29) */
#define SCFA_ERR_CUDA 6      /* launch / driver failure (no reference analogue) */

/* dtype codes for index-like inputs */
#define SCFA_DT_F32 0
#define SCFA_DT_F64 1
#define SCFA_DT_U8 2
#define SCFA_DT_I32 3
#define SCFA_DT_I64 4
#define SCFA_DT_BF16 5 /* activations only (scfa_lsh_buckets) */

/* attention flags */
#define SCFA_FLAG_EXCLUDE_SELF 1 /* strict causality q_idx > k_idx (_kernel.py:83-84) */
#define SCFA_FLAG_HASH 2         /* also require q_hash == k_hash (_kernel.py:87-88)  */

int scfa_abi_version(void);
const char* scfa_last_error(void);

/* ---------------------------------------------------------------- QK prep
 * Replaces compact()'s stable argsort of ~keep (pkg/src/scfa/qk_sparse.py:41-71).
 * keep: (B,T,H) with element strides (sb, st, sh), dtype code `keep_dtype`,
 *       entries must be 0 or 1 (else *err_flag = SCFA_ERR_SHAPE, qk_sparse.py:54-55).
 * perm   (B*H, T) int32: slot -> position; kept positions ascending, then
 *        dropped positions ascending == argsort(~kept, stable).
 * rank   (B*H, T) int32: position -> slot (inverse of perm).
 * counts (B*H)    int32: kept count per head (indices_per_head).            */
int scfa_qk_compact(const void* keep, int keep_dtype, int64_t B, int64_t T, int64_t H, int64_t sb,
                    int64_t st, int64_t sh, int32_t* perm, int32_t* rank, int32_t* counts,
                    int32_t* err_flag, void* stream);

/* Fused QK preparation for the static-size fused fwd + bwd (ABI 6), one launch for what
 * qk_preprocess does per head (pkg/src/scfa/qk_sparse.py:186-211) with the compacted buffer
 * holding every position (kept first, in position order, then the dropped ones) instead of
 * the max kept count (qk_sparse.py:58), so no size is read back to the host:
 *   perm_q / rank_q (B*H, T_Q), perm_k / rank_k (B*H, T_KV) int32: argsort(~kept, stable)
 *     (qk_sparse.py:59) and its inverse;
 *   q_idx (B*H, Tq_pad), k_idx (B*H, Tkv_pad) int32: pad_index (qk_sparse.py:74-83) —
 *     QUERY_PAD / KEY_PAD for dropped slots, past the end -1 / INT32_MAX;
 *   q_runs / k_runs (B*H, T*_pad) int32 pairs: the causal visibility runs of
 *     scfa_build_schedule (a kept query at t sees key slots [0, #kept keys <= t));
 *   q_rows / k_rows (B*H, T*_pad) int32: slot -> row (b*T + t)*H + h of the caller's
 *     (B, T, H, D) tensors (scfa_row_map);
 *   counts (2*B*H) int32: kept queries per head, then kept keys.
 * keep_q / keep_k: (B, T, H) with element strides; entries outside {0, 1} set SCFA_ERR_SHAPE in
 * *err_flag (qk_sparse.py:54-55).  T_Q, T_KV <= 16384.                                   */
int scfa_qk_prepare(const void* keep_q, int keep_q_dtype, int64_t sbq, int64_t stq, int64_t shq,
                    const void* keep_k, int keep_k_dtype, int64_t sbk, int64_t stk, int64_t shk, int64_t B,
                    int64_t T_Q, int64_t T_KV, int64_t H, int32_t* perm_q, int32_t* rank_q, int32_t* perm_k,
                    int32_t* rank_k, int32_t* q_idx, int32_t* k_idx, int32_t* q_runs, int32_t* k_runs,
                    int32_t* q_rows, int32_t* k_rows, int32_t* counts, int32_t* err_flag, void* stream);

/* ---------------------------------------------------------------- hash prep
 * Replaces _bucket_order / sort_by_bucket's stable argsort
 * (pkg/src/scfa/hash_sparse.py:89-133).  Stable LSD radix sort per (b,h) by
 * bucket id; with `pos` given (element strides ps_bh, ps_t; dtype pos_dtype),
 * the order is lexicographic (bucket, position) as the reference's
 * hash*span+idx key.  Bucket ids must be in [0, 2^31) (negative -> ShapeError,
 * hash_sparse.py:112-113).
 * hash: element (b,h,t) at b*sb + h*sh + t*st.   perm/rank: (B*H, T) int32.
 * scratch: (B*H, T) int32 workspace.                                          */
int scfa_hash_sort(const void* hash, int hash_dtype, int64_t B, int64_t T, int64_t H, int64_t sb,
                   int64_t st, int64_t sh, const void* pos, int pos_dtype, int64_t ps_bh,
                   int64_t ps_t, int32_t* perm, int32_t* rank, int32_t* scratch, int32_t* err_flag,
                   void* stream);

/* Fused hash preparation for SHARED bucket ids (q_hash is k_hash, T_Q == T_KV,
 * positions = arange: the reference's bench / LM setting, cli.py:481-487).
 * One launch replaces scfa_hash_sort + 2 x scfa_build_aux + the run pass of
 * scfa_build_schedule: the stable sort of _bucket_order (hash_sparse.py:89-94),
 * the sorted idx / hash vectors of sort_by_bucket (hash_sparse.py:127-133) and
 * the visibility runs for `flags` (SCFA_FLAG_EXCLUDE_SELF).  T <= 16384.
 * perm/rank (B*H, T); scratch (B*H, T + 257); q_idx/k_idx/q_hash/k_hash (B*H, T_pad) with the
 * same sentinels as scfa_build_aux; q_runs/k_runs (B*H, T_pad) int32 pairs as
 * scfa_build_schedule (pass runs_ready = 3 there); rows (optional, B*H x T_pad) the
 * scfa_row_map table of the sorted order for gather-mode attention.
 * sorted_event (optional cudaEvent_t) is recorded on `stream` as soon as perm and rank
 * are final (between the sort and the finishing launch), so a caller can start the
 * bucket-order row copies on another stream under the rest of the preparation.  */
int scfa_hash_prepare(const void* hash, int hash_dtype, int64_t B, int64_t T, int64_t H, int64_t sb,
                      int64_t st, int64_t sh, int flags, int32_t* perm, int32_t* rank, int32_t* scratch,
                      int32_t* q_idx, int32_t* k_idx, int32_t* q_hash, int32_t* k_hash, int32_t* q_runs,
                      int32_t* k_runs, int32_t* rows, int32_t* err_flag, void* sorted_event,
                      void* stream);

/* Row tables for the gather-mode attention kernels: rows[bh, s] = (b * T_src + perm[bh, s])
 * * H + h, the row of slot s of slice bh = (b, h) in a (B, T_src, H, D) tensor viewed as
 * [B*T_src*H, D]; slots s >= n_slots (up to T_pad) repeat the row of slot 0.  This is the
 * gather of compact() / sort_by_bucket (qk_sparse.py:68-70, hash_sparse.py:122-125) and the
 * inverse scatter of qk_postprocess / hash_scatter as an index table instead of a copy.
 * perm (B*H, T_perm) int32; rows (B*H, T_pad) int32.                               */
int scfa_row_map(const int32_t* perm, int64_t B, int64_t H, int64_t T_perm, int64_t n_slots,
                 int64_t T_pad, int64_t T_src, int32_t* rows, void* stream);

/* ---------------------------------------------------------------- gather / scatter
 * Row gather into engine layout (compact(...) take_along_axis, qk_sparse.py:68-70;
 * sort_by_bucket gather_rows, hash_sparse.py:122-125) fused with the
 * (B,T,H,D)->(B,H,T,D) transpose (to_heads, tensors.py:157-159).
 * src row (b, t, h) at b*sb + t*st + h*sh elements, D contiguous elements.
 * dst (B*H, n_slots, D) contiguous; dst[bh, s] = src[b, perm[bh, s], h].
 * elem_bytes: 2 (bf16/f16) or 4 (f32).                                        */
int scfa_gather_rows(const void* src, int elem_bytes, int64_t B, int64_t H, int64_t D, int64_t sb,
                     int64_t st, int64_t sh, const int32_t* perm, int64_t T_perm, int64_t n_slots,
                     void* dst, void* stream);

/* n (1..3) scfa_gather_rows in one launch (Q | K | V of one batch).  Host arrays:
 * srcs/dsts/perms[n]; strides[3n] = (sb, st, sh) per source; T_perm[n], n_slots[n].
 * All sources share elem_bytes, B, H, D.                                      */
int scfa_gather_rows3(int n, const void* const* srcs, void* const* dsts, const int32_t* const* perms,
                      const int64_t* strides, int elem_bytes, int64_t B, int64_t H, int64_t D,
                      const int64_t* T_perm, const int64_t* n_slots, void* stream);

/* Source-ordered variant of scfa_gather_rows3: rows are read in memory order and row
 * (b, t, h) is written to slot rank[b*H + h, t] of dst (B*H, n_slots, D) (slots >= n_slots
 * dropped).  ranks[n] are (B*H, T) int32 inverse permutations; strides as gather_rows3.  */
int scfa_permute_rows3(int n, const void* const* srcs, void* const* dsts, const int32_t* const* ranks,
                       const int64_t* strides, int elem_bytes, int64_t B, int64_t T, int64_t H, int64_t D,
                       const int64_t* n_slots, void* stream);

/* Inverse: dst row (b,t,h) = src[bh, rank[bh,t]] if rank < n_slots else 0.
 * Replaces qk_postprocess (qk_sparse.py:214-225) and hash_scatter +
 * from_heads (hash_sparse.py:216-220,238).  src (B*H, n_slots, D) contiguous
 * with element size src_bytes (2 = bf16, 4 = f32); dst strides (db, dt, dh)
 * elements of size dst_bytes (2 or 4).                                        */
int scfa_scatter_rows(const void* src, int src_bytes, int64_t B, int64_t H, int64_t T, int64_t D,
                      const int32_t* rank, int64_t n_slots, void* dst, int dst_bytes, int64_t db,
                      int64_t dt, int64_t dh, void* stream);

/* Per-slot index / bucket vectors for the kernels (pad_index, qk_sparse.py:74-83).
 * idx_out[bh, s] = pos[bh, perm[bh, s]] (pos NULL: perm[bh, s]) for s < counts[bh]
 *                  (counts NULL = all valid),
 *                  pad_value for counts[bh] <= s < n_slots, oob_value beyond.
 * hash_out (optional): bucket of perm[bh, s] read from `hash` (strides as in
 * scfa_hash_sort), hash_oob beyond n_slots.  Both (B*H, T_pad) int32.        */
int scfa_build_aux(const int32_t* perm, const int32_t* counts, int64_t B, int64_t H,
                   int64_t T_perm, int64_t n_slots, int64_t T_pad, int32_t pad_value,
                   int32_t oob_value, const void* hash, int hash_dtype, int64_t sb, int64_t st,
                   int64_t sh, int32_t hash_oob, const void* pos, int pos_dtype, int64_t ps_bh,
                   int64_t ps_t, int32_t* idx_out, int32_t* hash_out, void* stream);

/* rank[bh, idx[b, s, h]] = s for s < n_slots, n_slots elsewhere: the inverse
 * routing table behind qk_postprocess's put_along_axis (qk_sparse.py:218-224)
 * and hash_scatter (hash_sparse.py:216-220).  idx element (b,s,h) at
 * b*sb + s*ss + h*sh; out-of-range entries set *err_flag = SCFA_ERR_SHAPE.
 * rank (B*H, T) int32.                                                        */
int scfa_invert_index(const void* idx, int dtype, int64_t B, int64_t n_slots, int64_t H, int64_t sb,
                      int64_t ss, int64_t sh, int64_t T, int32_t* rank, int32_t* err_flag, void* stream);

/* Copy a caller index vector (element (bh,t) at bh*s_bh + t*s_t) into the
 * padded int32 kernel layout (B*H, T_pad), oob_value past T.                 */
int scfa_pack_index(const void* src, int dtype, int64_t BH, int64_t T, int64_t s_bh, int64_t s_t,
                    int64_t T_pad, int32_t oob_value, int32_t* dst, void* stream);

/* Contract checks (ContractError) on packed vectors.
 * qk: _check_padded/_check_indices (qk_sparse.py:95-117).
 * sorted: _check_sorted (hash_sparse.py:136-142).                           */
int scfa_validate_qk(const int32_t* q_idx, const int32_t* k_idx, int64_t BH, int64_t T_q,
                     int64_t T_kv, int64_t Tq_pad, int64_t Tkv_pad, int32_t* err_flag, void* stream);
int scfa_validate_sorted(const int32_t* idx, const int32_t* hash, int64_t BH, int64_t T,
                         int64_t T_pad, int32_t* err_flag, void* stream);

/* ---------------------------------------------------------------- schedules
 * scfa_build_schedule replaces the per-head schedules causal_j_stops
 * (_kernel.py:45-53) and hash_tile_ranges (_kernel.py:56-79), and the mask
 * construction of _tile_mask (_kernel.py:82-89).
 *
 * Visibility runs.  With keys sorted by position (QK / dense) or by
 * (bucket, position) (hash), the keys a query sees form ONE contiguous run of
 * key slots, and the queries that see a key form one run of query slots.
 *   q_runs (B*H, Tq_pad) int32 pairs [lo, hi): visible key slots of each query slot.
 *   k_runs (B*H, Tkv_pad) int32 pairs [lo, hi): query slots that see each key slot.
 * Slots past T get the empty run.  Either may be NULL if no list needs it.
 * runs_ready: bit 0 = q_runs already holds this problem's runs (not recomputed),
 * bit 1 = the same for k_runs.
 *
 * Tile lists (uint16 column-block ids, ascending; bit 15 = "every pair visible",
 * so no mask is needed).  They are exact: a tile is listed iff it holds at least
 * one visible pair.
 *   fwd : query rows in 128-row blocks x 128-key tiles   (scfa_attn_fwd)
 *   dq  : query rows in 128-row blocks x 64-key tiles    (scfa_attn_bwd_dq)
 *   dkdv: key rows in 128-row blocks x 64-query tiles    (scfa_attn_bwd_dkdv)
 * list_* (B*H, n_row_blocks, stride_*) with stride >= n_col_blocks; count_*
 * (3 * B*H * n_row_blocks + 4) int32 (ABI 6): the n = B*H*n_row_blocks counts, a
 * work-counter pair the attention kernels use to hand out items dynamically (zeroed here,
 * left zero by every launch), then at offset n + 2 + (n & 1) the order they hand them out in:
 * n {item, count} pairs, most tiles first (stable), so a persistent grid's last items are its
 * shortest.  A NULL list skips that list.  tiles[3] (may be
 * NULL) accumulates the listed-tile totals.  flags: SCFA_FLAG_*.            */
int scfa_build_schedule(const int32_t* q_idx, const int32_t* q_hash, const int32_t* k_idx,
                        const int32_t* k_hash, int64_t BH, int64_t T_q, int64_t T_kv, int64_t Tq_pad,
                        int64_t Tkv_pad, int flags, int32_t* q_runs, int32_t* k_runs,
                        int runs_ready, uint16_t* list_fwd, int32_t* count_fwd, int64_t stride_fwd, uint16_t* list_dq,
                        int32_t* count_dq, int64_t stride_dq, uint16_t* list_dkdv, int32_t* count_dkdv,
                        int64_t stride_dkdv, unsigned long long* tiles, void* stream);

/* Reference schedule at arbitrary BlockSpec(B_m, B_n) (tensors.py:63-78):
 * j_start/j_stop per query block exactly as causal_j_stops (flags without
 * SCFA_FLAG_HASH) or hash_tile_ranges (with it); tiles[bh] = sum(j_stop - j_start)
 * (FlashOutputs.tiles_computed, _kernel.py:28-29).  j_* (B*H, ceil(T_q/B_m)).  */
int scfa_ref_schedule(const int32_t* q_idx, const int32_t* q_hash, const int32_t* k_idx,
                      const int32_t* k_hash, int64_t BH, int64_t T_q, int64_t T_kv, int64_t Tq_pad,
                      int64_t Tkv_pad, int64_t B_m, int64_t B_n, int flags, int32_t* j_start,
                      int32_t* j_stop, int64_t* tiles, void* stream);

/* ---------------------------------------------------------------- attention
 * Forward: forward_head over the tile list (_kernel.py:92-123) via
 * qk_forward_kernel (qk_sparse.py:120-148) / hash_forward_kernel
 * (hash_sparse.py:145-179) / flash_forward (dense.py:33-63).
 * q (B*H, T_q, D), k/v (B*H, T_kv, D) bf16 contiguous, D in {64, 128}.
 * q_idx: padded query positions (output routing), q_runs / list_fwd / count_fwd
 * from scfa_build_schedule.  Causality, exclude_self and buckets are all encoded
 * in the runs.
 * o (B*H, T_q, D) bf16 (normalised output), m/l (B*H, T_q) f32 = FlashOutputs.M/L
 * (M = -inf, L = 0 for stranded rows), lse2 (B*H, Tq_pad) f32 log2-domain
 * logsumexp (+inf for stranded rows) consumed by the backward.
 * Output layout: out_boundary = 0 writes o as (B*H, T_q, D); out_boundary = 1 writes
 * row s of slice (b, h) to o[b, q_idx[bh, s], h, :] of a (B, T_out, H, D) tensor (H
 * heads) — the inverse scatter of qk_postprocess / hash_scatter fused into the
 * epilogue; pad rows (q_idx outside [0, T_out)) are not written.
 * Row tables (gather mode, ABI 3): with q_rows != NULL, q is a [R_q, D] row table (e.g. the
 * caller's (B, T, H, D) tensor, R_q = B*T*H) and slot s of slice bh is row q_rows[bh, s]
 * ((B*H, Tq_pad) int32, from scfa_row_map / scfa_hash_prepare); O is written to the same rows
 * of the [R_q, D] table `o` (this replaces out_boundary).  Likewise k_rows for k / v.  The
 * operands are then loaded with TMA tile::gather4: no compacted / sorted copies exist.
 * ABI 4: q_out (optional, needs q_rows) receives the gathered Q rows in kernel order as a
 * (B*H, T_q, D) bf16 tensor — each stationary tile is stored back with a TMA store once
 * loaded — so the backward passes can stream a sorted Q without a separate copy pass.
 * ABI 5: err_flag (optional, int32 device word) is set to SCFA_ERR_NUMERIC when a row's
 * output or softmax denominator is non-finite — the reference raises NumericError when o
 * turns non-finite inside update_stats (softmax.py:63-64).  First error code wins.     */
int scfa_attn_fwd(const void* q, const void* k, const void* v, int64_t BH, int64_t T_q,
                  int64_t T_kv, int64_t D, const int32_t* q_idx, const int32_t* q_runs,
                  int64_t Tq_pad, int64_t Tkv_pad, const uint16_t* list, const int32_t* list_count,
                  int64_t list_stride, float scale, int64_t H, int64_t T_out, int out_boundary,
                  void* o, float* m, float* l, float* lse2, const int32_t* q_rows,
                  const int32_t* k_rows, int64_t R_q, int64_t R_kv, void* q_out, int32_t* err_flag,
                  void* stream);

/* delta = rowsum(dO * O) (qk_sparse.py:168, hash_sparse.py:194, dense.py:81);
 * lse2 rebuilt from (M, L) when lse2_in is NULL (m_hat/inv_l, _kernel.py:152-154).
 * delta, lse2_out: (B*H, Tq_pad) f32 (pads: delta 0, lse2 +inf).
 * q_idx == NULL: o, d_out are (B*H, T_q, D).  q_idx != NULL (boundary mode): o, d_out
 * are (B, T_out, H, D) and row s of slice bh is read at position q_idx[bh, s]; the dO
 * rows are also written in kernel order to d_out_sorted (B*H, T_q, D) bf16 (pad rows 0). */
int scfa_bwd_prep(const void* o, const void* d_out, const float* lse2_in, const float* m,
                  const float* l, int64_t BH, int64_t T_q, int64_t D, int64_t Tq_pad,
                  const int32_t* q_idx, int64_t H, int64_t T_out, void* d_out_sorted, float* delta,
                  float* lse2_out, void* stream);

/* The same delta pass for shared hash ids (every position has a slot) driven from the
 * source side: o and d_out are (B, T, H, D) bf16 read in memory order; rank (B*H, T)
 * int32 position -> slot (scfa_hash_prepare); dO row (b, t, h) is written to slot
 * rank[bh, t] of d_out_sorted (B*H, T, D) and delta[bh, rank[bh, t]] = rowsum(dO * O)
 * (qk_sparse.py:168, hash_sparse.py:194); delta (B*H, Tq_pad) slots >= T are set to 0. */
int scfa_bwd_prep_rank(const void* o, const void* d_out, int64_t B, int64_t T, int64_t H, int64_t D,
                       int64_t Tq_pad, const int32_t* rank, void* d_out_sorted, float* delta, void* stream);

/* Zero the rows of dropped positions: for every (b, t, h) with keep[b*sb + t*st + h*sh]
 * == 0 (dtype keep_dtype), the row of out0 (row_bytes0 bytes at row (b*T + t)*H + h) and
 * of out1 (row_bytes1, may be NULL / 0) are set to 0.  With it the boundary-layout QK
 * outputs need no full zero-fill: the attention epilogues write every kept row and the
 * reference leaves dropped rows 0 (qk_postprocess, qk_sparse.py:214-225).              */
int scfa_zero_dropped(const void* keep, int keep_dtype, int64_t B, int64_t T, int64_t H, int64_t sb,
                      int64_t st, int64_t sh, void* out0, int64_t row_bytes0, void* out1,
                      int64_t row_bytes1, void* stream);

/* Backward pass 1 (dQ, query-block owner, _kernel.py:173-179).  q_runs, list_dq,
 * count_dq from scfa_build_schedule.  dq (B*H, T_q, D) f32, or (B, T_out, H, D)
 * scattered by q_idx when out_boundary (as scfa_attn_fwd), or the rows q_rows of a
 * [R_q, D] f32 table in gather mode (q / d_out row tables as in scfa_attn_fwd).
 * o != NULL fuses the delta pass: delta = rowsum(dO * O) (qk_sparse.py:168) is computed
 * per query slot from the O rows (addressed like d_out) and written to delta_out
 * (B*H, Tq_pad) for scfa_attn_bwd_dkdv; `delta` is then ignored.
 * ABI 4: do_out (optional, needs q_rows) receives the gathered dO rows in kernel order,
 * (B*H, T_q, D) bf16, for scfa_attn_bwd_dkdv's streamed operand.
 * ABI 6: q_sorted (optional, with q_rows): Q already in kernel order, (B*H, T_q, D) bf16 (the
 * forward's q_out) — loaded as tiled boxes; only dO goes through the row table.          */
int scfa_attn_bwd_dq(const void* q, const void* k, const void* v, const void* d_out, int64_t BH,
                     int64_t T_q, int64_t T_kv, int64_t D, const int32_t* q_idx,
                     const int32_t* q_runs, int64_t Tq_pad, int64_t Tkv_pad, const float* lse2,
                     const float* delta, const uint16_t* list, const int32_t* list_count,
                     int64_t list_stride, float scale, int64_t H, int64_t T_out, int out_boundary,
                     float* dq, const int32_t* q_rows, const int32_t* k_rows, int64_t R_q,
                     int64_t R_kv, const void* o, float* delta_out, void* do_out,
                     const void* q_sorted, void* stream);

/* Backward pass 2 (dK/dV, key-block owner over the transposed schedule,
 * _kernel.py:181-192).  k_runs, list_dkdv, count_dkdv from scfa_build_schedule.
 * dk, dv (B*H, T_kv, D) f32, or (B, T_out, H, D) scattered by k_idx when out_boundary,
 * or the rows k_rows of [R_kv, D] f32 tables in gather mode.
 * ABI 5: out_rows (optional, tiled operands only) routes key slot s of slice bh to row
 * out_rows[bh, s] of [B*T*H, D] dk / dv tables for every s < T_kv, pad slots included:
 * with the static QK compaction every dropped key has a pad slot whose dK / dV row is
 * zero, so the call writes every row and no zero-fill of dropped rows is needed.      */
int scfa_attn_bwd_dkdv(const void* q, const void* k, const void* v, const void* d_out, int64_t BH,
                       int64_t T_q, int64_t T_kv, int64_t D, const int32_t* k_idx,
                       const int32_t* k_runs, int64_t Tq_pad, int64_t Tkv_pad, const float* lse2,
                       const float* delta, const uint16_t* list, const int32_t* list_count,
                       int64_t list_stride, float scale, int64_t H, int64_t T_out, int out_boundary,
                       float* dk, float* dv, const int32_t* q_rows, const int32_t* k_rows,
                       int64_t R_q, int64_t R_kv, const int32_t* out_rows, void* stream);

/* Single-pass backward (ABI 5): dQ, dK, dV in one key-stationary sweep over the dK/dV
 * schedule (_kernel.py:139-193 with both of its passes fused).  Arguments as
 * scfa_attn_bwd_dkdv (engine-layout / kernel-order operands, no row tables) plus q_idx
 * (padded query positions, the dQ routing) and dq.  Each pair of 64-query tiles of a key
 * block issues dQ += scale * dS K on the tensor cores; the epilogue reduces it (fp32 add)
 * into dq, which the caller must zero-fill: (B*H, T_q, D) f32, or (B, Tq_out, H, D) at
 * the original positions when out_boundary.  dK / dV as scfa_attn_bwd_dkdv (Tkv_out).
 * D = 64 only.  dQ is not bitwise reproducible (the reduction order varies); dK / dV are. */
int scfa_attn_bwd(const void* q, const void* k, const void* v, const void* d_out, int64_t BH, int64_t T_q,
                  int64_t T_kv, int64_t D, const int32_t* q_idx, const int32_t* k_idx, const int32_t* k_runs,
                  int64_t Tq_pad, int64_t Tkv_pad, const float* lse2, const float* delta, const uint16_t* list,
                  const int32_t* list_count, int64_t list_stride, float scale, int64_t H, int64_t Tq_out,
                  int64_t Tkv_out, int out_boundary, float* dq, float* dk, float* dv, void* stream);

/* ---------------------------------------------------------------- diagnostics
 * Route per-tile clock64 stamps of subsequent attention launches into `buf`
 * (grid * tiles_per_cta * 8 int64; NULL disables).  Not part of the reference API. */
int scfa_debug_timing(void* buf, int64_t tiles_per_cta);

/* Resident CTAs per SM the attention launcher chose for pass `mode` (0 fwd, 1 dQ,
 * 2 dK/dV) at head dim D; 0 before the first launch, -1 for bad arguments.     */
int scfa_debug_ctas_per_sm(int mode, int64_t D);

/* Angular LSH bucket ids (lsh_buckets, hash_sparse.py:34-52) on the device.
 * x: (B, T, H, D) activations of dtype SCFA_DT_F32 / _F64 / _BF16 with element strides
 * (sb, st, sh, sd); R: (B*H, D, nb/2) float64 projections, contiguous (the reference draws
 * them per (b, h) from its Philox stream, tensors.py:86-93); out[b*ob + t*ot + h*oh] =
 * argmax([x R, -x R]) as int64 (first maximum).  Float64 arithmetic; nb even in [2, 64],
 * D <= 192.  Replaces the reference's per-(b, h) numpy loop (hash_sparse.py:44-51).     */
int scfa_lsh_buckets(const void* x, int x_dtype, int64_t B, int64_t T, int64_t H, int64_t D, int64_t sb,
                     int64_t st, int64_t sh, int64_t sd, const double* R, int nb, int64_t* out, int64_t ob,
                     int64_t ot, int64_t oh, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SCFA_B200_H */
