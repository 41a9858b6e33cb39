/* scfa_oracle.c — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference's tiled attention loop, used by the
 * tests as a second oracle and by bench.py as the CPU baseline / reference
 * arm ("kind": "port").  Never linked into the product library.
 *
 * Restated from /root/reference/pkg/src/scfa/:
 *   update_stats          softmax.py:35-65   (running max m, denominator l,
 *                                             normalised o; -inf -> 0 and
 *                                             1/0 -> 1 substitutions)
 *   forward_head          _kernel.py:92-123  (tile loop over [j_start, j_stop))
 *   _tile_mask            _kernel.py:82-89
 *   backward_head         _kernel.py:139-193 (dQ pass over query blocks, dK/dV
 *                                             pass over key blocks on the
 *                                             transposed schedule; P recomputed
 *                                             from (M, L) in both)
 *   causal_j_stops        _kernel.py:45-53
 *   hash_tile_ranges      _kernel.py:56-79
 * Work is split over (b, h) slices with a pthread pool, like map_heads
 * (tensors.py:178-189); results do not depend on the thread count.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <pthread.h>
#include <unistd.h>

typedef int64_t i64;

static i64 imin(i64 a, i64 b) { return a < b ? a : b; }

/* ---- tiny work-stealing pool over (b, h) slices ---- */
typedef void (*slice_fn)(void* ctx, i64 bh);
typedef struct {
  slice_fn fn;
  void* ctx;
  i64 n;
  i64 next;
} pool_t;

static void* pool_worker(void* arg) {
  pool_t* p = (pool_t*)arg;
  for (;;) {
    const i64 bh = __atomic_fetch_add(&p->next, 1, __ATOMIC_RELAXED);
    if (bh >= p->n) break;
    p->fn(p->ctx, bh);
  }
  return NULL;
}

int oracle_max_threads(void) {
  const long n = sysconf(_SC_NPROCESSORS_ONLN);
  return n > 0 ? (int)n : 1;
}

static void parallel_slices(i64 n, int threads, slice_fn fn, void* ctx) {
  if (threads <= 0) threads = oracle_max_threads();
  if (threads > n) threads = (int)n;
  pool_t p = {fn, ctx, n, 0};
  if (threads <= 1) {
    pool_worker(&p);
    return;
  }
  pthread_t* tid = (pthread_t*)malloc(sizeof(pthread_t) * threads);
  for (int t = 0; t < threads; ++t) pthread_create(&tid[t], NULL, pool_worker, &p);
  for (int t = 0; t < threads; ++t) pthread_join(tid[t], NULL);
  free(tid);
}

static void blk_minmax(const i64* a, i64 lo, i64 hi, i64* mn, i64* mx) {
  i64 x = INT64_MAX, y = INT64_MIN;
  for (i64 i = lo; i < hi; ++i) {
    if (a[i] < x) x = a[i];
    if (a[i] > y) y = a[i];
  }
  *mn = x;
  *mx = y;
}

/* causal_j_stops / hash_tile_ranges for one head. */
void oracle_schedule(const i64* q_idx, const i64* k_idx, const i64* q_hash, const i64* k_hash, i64 Tq, i64 Tkv,
                     i64 Bm, i64 Bn, i64* j_start, i64* j_stop) {
  const i64 nQ = (Tq + Bm - 1) / Bm, nK = (Tkv + Bn - 1) / Bn;
  for (i64 i = 0; i < nQ; ++i) {
    const i64 lo = i * Bm, hi = imin(Tq, lo + Bm);
    i64 mnq, mxq;
    blk_minmax(q_idx, lo, hi, &mnq, &mxq);
    if (!q_hash) {
      i64 c = 0;
      for (i64 j = 0; j < nK; ++j) {
        i64 mn, mx;
        blk_minmax(k_idx, j * Bn, imin(Tkv, (j + 1) * Bn), &mn, &mx);
        if (mn <= mxq) ++c;
      }
      j_start[i] = 0;
      j_stop[i] = c;
    } else {
      i64 mnqh, mxqh, a = 0, b = 0;
      blk_minmax(q_hash, lo, hi, &mnqh, &mxqh);
      for (i64 j = 0; j < nK; ++j) {
        i64 mn, mx;
        blk_minmax(k_hash, j * Bn, imin(Tkv, (j + 1) * Bn), &mn, &mx);
        if (mx < mnqh) ++a;
        if (mn <= mxqh) ++b;
      }
      i64 stop = a;
      for (i64 j = b - 1; j >= a; --j) {
        i64 mn, mx;
        blk_minmax(k_idx, j * Bn, imin(Tkv, (j + 1) * Bn), &mn, &mx);
        if (mn <= mxq) {
          stop = j + 1;
          break;
        }
      }
      j_start[i] = a;
      j_stop[i] = stop;
    }
  }
}

static int allowed(i64 qi, i64 ki, const i64* qh, const i64* kh, i64 r, i64 c, int excl) {
  int ok = excl ? (qi > ki) : (qi >= ki);
  if (qh) ok = ok && (qh[r] == kh[c]);
  return ok;
}

/* One (b, h) slice of forward_head. q (Tq, D), k/v (Tkv, D); o (Tq, D), m/l (Tq). */
static i64 forward_one(const float* q, const float* k, const float* v, const i64* qi, const i64* ki, const i64* qh,
                       const i64* kh, i64 Tq, i64 Tkv, i64 D, i64 Bm, i64 Bn, const i64* js, const i64* je, int excl,
                       double scale, float* o, float* m_out, float* l_out) {
  const i64 nQ = (Tq + Bm - 1) / Bm;
  float* s = (float*)malloc(sizeof(float) * Bm * Bn);
  i64 tiles = 0;
  for (i64 i = 0; i < nQ; ++i) {
    const i64 lo = i * Bm, hi = imin(Tq, lo + Bm), R = hi - lo;
    for (i64 r = 0; r < R; ++r) {
      m_out[lo + r] = -INFINITY;
      l_out[lo + r] = 0.f;
      memset(o + (lo + r) * D, 0, sizeof(float) * D);
    }
    for (i64 j = js[i]; j < je[i]; ++j) {
      const i64 klo = j * Bn, khi = imin(Tkv, klo + Bn), C = khi - klo;
      for (i64 r = 0; r < R; ++r) {
        const float* qr = q + (lo + r) * D;
        for (i64 c = 0; c < C; ++c) {
          const float* kr = k + (klo + c) * D;
          float acc = 0.f;
          for (i64 d = 0; d < D; ++d) acc += qr[d] * kr[d];
          acc *= (float)scale;
          s[r * Bn + c] = allowed(qi[lo + r], ki[klo + c], qh ? qh + lo : NULL, kh ? kh + klo : NULL, r, c, excl)
                              ? acc
                              : -INFINITY;
        }
      }
      /* update_stats (softmax.py:35-65), row by row */
      for (i64 r = 0; r < R; ++r) {
        float* sr = s + r * Bn;
        float mx = -INFINITY;
        for (i64 c = 0; c < C; ++c) mx = sr[c] > mx ? sr[c] : mx;
        const float m_old = m_out[lo + r];
        const float m_new = mx > m_old ? mx : m_old;
        const float m_hat = isinf(m_new) && m_new < 0 ? 0.f : m_new;
        float l2 = 0.f;
        for (i64 c = 0; c < C; ++c) {
          sr[c] = expf(sr[c] - m_hat);
          l2 += sr[c];
        }
        float l_old = expf(m_old - m_hat) * l_out[lo + r];
        const float l_new = l_old + l2;
        float z = 1.f / l_new;
        if (isinf(z)) z = 1.f;
        l_old *= z;
        float* orow = o + (lo + r) * D;
        for (i64 d = 0; d < D; ++d) orow[d] *= l_old;
        for (i64 c = 0; c < C; ++c) {
          const float p = sr[c] * z;
          if (p == 0.f) continue;
          const float* vr = v + (klo + c) * D;
          for (i64 d = 0; d < D; ++d) orow[d] += p * vr[d];
        }
        m_out[lo + r] = m_new;
        l_out[lo + r] = l_new;
      }
      ++tiles;
    }
  }
  free(s);
  return tiles;
}

/* One (b, h) slice of backward_head (both passes). */
static void backward_one(const float* q, const float* k, const float* v, const float* dO, const float* delta,
                         const float* m_vec, const float* l_vec, const i64* qi, const i64* ki, const i64* qh,
                         const i64* kh, i64 Tq, i64 Tkv, i64 D, i64 Bm, i64 Bn, const i64* js, const i64* je,
                         int excl, double scale, float* dq, float* dk, float* dv) {
  const i64 nQ = (Tq + Bm - 1) / Bm, nK = (Tkv + Bn - 1) / Bn;
  float* p = (float*)malloc(sizeof(float) * Bm * Bn);
  float* ds = (float*)malloc(sizeof(float) * Bm * Bn);
  memset(dq, 0, sizeof(float) * Tq * D);
  memset(dk, 0, sizeof(float) * Tkv * D);
  memset(dv, 0, sizeof(float) * Tkv * D);
  /* probabilities and dS of tile (i, j) from the stored (M, L) (_tile_probs, _kernel.py:126-136) */
#define TILE(i, j)                                                                                     \
  const i64 lo = (i)*Bm, hi = imin(Tq, lo + Bm), R = hi - lo;                                          \
  const i64 klo = (j)*Bn, khi = imin(Tkv, klo + Bn), C = khi - klo;                                    \
  for (i64 r = 0; r < R; ++r) {                                                                        \
    const float mh = (isinf(m_vec[lo + r]) && m_vec[lo + r] < 0) ? 0.f : m_vec[lo + r];                \
    const float il = l_vec[lo + r] == 0.f ? 0.f : 1.f / l_vec[lo + r];                                 \
    const float* qr = q + (lo + r) * D;                                                                \
    const float* dr = dO + (lo + r) * D;                                                               \
    for (i64 c = 0; c < C; ++c) {                                                                      \
      float pv = 0.f, dp = 0.f;                                                                        \
      if (allowed(qi[lo + r], ki[klo + c], qh ? qh + lo : NULL, kh ? kh + klo : NULL, r, c, excl)) {   \
        const float* kr = k + (klo + c) * D;                                                           \
        float acc = 0.f;                                                                               \
        for (i64 d = 0; d < D; ++d) acc += qr[d] * kr[d];                                              \
        pv = expf(acc * (float)scale - mh) * il;                                                       \
      }                                                                                                \
      const float* vr = v + (klo + c) * D;                                                             \
      for (i64 d = 0; d < D; ++d) dp += dr[d] * vr[d];                                                 \
      p[r * Bn + c] = pv;                                                                              \
      ds[r * Bn + c] = pv * (dp - delta[lo + r]);                                                      \
    }                                                                                                  \
  }
  for (i64 i = 0; i < nQ; ++i) {
    for (i64 j = js[i]; j < je[i]; ++j) {
      TILE(i, j)
      for (i64 r = 0; r < R; ++r)
        for (i64 c = 0; c < C; ++c) {
          const float g = ds[r * Bn + c];
          if (g == 0.f) continue;
          const float* kr = k + (klo + c) * D;
          float* out = dq + (lo + r) * D;
          for (i64 d = 0; d < D; ++d) out[d] += g * kr[d];
        }
    }
  }
  for (i64 j = 0; j < nK; ++j) {
    for (i64 i = 0; i < nQ; ++i) {
      if (!(j >= js[i] && j < je[i])) continue;
      TILE(i, j)
      for (i64 r = 0; r < R; ++r) {
        const float* qr = q + (lo + r) * D;
        const float* dr = dO + (lo + r) * D;
        for (i64 c = 0; c < C; ++c) {
          const float pv = p[r * Bn + c], g = ds[r * Bn + c];
          float* ov = dv + (klo + c) * D;
          float* ok = dk + (klo + c) * D;
          if (pv != 0.f)
            for (i64 d = 0; d < D; ++d) ov[d] += pv * dr[d];
          if (g != 0.f)
            for (i64 d = 0; d < D; ++d) ok[d] += g * qr[d];
        }
      }
    }
  }
#undef TILE
  for (i64 x = 0; x < Tq * D; ++x) dq[x] *= (float)scale;
  for (i64 x = 0; x < Tkv * D; ++x) dk[x] *= (float)scale;
  free(p);
  free(ds);
}

/* Whole (B*H) grid.  Index/bucket arrays (BH, T); q_hash NULL = no buckets
 * (then j_start = 0, j_stop = causal_j_stops, as qk_forward_kernel / flash_forward). */
typedef struct {
  i64 Tq, Tkv, D, Bm, Bn;
  const float *q, *k, *v, *o, *m, *l, *dO;
  const i64 *q_idx, *k_idx, *q_hash, *k_hash;
  int excl;
  double scale;
  float *o_out, *m_out, *l_out, *dq, *dk, *dv;
  i64* tiles;
} job_t;

static void fwd_slice(void* ctx, i64 bh) {
  job_t* J = (job_t*)ctx;
  const i64 Tq = J->Tq, Tkv = J->Tkv, D = J->D, nQ = (Tq + J->Bm - 1) / J->Bm;
  i64* js = (i64*)malloc(sizeof(i64) * (nQ + 1));
  i64* je = (i64*)malloc(sizeof(i64) * (nQ + 1));
  const i64* qh = J->q_hash ? J->q_hash + bh * Tq : NULL;
  const i64* kh = J->k_hash ? J->k_hash + bh * Tkv : NULL;
  oracle_schedule(J->q_idx + bh * Tq, J->k_idx + bh * Tkv, qh, kh, Tq, Tkv, J->Bm, J->Bn, js, je);
  J->tiles[bh] = forward_one(J->q + bh * Tq * D, J->k + bh * Tkv * D, J->v + bh * Tkv * D, J->q_idx + bh * Tq,
                             J->k_idx + bh * Tkv, qh, kh, Tq, Tkv, D, J->Bm, J->Bn, js, je, J->excl, J->scale,
                             J->o_out + bh * Tq * D, J->m_out + bh * Tq, J->l_out + bh * Tq);
  free(js);
  free(je);
}

static void bwd_slice(void* ctx, i64 bh) {
  job_t* J = (job_t*)ctx;
  const i64 Tq = J->Tq, Tkv = J->Tkv, D = J->D, nQ = (Tq + J->Bm - 1) / J->Bm;
  i64* js = (i64*)malloc(sizeof(i64) * (nQ + 1));
  i64* je = (i64*)malloc(sizeof(i64) * (nQ + 1));
  float* delta = (float*)malloc(sizeof(float) * (Tq + 1));
  const i64* qh = J->q_hash ? J->q_hash + bh * Tq : NULL;
  const i64* kh = J->k_hash ? J->k_hash + bh * Tkv : NULL;
  oracle_schedule(J->q_idx + bh * Tq, J->k_idx + bh * Tkv, qh, kh, Tq, Tkv, J->Bm, J->Bn, js, je);
  /* delta = sum(dO * O, -1)  (qk_sparse.py:168) */
  for (i64 t = 0; t < Tq; ++t) {
    float acc = 0.f;
    for (i64 d = 0; d < D; ++d) acc += J->dO[(bh * Tq + t) * D + d] * J->o[(bh * Tq + t) * D + d];
    delta[t] = acc;
  }
  backward_one(J->q + bh * Tq * D, J->k + bh * Tkv * D, J->v + bh * Tkv * D, J->dO + bh * Tq * D, delta,
               J->m + bh * Tq, J->l + bh * Tq, J->q_idx + bh * Tq, J->k_idx + bh * Tkv, qh, kh, Tq, Tkv, D, J->Bm,
               J->Bn, js, je, J->excl, J->scale, J->dq + bh * Tq * D, J->dk + bh * Tkv * D, J->dv + bh * Tkv * D);
  free(js);
  free(je);
  free(delta);
}

i64 oracle_forward(i64 BH, i64 Tq, i64 Tkv, i64 D, const float* q, const float* k, const float* v, const i64* q_idx,
                   const i64* k_idx, const i64* q_hash, const i64* k_hash, i64 Bm, i64 Bn, int exclude_self,
                   double scale, int threads, float* o, float* m, float* l) {
  i64* tiles = (i64*)calloc((size_t)(BH + 1), sizeof(i64));
  job_t J = {Tq, Tkv, D, Bm, Bn, q, k, v, NULL, NULL, NULL, NULL, q_idx, k_idx, q_hash, k_hash,
             exclude_self, scale, o, m, l, NULL, NULL, NULL, tiles};
  parallel_slices(BH, threads, fwd_slice, &J);
  i64 total = 0;
  for (i64 bh = 0; bh < BH; ++bh) total += tiles[bh];
  free(tiles);
  return total;
}

void oracle_backward(i64 BH, i64 Tq, i64 Tkv, i64 D, const float* q, const float* k, const float* v, const float* o,
                     const float* m, const float* l, const float* dO, const i64* q_idx, const i64* k_idx,
                     const i64* q_hash, const i64* k_hash, i64 Bm, i64 Bn, int exclude_self, double scale,
                     int threads, float* dq, float* dk, float* dv) {
  job_t J = {Tq, Tkv, D, Bm, Bn, q, k, v, o, m, l, dO, q_idx, k_idx, q_hash, k_hash,
             exclude_self, scale, NULL, NULL, NULL, dq, dk, dv, NULL};
  parallel_slices(BH, threads, bwd_slice, &J);
}
