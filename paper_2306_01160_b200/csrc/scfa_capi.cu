// scfa_capi.cu — extern "C" attention entry points, error reporting, TMA descriptors.
#include <cudaTypedefs.h>

#include <cstdarg>
#include <cstdio>
#include <mutex>

#include "scfa_common.cuh"
#include "scfa_internal.h"

namespace scfa {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

int encode_tensor_map_bf16_3d(CUtensorMap* map, const void* base, const cuuint64_t* dims,
                              const cuuint64_t* strides_bytes, const cuuint32_t* box, const cuuint32_t* elem_strides) {
  auto fn = get_encode();
  if (!fn) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return 1;
  }
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides_bytes, box,
                  elem_strides, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d)", static_cast<int>(r));
    return 1;
  }
  return 0;
}

int encode_tensor_map(CUtensorMap* map, int dtype_bytes, int rank, const void* base, const cuuint64_t* dims,
                      const cuuint64_t* strides_bytes, const cuuint32_t* box) {
  auto fn = get_encode();
  if (!fn) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return 1;
  }
  cuuint32_t es[5] = {1, 1, 1, 1, 1};
  CUresult r = fn(map, dtype_bytes == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank,
                  const_cast<void*>(base), dims, strides_bytes, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d)", static_cast<int>(r));
    return 1;
  }
  return 0;
}

static int check_attn_args(int64_t BH, int64_t T_q, int64_t T_kv, int64_t D, int64_t Tq_pad, int64_t Tkv_pad,
                           const void* q, const void* k, const void* v) {
  if (D != 64 && D != 128) {
    set_error("head dim %lld unsupported (64 or 128)", static_cast<long long>(D));
    return SCFA_ERR_SHAPE;
  }
  if (Tq_pad < ((T_q + 127) / 128) * 128 || Tkv_pad < ((T_kv + 127) / 128) * 128) {
    set_error("padded index vectors too short");
    return SCFA_ERR_SHAPE;
  }
  if ((reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(k) | reinterpret_cast<uintptr_t>(v)) & 15) {
    set_error("operands must be 16-byte aligned");
    return SCFA_ERR_SHAPE;
  }
  if (BH > 65535) {
    set_error("too many (b, h) slices");
    return SCFA_ERR_SHAPE;
  }
  return SCFA_OK;
}

}  // namespace scfa

using namespace scfa;

extern "C" int scfa_abi_version(void) { return 6; }

extern "C" const char* scfa_last_error(void) { return g_err; }

extern "C" int scfa_attn_fwd(const void* q, const void* k, const void* v, int64_t BH, int64_t T_q, int64_t T_kv,
                             int64_t D, const int32_t* q_idx, const int32_t* q_runs, int64_t Tq_pad, int64_t Tkv_pad,
                             const uint16_t* list, const int32_t* list_count, int64_t list_stride, float scale,
                             int64_t H, int64_t T_out, int out_boundary, void* o, float* m, float* l, float* lse2,
                             const int32_t* q_rows, const int32_t* k_rows, int64_t R_q, int64_t R_kv, void* q_out,
                             int32_t* err_flag, void* stream) {
  int rc = check_attn_args(BH, T_q, T_kv, D, Tq_pad, Tkv_pad, q, k, v);
  if (rc) return rc;
  if (BH == 0 || T_q == 0) return SCFA_OK;
  if (q_out && !q_rows) {
    set_error("attn_fwd: q_out needs row tables (it is the gathered Q in kernel order)");
    return SCFA_ERR_PARAM;
  }
  AttnLaunch L{};
  L.mode = 0;
  L.x_out = q_out;
  L.err_flag = err_flag;
  L.D = static_cast<int>(D);
  L.BH = static_cast<int>(BH);
  L.H = static_cast<int>(H);
  L.T_out = static_cast<int>(T_out);
  L.out_boundary = out_boundary;
  L.T_rows = static_cast<int>(T_q);
  L.T_cols = static_cast<int>(T_kv > 0 ? T_kv : 1);
  L.T_rows_pad = static_cast<int>(Tq_pad);
  L.T_cols_pad = static_cast<int>(Tkv_pad);
  L.x0 = q;
  L.x1 = nullptr;
  // With no keys every row is stranded and no tile is listed; the streamed maps
  // then only need a valid address, never a load.
  L.y0 = T_kv > 0 ? k : q;
  L.y1 = T_kv > 0 ? v : q;
  if (T_kv == 0) L.T_cols = static_cast<int>(T_q);
  L.row_idx = q_idx;
  L.row_runs = q_runs;
  L.list = list;
  L.list_count = list_count;
  L.list_stride = static_cast<int>(list_stride);
  L.n_row_blocks = static_cast<int>((T_q + 127) / 128);
  L.x_rows = q_rows;
  L.y_rows = T_kv > 0 ? k_rows : nullptr;
  L.x_nrows = R_q;
  L.y_nrows = R_kv;
  L.out_o = static_cast<__nv_bfloat16*>(o);
  L.out0 = m;
  L.out1 = l;
  L.out_lse2 = lse2;
  L.scale = scale;
  rc = launch_attention(L, static_cast<cudaStream_t>(stream));
  if (rc && !g_err[0]) set_error("attention forward launch failed: %s", cudaGetErrorString(cudaGetLastError()));
  return rc;
}

extern "C" int scfa_attn_bwd_dq(const void* q, const void* k, const void* v, const void* d_out, int64_t BH,
                                int64_t T_q, int64_t T_kv, int64_t D, const int32_t* q_idx, const int32_t* q_runs,
                                int64_t Tq_pad, int64_t Tkv_pad, const float* lse2, const float* delta,
                                const uint16_t* list, const int32_t* list_count, int64_t list_stride, float scale,
                                int64_t H, int64_t T_out, int out_boundary, float* dq, const int32_t* q_rows,
                                const int32_t* k_rows, int64_t R_q, int64_t R_kv, const void* o, float* delta_out,
                                void* do_out, const void* q_sorted, void* stream) {
  int rc = check_attn_args(BH, T_q, T_kv, D, Tq_pad, Tkv_pad, q, k, v);
  if (rc) return rc;
  if (BH == 0 || T_q == 0) return SCFA_OK;
  AttnLaunch L{};
  L.mode = 1;  // rows = queries
  L.D = static_cast<int>(D);
  L.BH = static_cast<int>(BH);
  L.H = static_cast<int>(H);
  L.T_out = static_cast<int>(T_out);
  L.out_boundary = out_boundary;
  L.scale = scale;
  L.lse2 = lse2;
  L.delta = delta;
  L.list = list;
  L.list_count = list_count;
  L.list_stride = static_cast<int>(list_stride);
  L.out0 = dq;
  L.T_rows = static_cast<int>(T_q);
  L.T_cols = static_cast<int>(T_kv > 0 ? T_kv : 1);
  L.T_rows_pad = static_cast<int>(Tq_pad);
  L.T_cols_pad = static_cast<int>(Tkv_pad);
  L.x0 = q;
  L.x1 = d_out;
  L.y0 = T_kv > 0 ? k : q;
  L.y1 = T_kv > 0 ? v : q;
  if (T_kv == 0) L.T_cols = static_cast<int>(T_q);
  L.row_idx = q_idx;
  L.row_runs = q_runs;
  L.x_rows = q_rows;
  L.y_rows = T_kv > 0 ? k_rows : nullptr;
  L.x_nrows = R_q;
  L.y_nrows = R_kv;
  if (o && !delta_out) {
    set_error("bwd_dq: the fused delta needs delta_out");
    return SCFA_ERR_PARAM;
  }
  if (o && !q_rows && out_boundary) {
    set_error("bwd_dq: the fused delta needs row tables or engine layout");
    return SCFA_ERR_PARAM;
  }
  if (do_out && !q_rows) {
    set_error("bwd_dq: do_out needs row tables (it is the gathered dO in kernel order)");
    return SCFA_ERR_PARAM;
  }
  L.x_out = do_out;
  L.x0_tiled = q_rows ? q_sorted : nullptr;
  L.o_src = o;
  L.delta_out = o ? delta_out : nullptr;
  L.n_row_blocks = (L.T_rows + 127) / 128;
  rc = launch_attention(L, static_cast<cudaStream_t>(stream));
  if (rc && !g_err[0]) set_error("attention backward (dQ) launch failed: %s", cudaGetErrorString(cudaGetLastError()));
  return rc;
}

extern "C" int scfa_attn_bwd_dkdv(const void* q, const void* k, const void* v, const void* d_out, int64_t BH,
                                  int64_t T_q, int64_t T_kv, int64_t D, const int32_t* k_idx, const int32_t* k_runs,
                                  int64_t Tq_pad, int64_t Tkv_pad, const float* lse2, const float* delta,
                                  const uint16_t* list, const int32_t* list_count, int64_t list_stride, float scale,
                                  int64_t H, int64_t T_out, int out_boundary, float* dk, float* dv,
                                  const int32_t* q_rows, const int32_t* k_rows, int64_t R_q, int64_t R_kv,
                                  const int32_t* out_rows, void* stream) {
  int rc = check_attn_args(BH, T_q, T_kv, D, Tq_pad, Tkv_pad, q, k, v);
  if (rc) return rc;
  if (BH == 0 || T_kv == 0) return SCFA_OK;
  if (out_rows && k_rows) {
    set_error("attn_bwd_dkdv: out_rows is for tiled operands (row tables route by k_rows)");
    return SCFA_ERR_PARAM;
  }
  AttnLaunch L{};
  L.mode = 2;  // rows = keys
  L.out_rows = out_rows;
  L.D = static_cast<int>(D);
  L.BH = static_cast<int>(BH);
  L.H = static_cast<int>(H);
  L.T_out = static_cast<int>(T_out);
  L.out_boundary = out_boundary;
  L.scale = scale;
  L.lse2 = lse2;
  L.delta = delta;
  L.list = list;
  L.list_count = list_count;
  L.list_stride = static_cast<int>(list_stride);
  L.out0 = dk;
  L.out1 = dv;
  L.T_rows = static_cast<int>(T_kv);
  L.T_cols = static_cast<int>(T_q > 0 ? T_q : 1);
  L.T_rows_pad = static_cast<int>(Tkv_pad);
  L.T_cols_pad = static_cast<int>(Tq_pad);
  L.x0 = k;
  L.x1 = v;
  L.y0 = T_q > 0 ? q : k;
  L.y1 = T_q > 0 ? d_out : k;
  if (T_q == 0) L.T_cols = static_cast<int>(T_kv);
  L.row_idx = k_idx;
  L.row_runs = k_runs;
  L.x_rows = k_rows;
  L.y_rows = T_q > 0 ? q_rows : nullptr;
  L.x_nrows = R_kv;
  L.y_nrows = R_q;
  L.n_row_blocks = (L.T_rows + 127) / 128;
  rc = launch_attention(L, static_cast<cudaStream_t>(stream));
  if (rc && !g_err[0]) set_error("attention backward (dK/dV) launch failed: %s", cudaGetErrorString(cudaGetLastError()));
  return rc;
}

extern "C" int scfa_attn_bwd(const void* q, const void* k, const void* v, const void* d_out, int64_t BH, int64_t T_q,
                             int64_t T_kv, int64_t D, const int32_t* q_idx, const int32_t* k_idx,
                             const int32_t* k_runs, int64_t Tq_pad, int64_t Tkv_pad, const float* lse2,
                             const float* delta, const uint16_t* list, const int32_t* list_count,
                             int64_t list_stride, float scale, int64_t H, int64_t Tq_out, int64_t Tkv_out,
                             int out_boundary, float* dq, float* dk, float* dv, void* stream) {
  int rc = check_attn_args(BH, T_q, T_kv, D, Tq_pad, Tkv_pad, q, k, v);
  if (rc) return rc;
  if (D != 64) {
    set_error("attn_bwd (single pass): head dim %lld unsupported (64; use the two-pass dQ + dK/dV)",
              static_cast<long long>(D));
    return SCFA_ERR_SHAPE;
  }
  if (!dq || !q_idx) {
    set_error("attn_bwd: dq and q_idx are required");
    return SCFA_ERR_PARAM;
  }
  if (BH == 0 || T_kv == 0 || T_q == 0) return SCFA_OK;  // dQ stays as given (zero), dK / dV: no rows
  AttnLaunch L{};
  L.mode = 3;  // rows = keys; dQ reduced per tile pair
  L.D = static_cast<int>(D);
  L.BH = static_cast<int>(BH);
  L.H = static_cast<int>(H);
  L.T_out = static_cast<int>(Tkv_out);
  L.T_out_cols = static_cast<int>(Tq_out);
  L.out_boundary = out_boundary;
  L.scale = scale;
  L.lse2 = lse2;
  L.delta = delta;
  L.list = list;
  L.list_count = list_count;
  L.list_stride = static_cast<int>(list_stride);
  L.out0 = dk;
  L.out1 = dv;
  L.out2 = dq;
  L.col_idx = q_idx;
  L.T_rows = static_cast<int>(T_kv);
  L.T_cols = static_cast<int>(T_q);
  L.T_rows_pad = static_cast<int>(Tkv_pad);
  L.T_cols_pad = static_cast<int>(Tq_pad);
  L.x0 = k;
  L.x1 = v;
  L.y0 = q;
  L.y1 = d_out;
  L.row_idx = k_idx;
  L.row_runs = k_runs;
  L.n_row_blocks = (L.T_rows + 127) / 128;
  rc = launch_attention(L, static_cast<cudaStream_t>(stream));
  if (rc && !g_err[0]) set_error("attention backward (single pass) launch failed: %s", cudaGetErrorString(cudaGetLastError()));
  return rc;
}
