// extern "C" boundary of libdoublep_b200.so (declared in include/doublep_b200.h).
#include <cuda_runtime.h>

#include <cstdio>
#include <string>

#include "common.cuh"
#include "decode_internal.h"

namespace {
thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}
int cuda_fail(cudaError_t e, const char* where) {
  cudaGetLastError();  // a failed launch must not leave its (non-sticky) error for the caller's next CUDA call
  return fail(DP_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

int check_view(const dp_cache_view* v, int G) {
  if (!v) return fail(DP_ERR_INVALID, "null cache view");
  if (v->batch < 1 || v->kv_heads < 1 || v->head_dim < 1)
    return fail(DP_ERR_INVALID, "cache dimensions must be positive");
  if (v->dtype != DP_F32 && v->dtype != DP_BF16) return fail(DP_ERR_INVALID, "unknown cache dtype");
  if (v->head_dim % 8 != 0 || v->head_dim > 256)
    return fail(DP_ERR_UNSUPPORTED, "head_dim must be a multiple of 8 and <= 256");
  if (G < 1 || G > dp::kMaxGroup) return fail(DP_ERR_UNSUPPORTED, "gqa_group must be in [1, 8]");
  if (v->sink < 0 || v->window < 0) return fail(DP_ERR_INVALID, "sink and window must be >= 0");
  if (v->n_tokens > v->row_cap || v->n_tokens < 1) return fail(DP_ERR_INVALID, "n_tokens outside [1, row_cap]");
  if (v->sink + v->window > v->n_tokens)
    return fail(DP_ERR_INVALID, "config/cache mismatch: sink + window exceed the context");
  if (v->cluster_cap < 1) return fail(DP_ERR_INVALID, "no clusters for this head");
  return DP_OK;
}
int check_p(double p, const char* name) {
  if (!(p > 0.0 && p <= 1.0)) return fail(DP_ERR_INVALID, std::string(name) + " must be in (0, 1]");
  return DP_OK;
}
int check_q(int qdt) {
  if (qdt != DP_F32 && qdt != DP_BF16) return fail(DP_ERR_INVALID, "unknown query dtype");
  return DP_OK;
}
}  // namespace

extern "C" {

int dp_version(void) { return 100; }

const char* dp_last_error(void) { return g_err.c_str(); }

int dp_device_info(int32_t* sm_count, int32_t* cc_major, int32_t* cc_minor) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  cudaDeviceProp p;
  e = cudaGetDeviceProperties(&p, dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDeviceProperties");
  if (sm_count) *sm_count = p.multiProcessorCount;
  if (cc_major) *cc_major = p.major;
  if (cc_minor) *cc_minor = p.minor;
  return DP_OK;
}

size_t dp_decode_workspace_bytes(const dp_cache_view* v, int32_t gqa_group) {
  if (!v) return 0;
  return dp::decode_ws_layout(v, gqa_group, nullptr, nullptr, nullptr, nullptr);
}

int dp_score(const dp_cache_view* v, const void* q, int32_t q_dtype, int32_t G, double scale,
             double* log_mass, void* stream) {
  int r = check_view(v, G);
  if (r) return r;
  if ((r = check_q(q_dtype))) return r;
  cudaError_t e = dp::launch_score(*v, q, q_dtype, G, scale, log_mass, (cudaStream_t)stream);
  return e == cudaSuccess ? DP_OK : cuda_fail(e, "dp_score");
}

int dp_select(const dp_cache_view* v, int32_t G, double p1, double p2, const double* log_mass,
              uint8_t* state, int32_t* counts, int32_t* order, double* cum_mass, double* probs, void* ws,
              size_t ws_bytes, void* stream) {
  int r = check_view(v, G);
  if (r) return r;
  if ((r = check_p(p1, "p1")) || (r = check_p(p2, "p2"))) return r;
  if (v->cluster_cap > 16384)
    return fail(DP_ERR_UNSUPPORTED, "cluster_cap > 16384 needs the sequence-sharded select path");
  (void)ws;
  (void)ws_bytes;
  cudaError_t e = dp::launch_select(*v, G, p1, p2, log_mass, state, counts, order, cum_mass, probs,
                                    (cudaStream_t)stream);
  return e == cudaSuccess ? DP_OK : cuda_fail(e, "dp_select");
}

int dp_build_worklist(const dp_cache_view* v, int32_t G, const double* log_mass, const uint8_t* state,
                      int32_t* stats, void* ws, size_t ws_bytes, void* stream) {
  int r = check_view(v, G);
  if (r) return r;
  if (ws_bytes < dp_decode_workspace_bytes(v, G)) return fail(DP_ERR_INVALID, "workspace too small");
  cudaError_t e = dp::launch_worklist(*v, G, state, stats, ws, (cudaStream_t)stream, log_mass);
  return e == cudaSuccess ? DP_OK : cuda_fail(e, "dp_build_worklist");
}

int dp_attend(const dp_cache_view* v, const void* q, int32_t q_dtype, int32_t G, double scale,
              const double* log_mass, float* out, float* lse, void* ws, size_t ws_bytes, void* stream) {
  int r = check_view(v, G);
  if (r) return r;
  if ((r = check_q(q_dtype))) return r;
  if (ws_bytes < dp_decode_workspace_bytes(v, G)) return fail(DP_ERR_INVALID, "workspace too small");
  cudaError_t e = dp::launch_attend(*v, q, q_dtype, G, scale, log_mass, out, lse, ws, false, (cudaStream_t)stream);
  return e == cudaSuccess ? DP_OK : cuda_fail(e, "dp_attend");
}

int dp_sparse_attention(const dp_cache_view* v, const void* q, int32_t q_dtype, int32_t G, double scale,
                        const double* log_mass, const uint8_t* state, float* out, float* lse, int32_t* stats,
                        void* ws, size_t ws_bytes, void* stream) {
  int r = check_view(v, G);
  if (r) return r;
  if ((r = check_q(q_dtype))) return r;
  if (ws_bytes < dp_decode_workspace_bytes(v, G)) return fail(DP_ERR_INVALID, "workspace too small");
  // with the query: the sink/window logits join the attention's reference max
  cudaError_t e = dp::launch_worklist(*v, G, state, stats, ws, (cudaStream_t)stream, log_mass, q, q_dtype, scale);
  if (e != cudaSuccess) return cuda_fail(e, "dp_sparse_attention");
  return dp_attend(v, q, q_dtype, G, scale, log_mass, out, lse, ws, ws_bytes, stream);
}

int dp_plan(const dp_cache_view* v, const void* q, int32_t q_dtype, int32_t G, double scale, double p1, double p2,
            double* log_mass, uint8_t* state, int32_t* counts, int32_t* stats, void* ws, size_t ws_bytes,
            void* stream) {
  int r = check_view(v, G);
  if (r) return r;
  if ((r = check_q(q_dtype)) || (r = check_p(p1, "p1")) || (r = check_p(p2, "p2"))) return r;
  if (ws_bytes < dp_decode_workspace_bytes(v, G)) return fail(DP_ERR_INVALID, "workspace too small");
  if (!dp::plan_supported(*v, G))
    return fail(DP_ERR_UNSUPPORTED, "fused plan needs cluster_cap <= 4096 and row_cap < 2^24");
  cudaError_t e = dp::launch_plan(*v, q, q_dtype, G, scale, p1, p2, log_mass, state, counts, stats, ws,
                                  (cudaStream_t)stream);
  return e == cudaSuccess ? DP_OK : cuda_fail(e, "dp_plan");
}

int dp_plan_score(const dp_cache_view* v, const void* q, int32_t q_dtype, int32_t G, double scale, double* log_mass,
                  void* ws, size_t ws_bytes, void* stream) {
  int r = check_view(v, G);
  if (r) return r;
  if ((r = check_q(q_dtype))) return r;
  if (!log_mass) return fail(DP_ERR_INVALID, "log_mass buffer required");
  if (ws_bytes < dp_decode_workspace_bytes(v, G)) return fail(DP_ERR_INVALID, "workspace too small");
  if (!dp::plan_supported(*v, G))
    return fail(DP_ERR_UNSUPPORTED, "fused plan needs cluster_cap <= 4096 and row_cap < 2^24");
  cudaError_t e = dp::launch_plan(*v, q, q_dtype, G, scale, 1.0, 1.0, log_mass, nullptr, nullptr, nullptr, ws,
                                  (cudaStream_t)stream, 1);
  return e == cudaSuccess ? DP_OK : cuda_fail(e, "dp_plan_score");
}

int dp_plan_given(const dp_cache_view* v, const void* q, int32_t q_dtype, int32_t G, double scale, double* log_mass,
                  const uint8_t* state, int32_t state_ld, int32_t* stats, void* ws, size_t ws_bytes, void* stream) {
  int r = check_view(v, G);
  if (r) return r;
  if ((r = check_q(q_dtype))) return r;
  if (!log_mass || !state) return fail(DP_ERR_INVALID, "log_mass and state buffers required");
  if (ws_bytes < dp_decode_workspace_bytes(v, G)) return fail(DP_ERR_INVALID, "workspace too small");
  if (!dp::plan_supported(*v, G))
    return fail(DP_ERR_UNSUPPORTED, "fused plan needs cluster_cap <= 4096 and row_cap < 2^24");
  if (state_ld != 0 && state_ld < v->cluster_cap) return fail(DP_ERR_INVALID, "state_ld below cluster_cap");
  cudaError_t e = dp::launch_plan(*v, q, q_dtype, G, scale, 1.0, 1.0, log_mass, const_cast<uint8_t*>(state), nullptr,
                                  stats, ws, (cudaStream_t)stream, 2, state_ld);
  return e == cudaSuccess ? DP_OK : cuda_fail(e, "dp_plan_given");
}

int dp_decode_step(const dp_cache_view* v, const void* q, int32_t q_dtype, int32_t G, double scale, double p1,
                   double p2, double* log_mass, uint8_t* state, int32_t* counts, float* out, float* lse,
                   int32_t* stats, void* ws, size_t ws_bytes, void* stream) {
  int r = check_view(v, G);
  if (r) return r;
  if (dp::step_supported(*v, G, q_dtype)) {  // the whole step in one launch (every head's cluster co-resident)
    if ((r = check_q(q_dtype)) || (r = check_p(p1, "p1")) || (r = check_p(p2, "p2"))) return r;
    if (!log_mass) return fail(DP_ERR_INVALID, "log_mass buffer required");
    cudaError_t e = dp::launch_step(*v, q, q_dtype, G, scale, p1, p2, log_mass, state, counts, stats, out, lse, ws,
                                    (cudaStream_t)stream);
    return e == cudaSuccess ? DP_OK : cuda_fail(e, "dp_decode_step");
  }
  if (dp::plan_supported(*v, G)) {  // fused score + select + worklist (one launch) -> attend
    r = dp_plan(v, q, q_dtype, G, scale, p1, p2, log_mass, state, counts, stats, ws, ws_bytes, stream);
    if (r) return r;
    return dp_attend(v, q, q_dtype, G, scale, log_mass, out, lse, ws, ws_bytes, stream);
  }
  r = dp_score(v, q, q_dtype, G, scale, log_mass, stream);
  if (r) return r;
  r = dp_select(v, G, p1, p2, log_mass, state, counts, nullptr, nullptr, nullptr, ws, ws_bytes, stream);
  if (r) return r;
  return dp_sparse_attention(v, q, q_dtype, G, scale, log_mass, state, out, lse, stats, ws, ws_bytes, stream);
}

int dp_cluster_topk(const dp_cache_view* v, const void* q, int32_t q_dtype, int32_t G, double scale,
                    int32_t budget, double* log_mass, uint8_t* state, int32_t* order, int32_t* counts, float* out,
                    float* lse, int32_t* stats, void* ws, size_t ws_bytes, void* stream) {
  int r = check_view(v, G);
  if (r) return r;
  if (budget < 1) return fail(DP_ERR_INVALID, "cluster budget must be >= 1");
  if (!log_mass || !state || !order) return fail(DP_ERR_INVALID, "log_mass, state and order are required");
  if ((r = dp_score(v, q, q_dtype, G, scale, log_mass, stream))) return r;
  if ((r = dp_select(v, G, 1.0, 1.0, log_mass, state, counts, order, nullptr, nullptr, ws, ws_bytes, stream)))
    return r;
  cudaError_t e = dp::launch_topk_state(*v, G, budget, order, state, counts, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "dp_cluster_topk");
  return dp_sparse_attention(v, q, q_dtype, G, scale, log_mass, state, out, lse, stats, ws, ws_bytes, stream);
}

int dp_dense_attention(const dp_cache_view* v, const void* q, int32_t q_dtype, int32_t G, double scale,
                       float* out, float* lse, void* ws, size_t ws_bytes, void* stream) {
  int r = check_view(v, G);
  if (r) return r;
  if ((r = check_q(q_dtype))) return r;
  if (ws_bytes < dp_decode_workspace_bytes(v, G)) return fail(DP_ERR_INVALID, "workspace too small");
  cudaError_t e = dp::launch_attend(*v, q, q_dtype, G, scale, nullptr, out, lse, ws, true, (cudaStream_t)stream);
  return e == cudaSuccess ? DP_OK : cuda_fail(e, "dp_dense_attention");
}

int dp_append_token(const dp_cache_view* v, const void* new_k, const void* new_v, void* stream) {
  int r = check_view(v, 1);
  if (r) return r;
  if (v->n_tokens >= v->row_cap) return fail(DP_ERR_INVALID, "row capacity exhausted");
  cudaError_t e = dp::launch_append(*v, new_k, new_v, (cudaStream_t)stream);
  return e == cudaSuccess ? DP_OK : cuda_fail(e, "dp_append_token");
}

/* ---- measurement side (metrics.cu) ---------------------------------- */

int dp_token_weights(const dp_cache_view* v, const void* q, int32_t q_dtype, int32_t G, double scale,
                     double* weights, double* lse, void* stream) {
  int r = check_view(v, G);
  if (r) return r;
  if ((r = check_q(q_dtype))) return r;
  if (!weights || !lse) return fail(DP_ERR_INVALID, "weights and lse are required");
  cudaError_t e = dp::launch_token_weights(*v, q, q_dtype, G, scale, weights, lse, (cudaStream_t)stream);
  return e == cudaSuccess ? DP_OK : cuda_fail(e, "dp_token_weights");
}

int dp_token_topk(const dp_cache_view* v, const int32_t* perm, int32_t perm_rows, int32_t G, int32_t budget,
                  const int32_t* budgets, const double* weights, double* out, double* captured, uint8_t* selected, void* stream) {
  int r = check_view(v, G);
  if (r) return r;
  if (budget < 1 || budget > v->n_tokens)
    return fail(DP_ERR_INVALID, "budget must be in [1, " + std::to_string(v->n_tokens) + "], got " +
                                    std::to_string(budget));
  if (!weights || !out || !captured) return fail(DP_ERR_INVALID, "weights, out and captured are required");
  cudaError_t e = dp::launch_token_topk(*v, perm, perm_rows, G, budget, budgets, weights, out, captured, selected,
                                        (cudaStream_t)stream);
  return e == cudaSuccess ? DP_OK : cuda_fail(e, "dp_token_topk");
}

int dp_recovered_mass(const dp_cache_view* v, int32_t G, const double* weights, const uint8_t* state,
                      double* recovered, void* stream) {
  int r = check_view(v, G);
  if (r) return r;
  if (!weights || !state || !recovered) return fail(DP_ERR_INVALID, "weights, state and recovered are required");
  cudaError_t e = dp::launch_recovered_mass(*v, G, weights, state, recovered, (cudaStream_t)stream);
  return e == cudaSuccess ? DP_OK : cuda_fail(e, "dp_recovered_mass");
}

int dp_cluster_approx_error(const dp_cache_view* v, int32_t G, const double* weights, const double* lse,
                            const double* log_mass, const int32_t* order, double* errors, void* stream) {
  int r = check_view(v, G);
  if (r) return r;
  if (!weights || !lse || !log_mass || !order || !errors)
    return fail(DP_ERR_INVALID, "weights, lse, log_mass, order and errors are required");
  cudaError_t e = dp::launch_cluster_error(*v, G, weights, lse, log_mass, order, errors, (cudaStream_t)stream);
  return e == cudaSuccess ? DP_OK : cuda_fail(e, "dp_cluster_approx_error");
}

int dp_adaptive_token_budget(const dp_cache_view* v, int32_t G, const double* weights, double p, int32_t* budget,
                             void* stream) {
  int r = check_view(v, G);
  if (r) return r;
  if (!weights || !budget) return fail(DP_ERR_INVALID, "weights and budget are required");
  cudaError_t e = dp::launch_adaptive_budget(*v, G, weights, p, budget, (cudaStream_t)stream);
  return e == cudaSuccess ? DP_OK : cuda_fail(e, "dp_adaptive_token_budget");
}

int dp_mixed_attention_f64(const dp_cache_view* v, const void* q, int32_t q_dtype, int32_t G, double scale,
                           const double* log_mass, const uint8_t* state, double* out, double* lse, void* stream) {
  int r = check_view(v, G);
  if (r) return r;
  if ((r = check_q(q_dtype))) return r;
  if (!out) return fail(DP_ERR_INVALID, "out is required");
  if (state && !log_mass) return fail(DP_ERR_INVALID, "log_mass is required with a state");
  cudaError_t e = dp::launch_mixed_f64(*v, q, q_dtype, G, scale, log_mass, state, out, lse, (cudaStream_t)stream);
  return e == cudaSuccess ? DP_OK : cuda_fail(e, "dp_mixed_attention_f64");
}

/* ---- sequence-sharded Double-P with global semantics (shard.cu) ---- */

int dp_kmpp_shard_dsq(const void* points, int32_t dtype, int32_t units, int32_t n, int32_t d, const double* centre,
                      int32_t first, double* dsq, double* sums, void* stream) {
  if (!points || !centre || !dsq || !sums) return fail(DP_ERR_INVALID, "dp_kmpp_shard_dsq: null buffer");
  if (dtype != DP_F32 && dtype != DP_BF16) return fail(DP_ERR_INVALID, "unknown points dtype");
  if (units < 1 || n < 1 || d < 1) return fail(DP_ERR_INVALID, "dp_kmpp_shard_dsq: empty shard");
  cudaError_t e = dp::launch_kmpp_dsq(points, dtype, units, n, d, centre, first, dsq, sums, (cudaStream_t)stream);
  return e == cudaSuccess ? DP_OK : cuda_fail(e, "dp_kmpp_shard_dsq");
}

int dp_kmpp_shard_pick(const void* points, int32_t dtype, int32_t units, int32_t n, int32_t d, const double* dsq,
                       const double* all_sums, int32_t world, int32_t rank, const double* uniforms,
                       const int32_t* pick_in, int64_t global_base, double* centre_out, int32_t* pick_out,
                       void* stream) {
  if (!points || !centre_out || !pick_out) return fail(DP_ERR_INVALID, "dp_kmpp_shard_pick: null buffer");
  if (!pick_in && (!dsq || !all_sums || !uniforms)) return fail(DP_ERR_INVALID, "dp_kmpp_shard_pick: null buffer");
  if (world < 1 || rank < 0 || rank >= world) return fail(DP_ERR_INVALID, "rank outside [0, world)");
  cudaError_t e = dp::launch_kmpp_pick(points, dtype, units, n, d, dsq, all_sums, world, rank, uniforms, pick_in,
                                       (long long)global_base, centre_out, pick_out, (cudaStream_t)stream);
  return e == cudaSuccess ? DP_OK : cuda_fail(e, "dp_kmpp_shard_pick");
}

size_t dp_lloyd_shard_workspace_bytes(int32_t units, int32_t n, int32_t k) { return dp::lloyd_sums_ws_bytes(units, n, k); }

int dp_lloyd_shard_sums(const void* points, int32_t dtype, int32_t units, int32_t n, int32_t d,
                        const int32_t* assign, int32_t k, double* sums, int64_t* counts, void* workspace,
                        size_t workspace_bytes, void* stream) {
  if (!points || !assign || !sums || !counts) return fail(DP_ERR_INVALID, "dp_lloyd_shard_sums: null buffer");
  if (workspace_bytes < dp::lloyd_sums_ws_bytes(units, n, k)) return fail(DP_ERR_INVALID, "workspace too small");
  cudaError_t e = dp::launch_lloyd_sums(points, dtype, units, n, d, assign, k, sums,
                                        reinterpret_cast<long long*>(counts), workspace, (cudaStream_t)stream);
  return e == cudaSuccess ? DP_OK : cuda_fail(e, "dp_lloyd_shard_sums");
}

size_t dp_select_global_workspace_bytes(int32_t rows, int32_t ld) { return dp::select_global_ws_bytes(rows, ld); }

int dp_select_global(const double* log_mass, int32_t rows, int32_t ld, const int32_t* nclusters, double p1,
                     double p2, uint8_t* state, int32_t* counts, void* workspace, size_t workspace_bytes,
                     void* stream) {
  int r;
  if ((r = check_p(p1, "p1")) || (r = check_p(p2, "p2"))) return r;
  if (!log_mass || !nclusters || !state || !counts) return fail(DP_ERR_INVALID, "dp_select_global: null buffer");
  if (rows < 1 || ld < 1) return fail(DP_ERR_INVALID, "dp_select_global: empty input");
  if (workspace_bytes < dp::select_global_ws_bytes(rows, ld)) return fail(DP_ERR_INVALID, "workspace too small");
  cudaError_t e = dp::launch_select_global(log_mass, rows, ld, nclusters, p1, p2, state, counts, workspace,
                                           (cudaStream_t)stream);
  return e == cudaSuccess ? DP_OK : cuda_fail(e, "dp_select_global");
}

int dp_select_global_parts(const double* log_mass_parts, int32_t rows, int32_t parts, int32_t part_len,
                           const int32_t* nclusters, double p1, double p2, uint8_t* state, int32_t* counts,
                           void* workspace, size_t workspace_bytes, void* stream) {
  int r;
  if ((r = check_p(p1, "p1")) || (r = check_p(p2, "p2"))) return r;
  if (!log_mass_parts || !nclusters || !state || !counts) return fail(DP_ERR_INVALID, "dp_select_global: null buffer");
  if (rows < 1 || parts < 1 || part_len < 1) return fail(DP_ERR_INVALID, "dp_select_global: empty input");
  if (!dp::select_global_parts_supported(parts, part_len))
    return fail(DP_ERR_UNSUPPORTED, "dp_select_global_parts: parts * part_len must be <= 65536");
  const int ld = parts * part_len;
  if (workspace_bytes < dp::select_global_ws_bytes(rows, ld)) return fail(DP_ERR_INVALID, "workspace too small");
  cudaError_t e = dp::launch_select_global(log_mass_parts, rows, ld, nclusters, p1, p2, state, counts, workspace,
                                           (cudaStream_t)stream, part_len);
  return e == cudaSuccess ? DP_OK : cuda_fail(e, "dp_select_global_parts");
}

int dp_lse_merge(const float* out_parts, const float* lse_parts, int32_t parts, int32_t rows, int32_t d, float* out,
                 float* lse, void* stream) {
  if (!out_parts || !lse_parts || !out || !lse) return fail(DP_ERR_INVALID, "dp_lse_merge: null buffer");
  if (parts < 1 || rows < 1 || d < 1) return fail(DP_ERR_INVALID, "dp_lse_merge: empty input");
  if (parts > 64) return fail(DP_ERR_UNSUPPORTED, "dp_lse_merge: at most 64 partials");
  cudaError_t e = dp::launch_lse_merge(out_parts, lse_parts, parts, rows, d, out, lse, (cudaStream_t)stream);
  return e == cudaSuccess ? DP_OK : cuda_fail(e, "dp_lse_merge");
}

}  // extern "C"

// error helper used by the clustering TU
namespace dp {
int set_error(int code, const char* msg) { return fail(code, msg); }
int set_cuda_error(cudaError_t e, const char* where) { return cuda_fail(e, where); }
}  // namespace dp
