/*
 * doublep_b200.h -- C ABI of the B200-native Double-P decode path.
 *
 * Double-P (arxiv 2602.05191): hierarchical top-p sparse decode attention
 * over a k-means-clustered KV cache.  This header is the drop-in boundary
 * that replaces the reference's kernel plugin seam
 * (/root/reference/pkg/src/doublep/kernels.py:47-96) one level higher: the
 * reference seam is per-query and host-memory based; these entry points are
 * batched over (sequence, kv head, q head) and take DEVICE pointers, so a
 * whole per-layer decode step is a few stream-ordered launches with no host
 * synchronisation (CUDA-graph capturable).
 *
 * Conventions
 *   - all buffers are caller-owned device memory; nothing allocates on the
 *     step path (workspace sized once with dp_*_workspace_bytes, ZERO-filled
 *     once before first use; the kernels leave it reusable);
 *   - every call is stream-ordered on the caller's cudaStream_t (passed as
 *     void* so this header needs no CUDA include);
 *   - return value: DP_OK or an error code; dp_last_error() gives a
 *     thread-local message.  DP_ERR_INVALID maps to the reference's
 *     ValueError messages (engine.py:118,162,259-261,270-274;
 *     clustering.py:73,281);
 *   - re-entrant across streams given distinct workspaces.
 *
 * Device cache layout (one layer, batch B, kv heads H, per (b,h) "head"):
 *   rows [0, sink)                         sink tokens, position order
 *   rows [sink, n_tokens - window)         clustered tokens, CLUSTER-CONTIGUOUS:
 *                                          cluster c owns rows [offs[c], offs[c+1])
 *                                          (prefill clusters in compacted k-means id
 *                                          order, then residual singletons appended
 *                                          by decode-time growth, clustering.py:219-229)
 *   rows [n_tokens - window, n_tokens)     sliding window, position order
 * keys/values [B,H,row_cap,d]; centroids/value_means fp32 [B,H,cluster_cap,d];
 * offs int32 [B,H,cluster_cap+1]; nclusters int32 [B,H].
 */
#ifndef DOUBLEP_B200_H
#define DOUBLEP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DP_OK 0
#define DP_ERR_INVALID 1     /* bad argument / reference ValueError class */
#define DP_ERR_CUDA 2        /* CUDA runtime error */
#define DP_ERR_UNSUPPORTED 3 /* shape outside what the kernels were built for */

#define DP_F32 0
#define DP_BF16 1

typedef struct dp_cache_view {
  int32_t batch, kv_heads, head_dim, dtype; /* dtype: DP_F32 | DP_BF16 */
  int32_t row_cap;     /* rows allocated per head */
  int32_t n_tokens;    /* rows in use per head (prefill + appended) */
  int32_t sink, window;
  int32_t cluster_cap; /* table capacity per head */
  int32_t _pad;
  const void* keys;           /* [B,H,row_cap,d] */
  const void* values;         /* [B,H,row_cap,d] */
  const int32_t* offs;        /* [B,H,cluster_cap+1] absolute row offsets */
  const int32_t* nclusters;   /* [B,H] */
  const float* centroids;     /* [B,H,cluster_cap,d] fp32 (exact means rounded) */
  const float* value_means;   /* [B,H,cluster_cap,d] fp32 */
} dp_cache_view;

/* ---------------------------------------------------------------------- */
/* library                                                                  */
/* ---------------------------------------------------------------------- */
int dp_version(void);
const char* dp_last_error(void);
/* number of SMs / compute capability of the current device (for callers) */
int dp_device_info(int32_t* sm_count, int32_t* cc_major, int32_t* cc_minor);

/* ---------------------------------------------------------------------- */
/* decode step                                                              */
/* ---------------------------------------------------------------------- */

/* Workspace for dp_select / dp_sparse_attention / dp_decode_step /
 * dp_dense_attention at this geometry and GQA group size. */
size_t dp_decode_workspace_bytes(const dp_cache_view* v, int32_t gqa_group);

/* Size-weighted centroid scores, replaces estimate_cluster_distribution
 * (engine.py:158-177; kernels.scaled_logits _kernels_cy.pyx:21-33):
 *   log_mass[b, h*G+g, c] = (C[b,h,c] . q[b,h*G+g]) * scale + log(|c|)
 * fp64 accumulation over fp32 centroids.  q [B, H*G, d] (q_dtype),
 * log_mass fp64 [B, H*G, cluster_cap] (entries >= nclusters untouched). */
int dp_score(const dp_cache_view* v, const void* q, int32_t q_dtype, int32_t gqa_group,
             double scale, double* log_mass, void* stream);

/* Two-stage top-p, replaces plan_selection + top_p_select
 * (engine.py:180-213, selection.py:36-65).  Per q head: stage 1 keeps the
 * minimal descending-probability prefix with cumsum/total >= p1 (ties ->
 * lower cluster id); stage 2 keeps the minimal prefix of that set reaching
 * p2 of its renormalised mass.  state[b,hq,c] = 2 exact, 1 approx, 0 drop.
 * counts[b,hq,0..1] = (|C_p|, |C_exact|).  Nullable debug outputs: order
 * [B,Hq,cluster_cap] the full descending order (estimate.order,
 * engine.py:169; its first counts[0] entries are stage1.selected), cum_mass
 * [B,Hq] the stage-1 normalised cumulative mass, probs [B,Hq,cluster_cap]
 * the estimated cluster distribution (engine.py:168). */
int dp_select(const dp_cache_view* v, int32_t gqa_group, double p1, double p2,
              const double* log_mass, uint8_t* state, int32_t* counts, int32_t* order,
              double* cum_mass, double* probs, void* workspace, size_t workspace_bytes,
              void* stream);

/* Mixed exact/approximate attention under one normaliser, replaces
 * mixed_attention / sparse_attention (engine.py:216-264):
 *   exact rows = sink + window + members of state==2 clusters,
 *   approx pseudo-rows = (log_mass, value_mean) of state==1 clusters.
 * out fp32 [B,Hq,d], lse fp32 [B,Hq] (log of the shared normaliser).
 * stats (nullable) int32 [B,H,4] = (union exact rows, union approx clusters,
 * row chunks, 0) -- the quantities the algorithmic byte count uses. */
int dp_sparse_attention(const dp_cache_view* v, const void* q, int32_t q_dtype,
                        int32_t gqa_group, double scale, const double* log_mass,
                        const uint8_t* state, float* out, float* lse, int32_t* stats,
                        void* workspace, size_t workspace_bytes, void* stream);

/* The two halves of dp_sparse_attention, for callers that time or overlap
 * them separately: dp_build_worklist turns the per-head states into the
 * GQA-union rows / approx lists and each q head's approx partial (in the
 * workspace); dp_attend runs the
 * gathered split-KV attention + LSE merge over them. */
int dp_build_worklist(const dp_cache_view* v, int32_t gqa_group, const double* log_mass,
                      const uint8_t* state, int32_t* stats, void* workspace,
                      size_t workspace_bytes, void* stream);
int dp_attend(const dp_cache_view* v, const void* q, int32_t q_dtype, int32_t gqa_group,
              double scale, const double* log_mass, float* out, float* lse, void* workspace,
              size_t workspace_bytes, void* stream);

/* score + select + worklist fused into ONE launch (one 8-CTA thread-block
 * cluster per (sequence, kv head), stages exchange data over distributed
 * shared memory): writes log_mass, counts, state (nullable) and the
 * workspace work lists that dp_attend consumes.  Needs cluster_cap <= 4096
 * (contexts up to ~128K at 32 tokens per cluster) and gqa_group <= 8;
 * stats as in dp_sparse_attention (slot 3 = union exact clusters). */
int dp_plan(const dp_cache_view* v, const void* q, int32_t q_dtype, int32_t gqa_group,
            double scale, double p1, double p2, double* log_mass, uint8_t* state,
            int32_t* counts, int32_t* stats, void* workspace, size_t workspace_bytes,
            void* stream);

/* The fused plan split around an OUTSIDE selection (config 5: the two-stage
 * top-p runs over the global, all-gathered log-mass table, dp_select_global):
 *   dp_plan_score: phase 1 only -- log_mass [B, H, G, cluster_cap] of this
 *     cache's clusters (-inf past each head's cluster count), then exit;
 *   dp_plan_given: the plan with the states READ from `state` ([B, H, G]
 *     rows of stride state_ld, 0 = cluster_cap; 0 dropped / 1 approximated /
 *     2 exact) instead of
 *     selected; builds the work lists dp_attend consumes (log_mass as
 *     written by dp_plan_score for the same q).
 * Same shape limits as dp_plan. */
int dp_plan_score(const dp_cache_view* v, const void* q, int32_t q_dtype, int32_t gqa_group, double scale,
                  double* log_mass, void* workspace, size_t workspace_bytes, void* stream);
int dp_plan_given(const dp_cache_view* v, const void* q, int32_t q_dtype, int32_t gqa_group, double scale,
                  double* log_mass, const uint8_t* state, int32_t state_ld, int32_t* stats, void* workspace,
                  size_t workspace_bytes, void* stream);

/* score + select + sparse attention in one call (decode_step,
 * engine.py:267-278).  Implementations, chosen by geometry:
 *   - dp_plan + dp_attend (fused plan, then a persistent attention grid
 *     balanced over every head's rows) when the plan supports the shape;
 *   - the separate dp_score / dp_select / dp_sparse_attention kernels;
 *   - opt-in (dp_debug_set(6, 0)): ONE launch when one thread-block cluster
 *     per (sequence, kv head) fits on the GPU in a single wave (bf16 cache,
 *     head_dim 128, G <= 8, cluster_cap <= 4096): score, select, attention
 *     over the cluster-contiguous runs (TMA) and the LSE merge, with
 *     distributed shared memory between the cluster's CTAs.
 * log_mass (required) / state / counts / stats are caller buffers so the
 * plan stays inspectable. */
int dp_decode_step(const dp_cache_view* v, const void* q, int32_t q_dtype, int32_t gqa_group,
                   double scale, double p1, double p2, double* log_mass, uint8_t* state,
                   int32_t* counts, float* out, float* lse, int32_t* stats, void* workspace,
                   size_t workspace_bytes, void* stream);

/* Fixed cluster-budget baseline, replaces baseline_cluster_topk
 * (engine.py:318-338, the RetroInfer-style comparator of PAPER.md:505): the
 * `budget` clusters with the largest estimated mass are attended exactly
 * (plus sink and window), every other cluster through its centroid
 * approximation, under one normaliser.  budget >= 1; a head with fewer
 * clusters keeps all of them exact.  order [B,Hq,cluster_cap] receives the
 * full descending cluster order; counts [B,Hq,2] = (clusters, exact). */
int dp_cluster_topk(const dp_cache_view* v, const void* q, int32_t q_dtype, int32_t gqa_group, double scale,
                    int32_t budget, double* log_mass, uint8_t* state, int32_t* order, int32_t* counts,
                    float* out, float* lse, int32_t* stats, void* workspace, size_t workspace_bytes,
                    void* stream);

/* Dense split-KV flash decoding over all n_tokens rows (the full_attention
 * comparator, engine.py:122-144). */
int dp_dense_attention(const dp_cache_view* v, const void* q, int32_t q_dtype,
                       int32_t gqa_group, double scale, float* out, float* lse,
                       void* workspace, size_t workspace_bytes, void* stream);

/* Decode-time growth (ClusteredCache.append_tokens, clustering.py:182-196):
 * writes one new token per (b,h) at row n_tokens (keys/values must have
 * row_cap > n_tokens) and turns the row leaving the window into a residual
 * singleton cluster (clustering.py:178-229).  The caller then uses
 * n_tokens + 1.  new_k/new_v [B,H,d] in the cache dtype. */
int dp_append_token(const dp_cache_view* v, const void* new_k, const void* new_v, void* stream);

/* ---------------------------------------------------------------------- */
/* measurement side: true distribution, token top-k baseline, metrics       */
/* (fp64 like the reference; not on the decode path)    */
/* ---------------------------------------------------------------------- */

/* True token distribution, replaces full_attention_weights / true_token_weights
 * (engine.py:122-132, :147-155): logits = (k . q) * scale in fp64 over all
 * n_tokens rows, lse = m + log(sum(exp(x - m))) (kernels.logsumexp,
 * _kernels_py.py:29-35), weights = exp(logits - lse).  weights fp64
 * [B,Hq,row_cap] in PHYSICAL row order (the clustered layout); lse fp64 [B,Hq]. */
int dp_token_weights(const dp_cache_view* v, const void* q, int32_t q_dtype, int32_t gqa_group, double scale,
                     double* weights, double* lse, void* stream);

/* Idealised fixed-budget baseline, replaces baseline_token_topk
 * (engine.py:293-315) with top_k_select (selection.py:85-92): the `budget`
 * rows of largest true weight (ties -> lower token position; perm int32
 * [B,H,row_cap] maps rows < perm_rows to positions, NULL = identity), then
 * out = sum (w / captured) v in fp64.  out fp64 [B,Hq,d]; captured fp64
 * [B,Hq] (the true mass of the subset; normalizer = exp(lse) * captured);
 * selected (nullable) uint8 [B,Hq,row_cap].  budget outside [1, n_tokens]
 * -> DP_ERR_INVALID with the reference message.  budgets (nullable) int32
 * [B,Hq] caps each q head's budget (min(budget, budgets[hq])): with the
 * output of dp_adaptive_token_budget this is
 * baseline_token_topp_fixed_budget (engine.py:340-370), the top-p prefix of
 * the top-`budget` candidates (selection.py:68-82). */
int dp_token_topk(const dp_cache_view* v, const int32_t* perm, int32_t perm_rows, int32_t gqa_group,
                  int32_t budget, const int32_t* budgets, const double* weights, double* out, double* captured, uint8_t* selected,
                  void* stream);

/* recovered_mass (metrics.py:26-39): true mass of a plan's exact tokens
 * (sink + window + members of state==2 clusters).  recovered fp64 [B,Hq]. */
int dp_recovered_mass(const dp_cache_view* v, int32_t gqa_group, const double* weights, const uint8_t* state,
                      double* recovered, void* stream);

/* cluster_approx_error (metrics.py:61-76): |true cluster mass -
 * exp(log_mass - lse)| for the cluster at each estimated rank (order from
 * dp_select).  errors fp64 [B,Hq,cluster_cap], rank order. */
int dp_cluster_approx_error(const dp_cache_view* v, int32_t gqa_group, const double* weights, const double* lse,
                            const double* log_mass, const int32_t* order, double* errors, void* stream);

/* adaptive_token_budget (metrics.py:41-50): the minimal number of tokens
 * whose true mass reaches p (searchsorted(cumsum(sorted desc), p, 'left')
 * + 1; n_tokens + 1 when the total never reaches p).  budget int32 [B,Hq]. */
int dp_adaptive_token_budget(const dp_cache_view* v, int32_t gqa_group, const double* weights, double p,
                             int32_t* budget, void* stream);

/* Mixed exact/approximate attention in fp64 (mixed_attention,
 * engine.py:216-252) with the same row/pseudo-row sets as
 * dp_sparse_attention, one CTA per q head, deterministic: the evaluation
 * path of the experiment runner (cli.py), not the decode hot path.
 * state == NULL treats every cluster as exact (full attention over all
 * rows).  out fp64 [B,Hq,d]; lse (nullable) fp64 [B,Hq]. */
int dp_mixed_attention_f64(const dp_cache_view* v, const void* q, int32_t q_dtype, int32_t gqa_group, double scale,
                           const double* log_mass, const uint8_t* state, double* out, double* lse, void* stream);

/* ---------------------------------------------------------------------- */
/* prefill clustering (build_clustered_cache, clustering.py:266-314)        */
/* ---------------------------------------------------------------------- */

typedef struct dp_cluster_params {
  int32_t batch, kv_heads, head_dim, dtype;
  int32_t n_tokens, sink, window;
  int32_t k;          /* requested clusters (already clamped to middle) */
  int32_t max_iters;
  int32_t fp64_assign; /* 1: fp64 distances (reference-exact); 0: fp32 FFMA; 2: tcgen05 tensor cores
                          (bf16 keys, head_dim 64/128, k <= 4096; winners re-scored in fp64) */
} dp_cluster_params;

/* Workspace for dp_cluster_build. */
size_t dp_cluster_workspace_bytes(const dp_cluster_params* p);

/* k-means++ init (clustering.py:36-55, replaying the host RNG stream),
 * Lloyd with empty-cluster drop (clustering.py:58-107), then the
 * cluster-contiguous tables.
 *   src_keys/src_values [B,H,n_tokens,d] position order (dtype)
 *   first_pick int32 [B*H]      rng.integers(n) of each head's stream
 *   uniforms  fp64 [B*H, k-1]   rng.random() draws of each head's stream
 *   alt_picks int32 [B*H, k-1]  (nullable) per-step explicit picks used from
 *                               step degenerate_from[b*H+h] on (rng.integers
 *                               draws once the sampling mass hits 0)
 *   degenerate_from int32 [B*H] (nullable; in/out) in: step from which
 *                               alt_picks apply (k = never); out: first step
 *                               whose sampling mass was 0 (k = none)
 * Outputs (device, caller-owned):
 *   dst_keys/dst_values [B,H,row_cap,d] cluster-ordered rows (row_cap >= n_tokens)
 *   offs [B,H,cluster_cap+1], nclusters [B,H], centroids/value_means fp32
 *   [B,H,cluster_cap,d] (cluster_cap >= k), perm int32 [B,H,row_cap]
 *   (original position of every row), objective fp64 [B*H, max_iters]
 *   (per-iteration sum of squared distances), iters int32 [B*H]. */
int dp_cluster_build(const dp_cluster_params* p, const void* src_keys, const void* src_values,
                     const int32_t* first_pick, const double* uniforms, const int32_t* alt_picks,
                     int32_t* degenerate_from, void* dst_keys, void* dst_values, int32_t row_cap,
                     int32_t* offs, int32_t* nclusters, float* centroids, float* value_means,
                     int32_t cluster_cap, int32_t* perm, double* objective, int32_t* iters,
                     void* workspace, size_t workspace_bytes, void* stream);

/* Profiling aid: %globaltimer stamps (ns) of the last dp_plan launch's first
 * cluster, [16 ranks][24 phase events], copied to host memory. */
int dp_debug_plan_timing(unsigned long long* out); /* [16][24] */
/* Profiling aid: clock64 at the first / last stamp of the same launch [16][2]. */
int dp_debug_plan_clock(unsigned long long* out);
/* Profiling aid: per-CTA %globaltimer stamps of the last bf16 attention
 * launch, [512 CTAs][12 events]: start, prefix loaded, first stage landed,
 * main loop done, flushed, exit. */
int dp_debug_attn_timing(unsigned long long* out);
/* Profiling switches: key 0 = attention flags (bit 0: skip the math, stream
 * K/V only); key 1 = force the plan cluster size (8 or 16; 0 = auto); key 3 = 1
 * runs k-means++ seeding on one CTA per head instead of an 8-CTA cluster;
 * key 4 = the one-launch step's L2 prefetch margin in 0.1-nat units (0 = off);
 * key 5 = force the one-launch step's cluster size (0 = auto); key 6 = 0
 * enables the one-launch step in dp_decode_step (default 1: off -- measured
 * slower than dp_plan + dp_attend at 32K and 128K); key 7 = the
 * one-launch step's profiling bits (1: skip the attention math, 2: skip the
 * K/V loads).
 * Never set on the product path. */
int dp_debug_set(int key, int value);
/* Profiling aid: %globaltimer stamps of the last one-launch step (cluster 0),
 * [16 ranks][16 events] followed by the selection's [16 CTAs][8 events]
 * (out must hold 384 values; built with DP_PROFILE=1). */
int dp_debug_step_timing(unsigned long long* out);
/* The thread-block cluster size the one-launch step uses at this geometry
 * (0: not supported -- dp_decode_step runs dp_plan + dp_attend). */
int dp_debug_step_cluster_size(const dp_cache_view* v, int G);
/* Profiling aid: co-resident plan clusters at this geometry for cluster size
 * cl (cudaOccupancyMaxActiveClusters). */
int dp_debug_plan_occupancy(const dp_cache_view* v, int G, int cl);

/* Lower-level pieces of the above (used by the parity tests). */
/* k-means++ picks only: picks int32 [B*H, k]. */
int dp_kmeanspp(const dp_cluster_params* p, const void* src_keys, const int32_t* first_pick,
                const double* uniforms, const int32_t* alt_picks, int32_t* degenerate_from,
                int32_t* picks, void* workspace, size_t workspace_bytes, void* stream);

/* nearest_centroid (_kernels_py.py:58-77, _kernels_cy.pyx:115-140): points
 * [n,d] (dtype), centroids fp64 [k,d]; assign int32 [n], sqdist fp64 [n];
 * ties -> lowest index. */
int dp_nearest_centroid(const void* points, int32_t dtype, int32_t n, int32_t d,
                        const double* centroids, int32_t k, int32_t fp64, int32_t* assign,
                        double* sqdist, void* stream);

/* ---------------------------------------------------------------------- */
/* sequence sharding with the reference's GLOBAL semantics (config 5,     */
/* >= 512K tokens over P GPUs).  The host layer             */
/* (paper_2602_05191_b200/seqshard.py) runs the collectives between them. */
/* ---------------------------------------------------------------------- */

/* One k-means++ step's distance update (clustering.py:45,53) over this
 * rank's middle points [units, n, d]: dsq = |x - centre|^2 (first != 0) or
 * min(dsq, |x - centre|^2), fp64; sums[u] = the local sum (fixed order). */
int dp_kmpp_shard_dsq(const void* points, int32_t dtype, int32_t units, int32_t n, int32_t d, const double* centre,
                      int32_t first, double* dsq, double* sums, void* stream);

/* The step's pick (clustering.py:49, Generator.choice(p = dsq / total)): with
 * all_sums [world, units] the all-gathered local sums, the centre is the first
 * GLOBAL point whose running dsq sum exceeds uniforms[u] * total; pick_in
 * (nullable) forces a global index per unit (the first centre,
 * clustering.py:42).  This rank holds global middle indices
 * [global_base, global_base + n).  centre_out [units, d] fp64 = the row on
 * the owning rank, zeros elsewhere (an all-reduce sum hands it to every
 * rank); pick_out [units] = the global index on the owner, -1 elsewhere, -2
 * when the total mass is zero (the reference then draws rng.integers). */
int dp_kmpp_shard_pick(const void* points, int32_t dtype, int32_t units, int32_t n, int32_t d, const double* dsq,
                       const double* all_sums, int32_t world, int32_t rank, const double* uniforms,
                       const int32_t* pick_in, int64_t global_base, double* centre_out, int32_t* pick_out,
                       void* stream);

/* Lloyd's local half (clustering.py:100-106): fp64 sums [units, k, d] and
 * member counts [units, k] of this rank's points per cluster, each cluster's
 * members added in ascending position order (deterministic; an all-reduce
 * of [k, d + 1] gives the global means).  assign [units, n] int32. */
size_t dp_lloyd_shard_workspace_bytes(int32_t units, int32_t n, int32_t k);
int dp_lloyd_shard_sums(const void* points, int32_t dtype, int32_t units, int32_t n, int32_t d,
                        const int32_t* assign, int32_t k, double* sums, int64_t* counts, void* workspace,
                        size_t workspace_bytes, void* stream);

/* Two-stage top-p (engine.py:180-213, selection.py:36-65) over log-mass rows
 * of ANY length -- the all-gathered per-shard slices of one global cluster
 * table (K = 32,766 at 1M tokens).  log_mass [rows, ld] fp64, nclusters
 * [rows] the valid length of each row; state [rows, ld] (2 exact / 1 approx
 * / 0 dropped), counts [rows, 2] = (|C_p|, |C_exact|).  One CTA per row. */
size_t dp_select_global_workspace_bytes(int32_t rows, int32_t ld);
int dp_select_global(const double* log_mass, int32_t rows, int32_t ld, const int32_t* nclusters, double p1,
                     double p2, uint8_t* state, int32_t* counts, void* workspace, size_t workspace_bytes,
                     void* stream);

/* The exchange step's merge (engine.py:234-246 across shards): partials
 * out_parts [parts, rows, d] fp32 with lse_parts [parts, rows] (-inf: empty)
 * -> out [rows, d], lse [rows]; fp64 weights. */
/* dp_select_global over the all-gathered slices read IN PLACE:
 * log_mass_parts [parts, rows, part_len] (slot k of part p is global entry
 * p * part_len + k; holes hold -inf), state [rows, parts * part_len].  The
 * one-launch cluster form only: parts * part_len <= 65536 (else
 * DP_ERR_UNSUPPORTED). */
int dp_select_global_parts(const double* log_mass_parts, int32_t rows, int32_t parts, int32_t part_len,
                           const int32_t* nclusters, double p1, double p2, uint8_t* state, int32_t* counts,
                           void* workspace, size_t workspace_bytes, void* stream);

int dp_lse_merge(const float* out_parts, const float* lse_parts, int32_t parts, int32_t rows, int32_t d, float* out,
                 float* lse, void* stream);

/* ---------------------------------------------------------------------- */
/* the reference's per-query kernel plugin seam (kernels.py:47-96) as     */
/* HOST-pointer calls: the eight operations a DOUBLEP_KERNELS backend     */
/* provides (_kernels_cy.pyx:21-157), computed on the current device      */
/* (csrc/seam.cu).  Synchronous; matrices DP_F32 or DP_F64 row-major      */
/* [rows, d]; idx (int64, NULL = all rows) must lie in [0, rows).  These  */
/* replace the Cython backend one call at a time; the decode path above   */
/* does not use them.                                                     */
/* ---------------------------------------------------------------------- */
#define DP_F64 2 /* seam matrices only */

/* scaled_logits / gather_scaled_logits (kernels.py:47-57): out[i] =
 * (keys[idx[i]] . q) * scale, fp64 sequential over d -- bit-identical to
 * _kernels_cy.pyx:21-50. */
int dp_kn_scaled_logits(const void* keys, int32_t dtype, int64_t rows, int32_t d, const int64_t* idx, int64_t n_idx,
                        const double* q, double scale, double* out);
/* logsumexp (kernels.py:60-62, _kernels_cy.pyx:53-65): n >= 1 (else
 * DP_ERR_INVALID); exact max for one element. */
int dp_kn_logsumexp(const double* x, int64_t n, double* out);
/* softmax (kernels.py:65-67, _kernels_cy.pyx:68-83): out [n]. */
int dp_kn_softmax(const double* x, int64_t n, double* out);
/* weighted_sum / gather_weighted_sum (kernels.py:70-76): out[d] =
 * sum_i w[i] * mat[idx[i]], fp64. */
int dp_kn_weighted_sum(const double* w, const void* mat, int32_t dtype, int64_t rows, int32_t d, const int64_t* idx,
                       int64_t n_idx, double* out);
/* nearest_centroid (kernels.py:79-87, _kernels_cy.pyx:115-140): direct
 * difference in fp64, strict '<' (ties -> lowest index); assign int64 [n],
 * sqdist fp64 [n]; k >= 1. */
int dp_kn_nearest_centroid(const void* points, int32_t dtype, int64_t n, int32_t d, const double* centroids,
                           int32_t k, int64_t* assign, double* sqdist);
/* sorted_prefix_count (kernels.py:90-96, _kernels_cy.pyx:143-157): smallest
 * prefix with running fp64 sum >= p (n if never); DP_ERR_INVALID "input not
 * sorted" on an ascent among the scanned entries. */
int dp_kn_sorted_prefix_count(const double* sorted_probs, int64_t n, double p, int64_t* count);

#ifdef __cplusplus
}
#endif
#endif /* DOUBLEP_B200_H */
