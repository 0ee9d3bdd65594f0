// Internal declarations shared by the decode translation units.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "doublep_b200.h"

namespace dp {

constexpr int kChunkRows = 128;   // rows per split-KV work item
constexpr int kAttnThreads = 512;  // one (head, row) logit / (head, dim) output per thread at G = 4
constexpr int kMaxPartSlots = 256;  // persistent attention grid cap (partials per head)

// Row stride of the sparse accumulators: o[d], l, 3 pad floats (16-B aligned rows
// for vector reductions).
__host__ __device__ constexpr int acc_stride(int d) { return 2 * d; }  // d/2 vectors (o[c], o[c+1], l, count)

// Device work lists (one set per (b, kv head)), carved from the workspace.
constexpr int kWlThreads = 256;    // split worklist: clusters per chunk CTA
constexpr int kWlMaxChunks = 64;   // up to 16384 clusters per head

struct WorkLists {
  int4* runs;     // [BH][cap+2] {row start, len, head mask, virtual row prefix}
  int2* approx;   // [BH][cap]   {cluster id, head mask}
  int* nruns;     // [BH]
  int* nrows;     // [BH]  union exact rows (incl. sink/window)
  int* napprox;   // [BH]  union approx clusters
  int* nchunks;   // [BH]
  int* stats;     // nullable [BH][4]
  int* rowidx;    // [BH][row_cap] packed union rows: (head mask << 24) | physical row
  int* counters;  // [BH] partial-completion counters (zero between launches)
  int* chunk_prefix;  // [BH+1] exclusive prefix of nchunks over heads (+ total)
  int* done;      // [1] producer-completion counter (zero between launches)
  float* apart;   // [BH][G][4+d] approx pseudo-row partial per q head (m, l, -, -, o[d]); m = -inf: none
  float* acc;     // [BH][G][acc_stride(d)] sparse attention accumulators: d/2 vectors (o[c], o[c+1], l, count) scaled by 2^-ref (zero between launches)
  float* refm;    // [BH][G] reference max (log2 units) of those accumulators, written by the plan
  int* wlp;       // [BH][kWlMaxChunks][4] split worklist: per-chunk (rows, approx, exact) totals
  unsigned long long* wkey;  // [BH][G][2] split worklist: ordered keys of the log-mass / sink-window maxima (0 = unset)
  int max_chunks;
};

template <typename Acc>
struct Partials {
  Acc* m;  // [BH][max_chunks][G]
  Acc* l;
  Acc* o;  // [BH][max_chunks][G][d]
  int max_chunks;
};

// Called by ONE thread of every producer block (one per head) after its
// nchunks entry is written: the last producer to finish writes the exclusive
// prefix of nchunks over all heads (and the total) and re-arms the counter.
__device__ __forceinline__ void publish_chunk_prefix(const WorkLists& wl, int BH) {
  __threadfence();
  if (atomicAdd(wl.done, 1) != BH - 1) return;
  __threadfence();
  int acc = 0;
  for (int b = 0; b < BH; ++b) {
    wl.chunk_prefix[b] = acc;
    acc += *((volatile int*)&wl.nchunks[b]);
  }
  wl.chunk_prefix[BH] = acc;
  *wl.done = 0;
  __threadfence();
}

size_t decode_ws_layout(const dp_cache_view* v, int G, WorkLists* wl, void** parts, size_t* part_bytes,
                        char* base);
int select_padded(int K);

cudaError_t launch_score(const dp_cache_view& v, const void* q, int qdt, int G, double scale, double* lm,
                         cudaStream_t st);
cudaError_t launch_select(const dp_cache_view& v, int G, double p1, double p2, const double* lm,
                          uint8_t* state, int* counts, int* order, double* cum, double* probs,
                          cudaStream_t st);
cudaError_t launch_worklist(const dp_cache_view& v, int G, const uint8_t* state, int* stats, void* ws,
                            cudaStream_t st, const double* lm, const void* q = nullptr, int qdt = 0,
                            double scale = 0.0);
cudaError_t launch_attend(const dp_cache_view& v, const void* q, int qdt, int G, double scale, const double* lm,
                          float* out, float* lse, void* ws, bool dense, cudaStream_t st);
cudaError_t launch_attn_tc(const dp_cache_view& v, const void* q, int qdt, int G, double scale, const double* lm,
                           WorkLists wl, Partials<float> pt, float* out, float* lse, bool dense, cudaStream_t st);
cudaError_t launch_plan(const dp_cache_view& v, const void* q, int qdt, int G, double scale, double p1, double p2,
                        double* lm, uint8_t* state, int* counts, int* stats, void* ws, cudaStream_t st, int mode = 0,
                        int state_ld = 0);
bool plan_supported(const dp_cache_view& v, int G);
// 2-D TMA map over all centroid rows [B*H*cap, d] fp32 (32-float x 128-row boxes, 128B swizzle), cached
cudaError_t centroid_tmap(const dp_cache_view& v, CUtensorMap* m);
// step.cu: the whole decode step (score + select + attention + merge) in ONE launch when every
// (sequence, kv head) thread-block cluster is co-resident (batch-1 latency path)
bool step_supported(const dp_cache_view& v, int G, int qdt);
cudaError_t launch_step(const dp_cache_view& v, const void* q, int qdt, int G, double scale, double p1, double p2,
                        double* lm, uint8_t* state, int* counts, int* stats, float* out, float* lse, void* ws,
                        cudaStream_t st);
cudaError_t launch_topk_state(const dp_cache_view& v, int G, int budget, const int* order, uint8_t* state,
                              int* counts, cudaStream_t st);
cudaError_t launch_append(const dp_cache_view& v, const void* nk, const void* nv, cudaStream_t st);
// metrics.cu
cudaError_t launch_token_weights(const dp_cache_view& v, const void* q, int qdt, int G, double scale, double* w,
                                 double* lse, cudaStream_t st);
cudaError_t launch_token_topk(const dp_cache_view& v, const int* perm, int perm_rows, int G, int budget,
                              const int* budgets, const double* w, double* out, double* captured, uint8_t* selected, cudaStream_t st);
cudaError_t launch_recovered_mass(const dp_cache_view& v, int G, const double* w, const uint8_t* state,
                                  double* recovered, cudaStream_t st);
cudaError_t launch_cluster_error(const dp_cache_view& v, int G, const double* w, const double* lse,
                                 const double* lm, const int* order, double* errors, cudaStream_t st);
cudaError_t launch_mixed_f64(const dp_cache_view& v, const void* q, int qdt, int G, double scale, const double* lm,
                             const uint8_t* state, double* out, double* lse, cudaStream_t st);
cudaError_t launch_adaptive_budget(const dp_cache_view& v, int G, const double* w, double p, int* budget,
                                   cudaStream_t st);
// shard.cu: sequence-sharded Double-P with global semantics (config 5)
cudaError_t launch_kmpp_dsq(const void* pts, int dtype, int units, int n, int d, const double* centre, int first,
                            double* dsq, double* sums, cudaStream_t st);
cudaError_t launch_kmpp_pick(const void* pts, int dtype, int units, int n, int d, const double* dsq,
                             const double* all_sums, int P, int rank, const double* u_draw, const int* pick_in,
                             long long gbase, double* centre_out, int* pick_out, cudaStream_t st);
size_t lloyd_sums_ws_bytes(int units, int n, int k);
cudaError_t launch_lloyd_sums(const void* pts, int dtype, int units, int n, int d, const int* assign, int k,
                              double* sums, long long* counts, void* ws, cudaStream_t st);
size_t select_global_ws_bytes(int rows, int ld);
extern int g_gsel_path;  // dp_debug_set(11, .)
int set_gsel_dbg(int v);  // dp_debug_set(12, .)
cudaError_t launch_select_global(const double* lm, int rows, int ld, const int* Ks, double p1, double p2,
                                 uint8_t* state, int* counts, void* ws, cudaStream_t st, int part_len = 0);
bool select_global_parts_supported(int parts, int part_len);
cudaError_t launch_lse_merge(const float* out_parts, const float* lse_parts, int P, int rows, int d, float* out,
                             float* lse, cudaStream_t st);

}  // namespace dp
