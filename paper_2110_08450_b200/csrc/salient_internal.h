// Internal (C++) interface between the kernel files and the C-ABI layer.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "salient_b200.h"

namespace sal {

constexpr int kRngSplitmix = SAL_RNG_SPLITMIX;
constexpr int kRngPhilox = SAL_RNG_PHILOX;

struct GraphDev {
  int64_t num_nodes;
  int64_t num_edges;
  const int64_t* indptr;
  const int32_t* indices;
};

typedef sal_batch_desc BatchDesc;

struct IdMapDev {
  unsigned long long* table;
  int log2cap;
  int32_t* globals;
  int64_t* size_out;  // seed insertion writes the initial size here
};

struct HopKey {
  uint64_t prefix;       // splitmix key prefix (used when derive == 0)
  uint64_t global_seed;  // derive the prefix on device from desc->batch_id
  uint32_t hop;
  uint32_t batch;        // batch id when no device descriptor is given
  int32_t derive;
};


int num_sms();
// thread-local error message of sal_last_error(); returns `code`
int set_error(int code, const char* fmt, ...);
void count_launch(int kernels);
int log2_exact(int64_t cap);
size_t scan_ws_bytes(int64_t max_items);

// a device epoch plan: desc_all[3 * step] rows, the next step at *cursor
struct PlanCursor {
  const int64_t* desc_all;
  int64_t n_steps;
  int64_t* cursor;
};
cudaError_t launch_seed_insert_next(const int64_t* seeds_base, const PlanCursor& pc,
                                    BatchDesc* desc_out, const IdMapDev& m, cudaStream_t st);
cudaError_t launch_seed_insert(const int64_t* seeds_base, const BatchDesc* desc,
                               const IdMapDev& m, int64_t max_seeds, cudaStream_t st);
cudaError_t launch_hop_count(const GraphDev& g, const int32_t* globals, const int64_t* n_dst,
                             int64_t max_dst, int32_t fanout, int32_t* dst_indptr,
                             int64_t* e_total, void* scan_ws, cudaStream_t st, bool ws_zeroed = false);
cudaError_t launch_hop_sample(const GraphDev& g, const IdMapDev& m, const int64_t* n_dst,
                              int64_t max_dst, int32_t fanout, HopKey hk, const BatchDesc* desc,
                              int32_t policy, const int64_t* inject_pos,
                              const int32_t* dst_indptr, int32_t* src_glob, int32_t* slot,
                              int32_t* draws_out, cudaStream_t st, int lanes = 0,
                              int blocks_per_sm = 0);
cudaError_t launch_rehash(const IdMapDev& m, int64_t n, cudaStream_t st);
cudaError_t launch_keys_insert(const int64_t* keys, int64_t n, const IdMapDev& m,
                               int32_t* src_glob, int32_t* slot, int64_t* e_total,
                               cudaStream_t st);
// a hop's deferred resolve (flag_scan kept each edge's table word in `words`)
struct ResolveJob {
  const int32_t* words;
  const int64_t* e_total;
  const int64_t* size_old;
  const int32_t* rank_of;
  int32_t* src_local;   // null: no job
};
// the next hop's count + scan, fused into the resolve launch of this hop
struct NextCount {
  GraphDev g;
  int32_t fanout;
  int64_t max_dst;
  int32_t* dst_indptr;
  int64_t* e_total;
  void* scan_ws;  // zeroed by the caller
};
cudaError_t launch_hop_relabel(const IdMapDev& m, const int64_t* e_total, int64_t max_edges,
                               const int64_t* size_old, int64_t* size_new,
                               const int32_t* src_glob, const int32_t* slot, int32_t* rank_of,
                               int32_t* src_local, void* scan_ws, cudaStream_t st,
                               bool ws_zeroed = false, const NextCount* next = nullptr,
                               bool defer_resolve = false);

cudaError_t launch_sample_mean(const GraphDev& g, const int32_t* globals, const int64_t* n_dst,
                               int64_t max_dst, int32_t fanout, HopKey hk, const BatchDesc* desc,
                               int32_t policy, const void* table, int64_t t_stride, int32_t cols,
                               void* out, int32_t out_dtype, int64_t out_stride, int64_t self_off,
                               int64_t* size_unknown, int bps_cap, unsigned long long* reset_table,
                               int64_t table_words, void* reset_scan, int64_t scan_bytes,
                               const ResolveJob& resolve, cudaStream_t st);
cudaError_t launch_gather_rows(const void* x, int64_t x_rows, int32_t cols, int64_t x_stride,
                               int32_t in_dtype, const void* ids, int32_t id_bytes,
                               const int64_t* n_dev, int64_t n, void* out, int64_t out_stride,
                               int32_t out_dtype, cudaStream_t st);
cudaError_t launch_gather_labels(const int64_t* y, const int64_t* seeds_base,
                                 const BatchDesc* desc, int64_t max_n, int64_t* out,
                                 cudaStream_t st);

cudaError_t launch_segment_mean_fwd(const int32_t* indptr, const int32_t* src,
                                    const int32_t* globals, const int64_t* n_dst_dev,
                                    int64_t n_pad, const void* h, int32_t h_dtype,
                                    int64_t h_stride, int32_t f, void* out, int32_t out_dtype,
                                    int64_t out_stride, cudaStream_t st, bool pad_fill = true);
cudaError_t launch_segment_mean_bwd(const int32_t* indptr, const int32_t* src,
                                    const int64_t* n_dst_dev, int64_t n_pad, const void* g_out,
                                    int32_t g_dtype, int64_t g_stride, int32_t f, float* g_h,
                                    int64_t gh_stride, cudaStream_t st);

}  // namespace sal
