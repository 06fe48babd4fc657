// train.cuh -- launch interface of the per-batch training kernels (train.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace lgd {

// ComplEx / TransE: K4's dst / negative items read IR1 = combine(src, rel) as
// K3 wrote it (P x d f64) instead of recombining the src snapshot with the
// relation row (FM +4.6%, Friendster +0.5%).  DistMult keeps the snapshot: its
// recombination is cheaper than reading the 2x wider row (TW -1.8% with the
// snapshot's 48 MB L2 window on IR1, -2.0% without; -DLGD_K4_IR1_ALL to measure).
__host__ __device__ constexpr bool k4_ir1(int kind) {
#if defined(LGD_K4_IR1_ALL)
  return kind != 0;
#elif !defined(LGD_NO_K4_IR1)
  return kind == 2 || kind == 3;
#else
  return false && kind;
#endif
}

struct SegLists {  // K4 v2 long-segment list (launch_long_list)
  uint32_t* long_head;        // <= n / 33 + 1 (heads of segments of > 32 items, ascending)
  uint32_t* long_end;         // same count: end item of each
  uint32_t* long_chunk_base;  // + 1: exclusive prefix of their 32-item chunk counts
  uint32_t* long_first;       // nb + 1: first long segment of each batch
  uint32_t* nlong;            // 1
  void* temp;
  size_t temp_bytes;
};

struct GradCompact {  // compact batch_gradients (launch_train_batch phase 1, then phase 2)
  uint32_t* node_seg;         // segment heads of the sorted node contributions (P (k+2))
  uint32_t* rel_seg;          // of the sorted relation ids (P), or null (untyped)
  uint32_t* rel_skeys;        // the relation sort's output (P)
  uint32_t* rel_svals;
  uint32_t* counts;           // [unique nodes, unique relations] (device)
  void* temp;
  size_t temp_bytes;
};

struct BatchArgs {
  int kind;
  uint32_t dim;
  uint32_t k;
  uint64_t P;                 // positives in this batch
  uint64_t num_nodes;         // table rows (LGD_CHECKED bounds; num_rels below)
  const uint32_t* edges;      // P x 3 (src, rel, dst), device
  const uint32_t* negs;       // P x k, device
  float* theta;               // V x d embeddings
  float* state;               // V x d Adagrad accumulators
  float* rel_theta;           // R x d
  double* rel64;              // R x d FP64 copy K3 writes for K4 (small R), or null
  float* rel_state;           // R x d
  double lr;
  double eps;
  // scratch (sized for the largest batch)
  double* w;                  // P x k softmax weights
  double* mix;                // P x d  sum_j w_j neg_j - dst
  double* ir1;                // P x d  IR1 = combine(src, rel): written by K3 and read by K4's dst /
                              // negative items when non-null (k4_ir1 models, vector-lane dims)
  float* snap;                // P x d  pre-update source rows
  double* loss;               // per-positive loss: P values (shared mode), or K3's
                              // parts f_pos | row_max | sum (3 x P, loss_parts)
  int loss_parts;
  uint32_t* node_keys;        // P x (k+2) contribution node ids (dst, negs, src)
  uint32_t* node_vals;        // P x (k+2) payloads (p << slot_bits) | slot
  uint32_t* rel_keys;         // P relation ids
  // presorted: the node contributions were keyed and sorted once for the whole
  // bucket (launch_bucket_keys / sort_bucket): skeys / svals point at this
  // batch's run of the bucket's sorted arrays, whose keys carry the batch
  // index above key_mask; K3 writes no node keys and the batch sorts nothing
  int presorted;
  uint32_t key_mask;          // pool-index bits of a sorted key (all ones unless presorted)
  const uint32_t* iota;       // 0..P*(k+2)-1
  uint32_t* skeys;            // sorted keys
  uint32_t* svals;            // sorted contribution indices
  void* sort_temp;
  size_t sort_temp_bytes;
  double* part_first;         // chunks x d
  double* part_last;          // chunks x d
  uint8_t* chunk_flags;       // chunks
  uint32_t* span_list;        // chunks holding the head of a chunk-spanning segment
  unsigned int* span_count;   // entries in span_list
  unsigned long long* counters;  // [0] unique nodes, [1] unique rels (accumulated)
  double* batch_loss_out;     // one double: this batch's loss
  int slot_bits;              // bits for a slot in [0, k+1]
  int rel_bits;               // > 0: the relation id rides in the payload above the slot
                              // (p << (slot_bits + rel_bits) | rel << slot_bits | slot)
  // resident sampling pool (<= 3 node ranges, ascending): contribution keys
  // are pool indices, so the radix sort needs bits_for(pool size) bits only
  uint64_t pool_first[3];
  uint64_t pool_end[3];       // inclusive prefix of range sizes
  int pool_n;
  int node_key_bits;
  int rel_key_bits;
  // gradient-only mode (operator-level batch_gradients): dense V x d / R x d
  double* grad_nodes;
  uint8_t* grad_node_flag;
  double* grad_rels;
  uint8_t* grad_rel_flag;
  int sm_count;
  // shared-negative chunks (shared.cu): chunk = 0 is the reference's
  // per-positive mode; otherwise negs holds nch x k shared ids
  uint32_t chunk;
  uint32_t kpad, dpad, tpc;   // k -> multiple of 128, dim -> multiple of 16, tiles per chunk
  uint64_t nch;               // chunks in this batch
  float* sh_A;                // IR1 tiles, core-matrix layout (nch x tpc x 128 rows x dpad)
  float* sh_AT;               // IR1^T per 64-positive slice (dpad x 64), core-matrix layout
  float* sh_D;                // dst rows per padded tile row (rows x dim), prep -> SG2's tail
  float* sh_B;                // negative rows, core-matrix layout (nch x kpad x dpad)
  float* sh_BT;               // N^T per 64-negative block (dpad x 64)
  float* sh_rowc;             // per padded tile row: log2 of the softmax denominator,
                              // M log2e + log2 Z (weight = 2^(s log2e - c))
  double* sh_pos;             // P positive scores (FP64)
  float* sh_G;                // nch x kpad x dim: gradient of every shared negative
  // relation pass on a side stream (typed models, updating batches): it needs
  // only K3's outputs, so its sort and segmented sums overlap the node pass;
  // the relation rows are updated after K4, which reads them pre-update.
  // side == nullptr: sequential relation pass.
  // K4 v2 (segment_heads): 0 = chunked pass 1 / pass 2; 1 = the bucket's
  // long-segment list is ready (seg_keys / seg_vals = the bucket's sorted
  // arrays, this batch = items [seg_b0, seg_b0 + P(k+2)), batch index
  // seg_batch); 2 = build a one-batch list after this batch's sort
  int seg_mode;
  int k4_ws;                  // K4 v3: warp-specialised producer / consumer kernel
  const uint32_t* seg_keys;
  const uint32_t* seg_vals;
  uint64_t seg_b0;
  uint32_t seg_batch;
  uint32_t* long_head;
  uint32_t* long_end;
  uint32_t* long_chunk_base;
  uint32_t* long_first;
  SegLists seg_lists;         // the buffers, for a one-batch list (seg_mode 2)
  cudaEvent_t ev_long, ev_long_done;  // long segments on the side stream
  const GradCompact* gc;      // non-null: stop after the sorts (compact gradients, phase 1)
  cudaStream_t side;
  cudaEvent_t ev_scored, ev_rel;
  uint64_t num_rels;
  uint32_t* rel_skeys;
  uint32_t* rel_svals;
  void* rel_sort_temp;
  size_t rel_sort_temp_bytes;
  double* rel_part_first;
  double* rel_part_last;
  uint8_t* rel_chunk_flags;
  uint32_t* rel_span_list;
  unsigned int* rel_span_count;
  double* rel_grad;           // R x dim, rows written for touched relations
  uint8_t* rel_touched;       // R
};

struct SharedShape {
  uint32_t dpad, kpad, tpc;
  uint64_t nch;
};
SharedShape shared_shape(uint32_t dim, uint32_t k, uint32_t chunk, uint64_t P);
size_t shared_smem_bytes(uint32_t dpad);
// prep + negative gather + the three tcgen05 kernels (scores, mix, gradients)
void launch_shared_scores(const BatchArgs& a, cudaStream_t st);

struct BatchEvents {  // optional per-phase timing (profiling mode)
  cudaEvent_t ev[5];
  bool enabled;
};

size_t batch_sort_temp_bytes(uint64_t max_items);
// Bucket-level node contributions: keys (batch << node_key_bits) | pool index
// and payloads of every batch of an m-edge bucket (batches of B positives;
// a = the bucket's batch arguments), then one stable radix sort of them all.
// The sorted run of batch b starts at item b * B * (k + 2) and equals the
// per-batch sort of K3's keys.  Returns the buffer holding the result.
void launch_bucket_keys(const BatchArgs& a, uint64_t m, uint64_t B, uint32_t* keys,
                        uint32_t* vals, cudaStream_t st);
size_t bucket_sort_temp_bytes(uint64_t max_items);
// Long-segment list of sorted keys (K4 v2): heads of the segments of more
// than 32 items (ascending), their ends, the exclusive prefix of their
// 32-item chunk counts and, per batch b < nb (items [b batch_items, ...)),
// the first long segment of the batch; first[nb] = nlong (device count).
size_t long_list_temp_bytes(uint64_t max_items);
void launch_long_list(const uint32_t* keys, uint64_t n, uint64_t batch_items, uint32_t nb,
                      const SegLists& lists, cudaStream_t st);
// Compact gradients, phase 2 (after launch_train_batch with a.gc set and the
// counts read back): row s of node_grads / rel_grads = the FP64 gradient of
// unique id s, ids ascending.
void launch_grads_phase2(const BatchArgs& a, uint64_t num_nodes, uint64_t num_rels,
                         uint32_t* node_ids, double* node_grads, uint32_t* rel_ids,
                         double* rel_grads, cudaStream_t st);
size_t grads_select_temp_bytes(uint64_t max_items);
// 16-byte vectors per lane of K4's vector kernels for (kind, dim); 0 = the
// 8-lane-group fallback (which never reads K3's IR1 rows)
int k4_vec_width(int kind, uint32_t dim);
void launch_segment_list(const uint32_t* keys, uint64_t n, int shift, uint32_t nb,
                         const SegLists& lists, int sm_count, cudaStream_t st);
int sort_bucket(void* temp, size_t temp_bytes, uint32_t* keys[2], uint32_t* vals[2],
                uint64_t items, int key_bits, cudaStream_t st);
size_t score_smem_bytes(uint32_t dim, uint32_t k);
// K3 -> loss reduce -> sort -> K4 (pass 1, 2) -> relation path.
void launch_train_batch(const BatchArgs& a, cudaStream_t st, const BatchEvents* ev);
// Multi-GPU lock-step relations: pack a dense gradient [R x d] + touched
// flags into [R x (d+1)] (the buffer the ranks sum), and apply one Adagrad
// step to every touched row from a summed buffer.
void launch_rel_pack(const double* grad, const uint8_t* flag, uint64_t R, uint32_t d, double* out,
                     cudaStream_t st);
void launch_rel_apply(const double* summed, float* rel_theta, float* rel_state, uint64_t R,
                      uint32_t d, double lr, double eps, cudaStream_t st);

}  // namespace lgd
