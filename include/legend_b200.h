/*
 * legend_b200.h -- C ABI of the B200-native partitioned graph-embedding
 * trainer (drop-in for the reference trainer's hot path, arXiv 2505.09258
 * "Legend", reference sources under proj/ of the reference tree).
 *
 * Plain pointers and sizes only.  Host pointers unless a name says "device".
 * Every entry point returns an LGD_* code; the codes map 1:1 onto the
 * exception classes the reference throws, and
 * lgd_last_error() returns the message of the calling thread's last failure.
 * One host thread per context; device work runs on the context's streams.
 *
 * Layouts (identical to the reference so files / buffers move unchanged):
 *   edge record    u32 src, u32 rel, u32 dst (12 B)        graph.hpp:19-25
 *   untyped rel    0xffffffff                              graph.hpp:17
 *   partition p    node rows [stride*p, min(stride*(p+1), V)),
 *                  stride = ceil(V / n)                    graph.hpp:55-72
 *   E||S blob      rows*dim f32 embeddings, then rows*dim f32 Adagrad
 *                  state, row major, little endian         store.hpp:14-33
 */
#ifndef LEGEND_B200_H
#define LEGEND_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LGD_OK 0
#define LGD_INVALID_ARGUMENT 1 /* std::invalid_argument */
#define LGD_LOGIC_ERROR 2      /* std::logic_error      */
#define LGD_OUT_OF_RANGE 3     /* std::out_of_range     */
#define LGD_RUNTIME_ERROR 4    /* std::runtime_error, CUDA failures */

/* ScoreKind (train.hpp:13) */
#define LGD_MODEL_DOT 0
#define LGD_MODEL_DISTMULT 1
#define LGD_MODEL_COMPLEX 2
#define LGD_MODEL_TRANSE 3 /* -||s + r - t||; not in the reference */

#define LGD_NO_RELATION 0xffffffffu /* kNoRelation, graph.hpp:17 */

typedef struct lgd_context lgd_context;

/* TrainOptions (pipeline.hpp:89-97) + AdagradHyper (train.hpp:109-112).
 * Defaults of the reference CLI: lr 0.1, eps 1e-10, batch 100000, k 16,
 * shuffle on, seed 42 (legend_main.cpp:23-50). */
typedef struct {
  double learning_rate;
  double adagrad_epsilon;
  uint32_t batch_size;
  uint32_t negatives;
  int32_t shuffle;
  /* 0: the reference's independent negatives, `negatives` per positive
   * (train.cpp:365-373).  C > 0: shared-negative chunks -- every C
   * consecutive positives of a batch share `negatives` ids, drawn
   * ceil(P / C) * negatives per batch from the same bucket stream; scores on
   * the tensor cores (TF32 in, FP32 accumulate).  Dot / DistMult / ComplEx,
   * dim % 4 == 0, dim <= 128.  Not a reference mode: its oracle is the
   * reference batch math on the expanded negative list. */
  uint32_t shared_chunk;
  uint64_t seed;
} lgd_train_options;

/* EpochResult (pipeline.hpp:99-107) plus device-side accounting. */
typedef struct {
  double loss_sum;
  double loss_per_edge;
  uint64_t edges_trained;
  uint64_t buckets_trained; /* non-empty buckets only (pipeline.cpp:291, 314) */
  uint64_t batches;
  double wall_seconds;      /* host wall clock of the call */
  double device_ms;         /* CUDA-event time of the trained buckets */
  uint64_t unique_nodes;    /* sum over batches of |GradientSet.nodes| */
  uint64_t unique_rels;     /* sum over batches of |GradientSet.rels| */
  double algorithmic_bytes; /* sum_b P_b(12 + 4d(2+k+t)) + 16d(N_b + R_b) */
  uint64_t h2d_bytes;       /* host -> device bytes copied by the call's training loop */
  uint64_t d2h_bytes;       /* device -> host bytes of the results */
} lgd_epoch_result;

/* Per-kernel-class CUDA-event statistics (profiling mode). */
typedef struct {
  uint64_t launches;
  double total_ms;
  double algorithmic_bytes;
} lgd_kernel_stats;

#define LGD_KSTAT_SCORE 0   /* fused score / loss / gradient prep (K3)      */
#define LGD_KSTAT_SORT 1    /* contribution radix sort                        */
#define LGD_KSTAT_UPDATE 2  /* node segmented reduce + Adagrad (K4)           */
#define LGD_KSTAT_REL 3     /* relation sort + segmented reduce + Adagrad     */
#define LGD_KSTAT_SAMPLE 4  /* per-bucket negative draws (K2)                 */
#define LGD_KSTAT_SHUFFLE 5 /* per-bucket Fisher-Yates permutation + gather (K1) */
#define LGD_KSTAT_EVAL 6    /* lgd_evaluate: candidates + scores (K6)          */
#define LGD_KSTAT_COUNT 7

const char* lgd_last_error(void);

/* ---------------------------------------------------------------- context */

/* ScoreModel{kind, dim} (train.hpp:15-23) + options; device = CUDA ordinal. */
int lgd_create(lgd_context** out, int model_kind, uint32_t dim, const lgd_train_options* options,
               int device);
void lgd_destroy(lgd_context* ctx);
int lgd_set_options(lgd_context* ctx, const lgd_train_options* options);

/* ------------------------------------------------------------------ graph */

/* Graph (graph.hpp:29-35): edges = num_edges 12-byte records. */
int lgd_set_graph(lgd_context* ctx, const uint32_t* edges, uint64_t num_edges, uint64_t num_nodes,
                  uint64_t num_relations);
/* Synthetic power-law graph generated on the device (bench workloads). */
int lgd_generate_graph(lgd_context* ctx, uint64_t num_nodes, uint64_t num_relations,
                       uint64_t num_edges, double zipf_exponent, uint64_t seed);
int lgd_get_graph(lgd_context* ctx, uint32_t* edges_out);

/* write_graph / read_graph (graph.cpp:152-192), host only (no context, no
 * device): dir/edges.bin = the raw 12-byte records, dir/graph_meta.json =
 * {"num_edges", "num_nodes", "num_relations"} in the reference's exact text
 * (nlohmann dump(2) + newline).  Read the metadata first to size edges_out.
 * I/O failures are LGD_RUNTIME_ERROR (std::runtime_error), as in the
 * reference. */
int lgd_write_graph(const char* dir, const uint32_t* edges, uint64_t num_edges, uint64_t num_nodes,
                    uint64_t num_relations);
int lgd_read_graph_meta(const char* dir, uint64_t* num_edges, uint64_t* num_nodes,
                        uint64_t* num_relations);
int lgd_read_graph(const char* dir, uint32_t* edges_out, uint64_t num_edges);
/* ingest (graph.cpp:39-118), host only: a TSV edge list of 3 (triples != 0)
 * or 2 decimal columns per line, '#' lines and blank lines skipped, parsed by
 * `threads` host threads (0 = all).  remap_ids: dense ids in first-appearance
 * order.  *edges_out: num_edges records allocated by the library, released
 * with lgd_free_edges.  Malformed input is LGD_RUNTIME_ERROR carrying the
 * reference's ParseError text with the line number. */
int lgd_ingest_tsv(const char* path, int triples, int remap_ids, int threads, uint32_t** edges_out,
                   uint64_t* num_edges, uint64_t* num_nodes, uint64_t* num_relations);
void lgd_free_edges(uint32_t* edges);

/* make_partition_plan (graph.cpp:120-150), computed on the device.  Outputs
 * may be NULL; bucket_offsets has n*n+1 entries, edge_order num_edges. */
int lgd_make_partition_plan(lgd_context* ctx, uint32_t n, uint64_t* bucket_offsets_out,
                            uint64_t* edge_order_out);
/* A caller-built PartitionPlan (graph.hpp:58-82). */
int lgd_set_partition_plan(lgd_context* ctx, uint32_t n, const uint64_t* bucket_offsets,
                           const uint64_t* edge_order);

/* ------------------------------------------------------------------- plan */

/* plan_loading_order + plan_iteration_order (ordering.hpp:49-54), host C++.
 * n >= 4.  Call with capacity 0 to learn num_states; arrays then hold
 * states[3*S], swaps[2*(S-1)] (evicted, loaded), bucket_order[2*n*n],
 * state_offsets[S+1], prefetch_points[S-1]. */
int lgd_plan_iteration_order(uint32_t n, uint64_t capacity, uint64_t* num_states, uint32_t* states,
                             uint32_t* swaps, uint32_t* bucket_order, uint64_t* state_offsets,
                             uint64_t* prefetch_points);
/* IterationPlan (ordering.hpp:40-47).  States may hold 0xffffffff in unused
 * slots (n <= 3 runs as one all-resident state). */
int lgd_set_iteration_plan(lgd_context* ctx, uint64_t num_states, const uint32_t* states,
                           const uint32_t* swaps, const uint32_t* bucket_order,
                           const uint64_t* state_offsets, const uint64_t* prefetch_points);

/* Multi-GPU partition-round schedule: rounds of disjoint
 * partition pairs; every bucket once, numbered in one global order that keys
 * its RNG stream; the pair is its negative pool; pair j of a round runs on
 * rank j % num_ranks.  Call with capacity 0 to learn count. */
typedef struct {
  uint32_t src_part, dst_part; /* bucket (i, j) */
  uint64_t g;                  /* RNG stream index (global position) */
  uint32_t pool[3];            /* negative pool partitions, 0xffffffff = unused */
  uint32_t round, pair;
} lgd_bucket_item;
int lgd_round_schedule(uint32_t n, uint64_t capacity, uint64_t* count, lgd_bucket_item* items,
                       uint32_t* num_rounds, uint32_t* pairs_per_round);

/* ------------------------------------------------------ embedding store */

/* EmbeddingStore::create initial values (store.cpp:59-86), on the device. */
int lgd_init_store(lgd_context* ctx, uint64_t seed);
int lgd_load_partition(lgd_context* ctx, uint32_t p, const float* e_s, uint64_t rows);
int lgd_store_partition(lgd_context* ctx, uint32_t p, float* e_s, uint64_t rows);
/* Asynchronous write-back of partition p into e_s (E then S, the layout above;
 * pinned memory from lgd_host_alloc makes it truly asynchronous): the copy sees
 * the tables as the work queued so far leaves them and overlaps whatever is
 * queued next that only reads them (lgd_evaluate). Every later call that writes
 * the tables orders itself after the pending copies; lgd_device_tables waits
 * for them on the host. e_s must stay valid until lgd_wait_stores returns.
 * Replaces the epoch-end partition writes of pipeline.cpp:173-193 /
 * store.cpp:27-57 (EmbeddingStore::write_partition). */
int lgd_store_partition_async(lgd_context* ctx, uint32_t p, float* e_s, uint64_t rows);
int lgd_wait_stores(lgd_context* ctx);
int lgd_set_relations(lgd_context* ctx, const float* e_s, uint64_t count);
int lgd_get_relations(lgd_context* ctx, float* e_s, uint64_t count);

/* --------------------------------------------------------------- training */

/* run_epoch real-train branch (pipeline.cpp:273-322) over the HBM-resident
 * table: per bucket of the plan, seeded shuffle, per-batch negatives, loss,
 * gradients and sparse Adagrad.  Synchronous. */
int lgd_train_epoch(lgd_context* ctx, uint32_t epoch, lgd_epoch_result* out);
/* Same, restricted to bucket_order positions [g_begin, g_end) (the plan
 * state of each position still selects the sampling pool).  Used to time a
 * bounded slice of an epoch. */
int lgd_train_buckets(lgd_context* ctx, uint32_t epoch, uint64_t g_begin, uint64_t g_end,
                      lgd_epoch_result* out);

/* The bucket at plan position g alone, cut after its first max_batches
 * batches (0 = all): the loop of pipeline.cpp:289-312 over a bounded prefix,
 * with the bucket's full shuffle and its stream consumed exactly as far as
 * the reference's.  Optional outputs (capacity = the batches run): per-batch
 * loss (batch_loss, train.cpp:217-278) and |GradientSet.nodes|.  Used to check
 * full-scale shapes against a CPU restatement in seconds. */
int lgd_train_bucket_prefix(lgd_context* ctx, uint32_t epoch, uint64_t g, uint64_t max_batches,
                            double* batch_losses, uint64_t* batch_nodes, lgd_epoch_result* out);

/* Same, streaming each bucket's edges from a host copy of the edge list in
 * bucket order (lgd_get_bucketed_edges; pinned memory from lgd_host_alloc for
 * full bandwidth): the H2D copy of bucket g+1 overlaps the training of g. */
int lgd_train_buckets_from_host(lgd_context* ctx, uint32_t epoch, uint64_t g_begin,
                                uint64_t g_end, const uint32_t* host_bucketed_edges,
                                lgd_epoch_result* out);
/* Registers (or, with NULL, clears) a host copy of the edge list in bucket
 * order: lgd_train_buckets, lgd_train_items and the lock-step rounds then copy
 * every bucket H2D from it (the end-to-end path) instead of reading the
 * device-resident copy.  The memory must stay valid while registered. */
int lgd_set_host_edges(lgd_context* ctx, const uint32_t* host_bucketed_edges);
/* The edge list in bucket order (edge_order applied), num_edges records. */
int lgd_get_bucketed_edges(lgd_context* ctx, uint32_t* edges_out);
/* Pinned host memory for the E||S blobs and edge lists. */
int lgd_host_alloc(uint64_t bytes, void** out);
int lgd_host_free(void* p);

/* Trains an explicit list of buckets (e.g. this rank's share of a round),
 * each with its own RNG stream index and negative pool. */
int lgd_train_items(lgd_context* ctx, uint32_t epoch, const lgd_bucket_item* items,
                    uint64_t count, lgd_epoch_result* out);
/* Lock-step rounds for typed models on several ranks: after each step the
 * caller sums the dense relation gradient [R x (dim+1)] (device, last column
 * = touched flag) across ranks, then applies it on every rank. */
int lgd_round_begin(lgd_context* ctx, uint32_t epoch, const lgd_bucket_item* items,
                    uint64_t count, uint64_t* my_batches);
int lgd_round_step(lgd_context* ctx, uint64_t step, double* rel_grad_device);
int lgd_round_apply_relations(lgd_context* ctx, const double* summed_device);
int lgd_round_end(lgd_context* ctx, lgd_epoch_result* out);
/* ---------------------------------- multi-GPU partition-round runner ----
 * One process per GPU.  Every rank builds the same graph, partition plan and
 * store (identical initial tables), then joins the runner; a round is
 * enqueued, its partition hand-offs issued, and its results collected:
 *   lgd_train_round = lgd_round_enqueue + lgd_round_handoff + lgd_round_collect.
 * Hand-offs are pulls over NVLink on a side stream (CUDA IPC mappings of the
 * peers' tables, inter-process ready events), overlapped with the buckets
 * that do not touch the moving partitions; typed models sum relation
 * gradients per lock-step batch with NCCL (loaded at run time).  DESIGN.md 6. */

/* A fresh NCCL unique id (128 bytes) on rank 0, to share with every rank. */
int lgd_comm_unique_id(void* id128);
/* Joins rank `rank` of `world` over NCCL communicators built from id128
 * (required for world > 1; at world = 1 a null id runs a local runner with
 * no NCCL, a non-null id still builds the one-rank communicators).  The
 * tables must exist and stay allocated (lgd_init_store / lgd_load_partition
 * first).  Collective over the ranks. */
int lgd_comm_init(lgd_context* ctx, const void* id128, uint32_t rank, uint32_t world);
/* Virtual ranks in one process: contexts[q] plays rank q (untyped models,
 * or world 1).  The caller enqueues every rank's round before any hand-off. */
int lgd_comm_init_local(lgd_context** contexts, uint32_t world);
int lgd_round_count(lgd_context* ctx, uint32_t* rounds);
int lgd_round_enqueue(lgd_context* ctx, uint32_t epoch, uint32_t round);
int lgd_round_handoff(lgd_context* ctx);
/* Waits for the round; handoff_ms = the hand-off copies' span on the side
 * stream, handoff_bytes = theta + state bytes pulled for the next round. */
int lgd_round_collect(lgd_context* ctx, lgd_epoch_result* out, double* handoff_ms,
                      uint64_t* handoff_bytes);
int lgd_train_round(lgd_context* ctx, uint32_t epoch, uint32_t round, lgd_epoch_result* out,
                    double* handoff_ms, uint64_t* handoff_bytes);

/* The runner's plan for one rank and round, host only (CPU tests, other
 * executors): ARRIVE partitions pulled from `peer` before their first bucket,
 * TRAIN buckets (item = index into lgd_round_schedule's list) in order,
 * DEPART partitions ready for their next holder (`peer`) after their last
 * bucket.
 * owner_in[p] (may be NULL = all -1): rank holding partition p's current rows
 * before the round, -1 = identical on every rank; owner_out: after it. */
#define LGD_ACT_ARRIVE 0
#define LGD_ACT_TRAIN 1
#define LGD_ACT_DEPART 2
typedef struct {
  uint32_t kind;
  uint32_t part;
  int32_t peer;
  uint64_t item;
} lgd_round_action;
int lgd_round_actions(uint32_t n, uint32_t world, uint32_t rank, uint32_t round,
                      const int32_t* owner_in, uint64_t capacity, uint64_t* count,
                      lgd_round_action* out, int32_t* owner_out);

/* The context's CUDA stream (cudaStream_t): every kernel of the context runs
 * on it, in order.  The call orders the stream after pending asynchronous
 * write-backs (lgd_store_partition_async), so work the caller then queues on
 * it may write the tables; writers on other streams, or through pointers
 * taken earlier, must call lgd_wait_stores first. */
int lgd_get_stream(lgd_context* ctx, void** cuda_stream);
/* on != 0: lgd_round_step and lgd_round_apply_relations return as soon as
 * their work is queued, without draining the stream.  The caller then orders
 * the relation all-reduce between them on that stream (e.g. NCCL with the
 * context's stream current), so a lock-step batch costs no host round trip.
 * Default 0: both return with the stream drained. */
int lgd_set_stream_ordered(lgd_context* ctx, int on);
/* Device pointers of the resident tables (partition hand-off between ranks). */
int lgd_device_tables(lgd_context* ctx, float** theta, float** state, float** rel_theta,
                      float** rel_state);

/* Operator level: batch_loss + batch_gradients + adagrad_step
 * (train.cpp:217-363) on one batch of host edges / negatives. */
int lgd_train_batch(lgd_context* ctx, const uint32_t* edges, uint64_t num_positives,
                    const uint32_t* negatives, int apply, double* loss, uint64_t* unique_nodes,
                    uint64_t* unique_rels);
/* batch_gradients (train.cpp:280-340) without the update: sorted unique ids
 * and FP64 gradient rows.  Output capacities: nodes num_positives*(k+2),
 * rels num_positives. */
int lgd_batch_gradients(lgd_context* ctx, const uint32_t* edges, uint64_t num_positives,
                        const uint32_t* negatives, double* loss, uint64_t* num_nodes,
                        uint32_t* node_ids, double* node_grads, uint64_t* num_rels,
                        uint32_t* rel_ids, double* rel_grads);

/* evaluate (train.cpp:375-412) over every partition: unfiltered ranking of
 * each test edge against num_candidates sampled destinations, pessimistic
 * ties, candidates from Rng(derive_seed(seed, "evay", t)). */
int lgd_evaluate(lgd_context* ctx, const uint32_t* test_edges, uint64_t count,
                 uint32_t num_candidates, uint32_t hits_k, uint64_t seed, double* mrr,
                 double* hits_at_k);

/* -------------------------------------------------- sampler primitives */

/* next_below(bound) x count from Rng(seed) after `skip` raw draws
 * (rng.hpp:42-48), on the device; consumed = raw draws used. */
int lgd_rng_below(int device, uint64_t seed, uint64_t skip, uint64_t bound, uint64_t count,
                  uint64_t* out, uint64_t* consumed);
/* sample_negatives (train.cpp:365-373) over resident ranges. */
int lgd_sample_negatives(int device, uint64_t seed, uint64_t skip, const uint64_t* first,
                         const uint64_t* counts, int num_ranges, uint32_t k,
                         uint64_t num_positives, uint32_t* out, uint64_t* consumed);
/* The Fisher-Yates permutation of pipeline.cpp:297-301 for a bucket of m
 * edges: perm[i] = original in-bucket position of the edge that ends at i. */
int lgd_shuffle_permutation(int device, uint64_t seed, uint64_t m, uint32_t* perm,
                            uint64_t* consumed);

/* ------------------------------------------------------------- profiling */
int lgd_set_profiling(lgd_context* ctx, int enabled);
int lgd_get_kernel_stats(lgd_context* ctx, int which, lgd_kernel_stats* out);
int lgd_reset_kernel_stats(lgd_context* ctx);
/* Kernel launches issued by the library since the last reset (all classes). */
uint64_t lgd_launch_count(lgd_context* ctx);
int lgd_synchronize(lgd_context* ctx);

#ifdef __cplusplus
}
#endif

#endif /* LEGEND_B200_H */
