// legend_reference_adapter.hpp -- the reference trainer's own entry points on
// the B200 path: drop-in replacements with the reference's exact signatures
// and types (proj/include/legend/*.hpp of the reference tree), implemented
// over the C ABI of include/legend_b200.h.
//
//   legend_b200::run_epoch  <- legend::run_epoch (pipeline.hpp:113-115), the
//                              real-train branch: the store's partitions and
//                              relations are uploaded to HBM, the plan's
//                              buckets trained on the device, every partition
//                              and the relations written back (the reference's
//                              end-of-epoch drain, pipeline.cpp:316-322).
//                              kCostOnly is delegated to the reference.
//   legend_b200::evaluate   <- legend::evaluate(model, store, ...)
//                              (train.hpp:139-140).
//
// Compile this file with the reference's include path (the maintainer's
// build); oracle/Makefile builds it that way for the adapter test
// (oracle/adapter_test.cpp: the reference's own test_pipeline.cpp:197-289
// check, with this run_epoch in place of the reference's).
#pragma once

#include <span>

#include "legend/graph.hpp"
#include "legend/ordering.hpp"
#include "legend/pipeline.hpp"
#include "legend/store.hpp"
#include "legend/train.hpp"

namespace legend_b200 {

// device = CUDA ordinal; errors rethrow the reference's exception classes
legend::EpochResult run_epoch(const legend::IterationPlan& plan, legend::EmbeddingStore& store,
                              const legend::Graph& graph, const legend::PartitionPlan& parts,
                              const legend::ScoreModel& model, const legend::CostModel& cost,
                              legend::EpochMode mode, const legend::TrainOptions& train,
                              bool prefetch = true, int device = 0);

legend::EvalResult evaluate(const legend::ScoreModel& model, const legend::EmbeddingStore& store,
                            std::span<const legend::Edge> test_edges,
                            const legend::EvalOptions& options, int device = 0);

}  // namespace legend_b200
