// evaluate.cuh -- launch interface of the device evaluator (evaluate.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace lgd {

struct EvalArgs {
  int kind;
  uint32_t dim;
  const float* theta;   // V x d (all partitions)
  const float* rel;     // R x d
  const uint32_t* edges;  // T x 3 test edges (device)
  uint64_t T;
  uint32_t ncand;
  uint32_t hits_k;
  uint64_t V;
  uint64_t seed;
  uint32_t* cand;       // T x ncand scratch
  double* rr;           // T scratch
  double* hit;          // T scratch
  double* out;          // [mrr, hits]
};

void launch_evaluate(const EvalArgs& a, cudaStream_t st);

}  // namespace lgd
