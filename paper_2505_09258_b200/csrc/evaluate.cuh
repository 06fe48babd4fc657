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
  uint32_t* cand;       // tile x ncand scratch
  double* rr;           // T reciprocal ranks
  double* hit;          // T hits (0 / 1)
};

// test edges [t0, t0 + T): candidates then scores (rr, hit at index t)
void launch_evaluate_tile(const EvalArgs& a, uint64_t t0, uint64_t T, cudaStream_t st);
size_t eval_smem_bytes(uint32_t dim);

}  // namespace lgd
