// gram_shard.h — plan and kernels of the rank-count-independent sharded Gram
// (gram_shard.cu); internal, the C-ABI view is cqr_gram_shard in include/cqr.h.
#pragma once

#include <cuda_runtime.h>

#include <utility>
#include <vector>

#include "../../include/cqr.h"

namespace cqr {

struct DevStatus;

// Rank b's part of the global-leaf Gram of an m-row matrix split as parexec.cpp:9-18.
struct ShardGram {
  long long m = 0, r0 = 0, r1 = 0, leaves = 0;
  bool head = false;  // rows [r0, head_end) continue a leaf begun on rank b-1
  bool tail = false;  // rows [tail_start, r1) begin a leaf finished on rank b+1
  bool span = false;  // head and tail are the same leaf: continue and forward
  long long head_end = 0, tail_start = 0;
  long long full0 = 0, full1 = 0;  // rows of the leaves complete on this rank
  long long lo = 0, hi = 0;        // owned leaves (last row on this rank)
  std::vector<long long> node_start, node_count;  // tree nodes covering [lo, hi)
};

long long shard_offset(long long m, int p, int b);
std::vector<std::pair<long long, long long>> tree_nodes(long long L, long long lo, long long hi);
ShardGram shard_gram_plan(long long m, int p, int b);
// postfix program over slots b*K + k (-1 = add); K = max nodes per rank
std::vector<int> tree_program(long long m, int p, int* slots_per_rank);

cudaError_t launch_gram_chain(const double* x, long long ldx, long long rows, int n, int np, const double* init,
                              double* out, int check, DevStatus* st, cudaStream_t s);
// host tables for launch_gram_nodes; returns the group count
size_t gram_nodes_tables(const ShardGram& g, std::vector<int>& ta, std::vector<int>& tb);
cudaError_t launch_gram_nodes(const double* partial, int np, int n, const int* ta_dev, int groups, const int* tb_dev,
                              int nodes, double* gsum, double* slots, const DevStatus* st, cudaStream_t s);
cudaError_t launch_gram_program(const double* slots, int n, const int* prog_dev, int len, double* g,
                                const DevStatus* st, cudaStream_t s);

}  // namespace cqr
