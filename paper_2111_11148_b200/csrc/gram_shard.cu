// gram_shard.cu — the Gram of a row-block-partitioned matrix, bitwise equal to
// the one-GPU Gram for any number of ranks (SURVEY 8e "determinism option").
//
// The reference's parallel Gram splits the GLOBAL 1024-row leaves over its
// workers and combines them with one fixed pairwise tree, so the result does not
// depend on the worker count (engine.cpp:24-39, kernels.hpp:17-71;
// test_parexec.cpp:47-56 asserts bitwise identity across p). Row blocks
// [ceil(b m/p), ceil((b+1) m/p)) (parexec.cpp:9-18) do not fall on leaf
// boundaries, so per rank b:
//  * a leaf that begins on an earlier rank continues here: its fma chain (rows
//    ascending from +0, the leaf order) arrives as a partial n x n value from
//    rank b-1 and is continued over this rank's first rows (the "head");
//  * the leaf this rank's rows end inside begins here: its chain over the last
//    rows (the "tail") goes to rank b+1; a rank inside a single leaf continues
//    and forwards it ("span");
//  * the leaves whose last row lies on this rank ("owned") are combined into the
//    largest nodes of the global pairwise tree that fit inside the owned range;
//  * every rank all-gathers the nodes and evaluates the remaining top of the
//    tree with one postfix program, in the tree's own operand order.
// A continued chain is the same sequence of fma as the one-GPU DMMA leaf, the
// nodes are subtrees of the same tree, so G is bit-identical to p = 1.

#include <algorithm>
#include <vector>

#include "common.cuh"
#include "gram_shard.h"

namespace cqr {

namespace {
constexpr long long kLeaf = 1024;  // kernels.hpp:20

long long ceil_div(long long a, long long b) { return (a + b - 1) / b; }
}  // namespace

long long shard_offset(long long m, int p, int b) {  // parexec.cpp:13-15
  if (b <= 0) return 0;
  if (b >= p) return m;
  return ((long long)b * m + p - 1) / p;
}

std::vector<std::pair<long long, long long>> tree_nodes(long long L, long long lo, long long hi) {
  // node (l, i) of the pairwise tree over L slots covers [i 2^l, min((i+1) 2^l, L))
  // (kernels.hpp:42-57: pairs (0+1),(2+3),..., an odd last slot carried up)
  std::vector<std::pair<long long, long long>> out;
  long long s = lo;
  while (s < hi) {
    long long size = 1;
    while (s + size < L && s % (2 * size) == 0 && std::min(s + 2 * size, L) <= hi) size *= 2;
    const long long e = std::min(s + size, L);
    out.emplace_back(s, e - s);
    s = e;
  }
  return out;
}

ShardGram shard_gram_plan(long long m, int p, int b) {
  ShardGram g;
  g.m = m;
  g.r0 = shard_offset(m, p, b);
  g.r1 = shard_offset(m, p, b + 1);
  g.leaves = ceil_div(m, kLeaf);
  if (g.r1 <= g.r0) {  // empty block (p > m): owns nothing, forwards nothing
    g.full0 = g.full1 = g.r0;
    g.lo = g.hi = g.r0 / kLeaf;
    return g;
  }
  const long long hl = g.r0 / kLeaf, tl = (g.r1 - 1) / kLeaf;
  g.head = g.r0 % kLeaf != 0;
  g.tail = g.r1 % kLeaf != 0 && g.r1 < m;
  g.span = g.head && g.tail && hl == tl;
  g.head_end = std::min((hl + 1) * kLeaf, g.r1);
  g.tail_start = std::max(tl * kLeaf, g.r0);
  const long long fa = g.head ? hl + 1 : hl, fb = g.tail ? tl : tl + 1;
  if (g.span || fb <= fa) {
    g.full0 = g.full1 = g.span ? g.r0 : g.head_end;
  } else {
    g.full0 = fa * kLeaf;
    g.full1 = std::min(fb * kLeaf, m);
  }
  g.lo = hl;
  g.hi = g.span ? hl : fb;
  for (auto& nd : tree_nodes(g.leaves, g.lo, g.hi)) {
    g.node_start.push_back(nd.first);
    g.node_count.push_back(nd.second);
  }
  return g;
}

// Postfix evaluation of node(l, i): a slot when the node is one of the
// gathered ones, else left + right (right absent: carried), as kernels.hpp:42-57.
static void emit(long long L, int l, long long i, const std::vector<std::vector<std::pair<long long, long long>>>& nodes,
                 int K, std::vector<int>& prog) {
  const long long s = i << l, e = std::min((i + 1) << l, L);
  for (size_t b = 0; b < nodes.size(); ++b)
    for (size_t k = 0; k < nodes[b].size(); ++k)
      if (nodes[b][k].first == s && nodes[b][k].first + nodes[b][k].second == e) {
        prog.push_back((int)(b * K + k));
        return;
      }
  emit(L, l - 1, 2 * i, nodes, K, prog);
  if (((2 * i + 1) << (l - 1)) < L) {
    emit(L, l - 1, 2 * i + 1, nodes, K, prog);
    prog.push_back(-1);
  }
}

std::vector<int> tree_program(long long m, int p, int* slots_per_rank) {
  const long long L = ceil_div(m, kLeaf);
  std::vector<std::vector<std::pair<long long, long long>>> nodes(p);
  int K = 1;
  for (int b = 0; b < p; ++b) {
    ShardGram g = shard_gram_plan(m, p, b);
    for (size_t k = 0; k < g.node_start.size(); ++k) nodes[b].emplace_back(g.node_start[k], g.node_count[k]);
    K = std::max(K, (int)nodes[b].size());
  }
  int top = 0;
  while ((1LL << top) < L) ++top;
  std::vector<int> prog;
  if (L > 0) emit(L, top, 0, nodes, K, prog);
  if (slots_per_rank) *slots_per_rank = K;
  return prog;
}

// ---- kernels -------------------------------------------------------------------------
namespace {

// out(i, j) = fma chain over `rows` rows from init(i, j) (or +0), j >= i; the
// continuation of a leaf chain across a block boundary.
__global__ void gram_chain_kernel(const double* __restrict__ x, long long ldx, int rows, int n, int np,
                                  const double* __restrict__ init, double* __restrict__ out, int check,
                                  DevStatus* st) {
  if (failed(st)) return;
  const int i = blockIdx.y;
  const int j = i + blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  double acc = init ? init[(long long)i * np + j] : 0.0;
  bool bad = false;
  int r = 0;
  for (; r + 8 <= rows; r += 8) {
    double a[8], c[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      a[u] = __ldg(x + (long long)(r + u) * ldx + i);
      c[u] = __ldg(x + (long long)(r + u) * ldx + j);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      bad |= nonfinite(c[u]);
      acc = fma(a[u], c[u], acc);
    }
  }
  for (; r < rows; ++r) {
    const double a = __ldg(x + (long long)r * ldx + i), c = __ldg(x + (long long)r * ldx + j);
    bad |= nonfinite(c);
    acc = fma(a, c, acc);
  }
  if (check && i == 0 && bad) set_status_invalid(st);
  out[(long long)i * np + j] = acc;
}

__device__ __forceinline__ void push_merge(double* stk, int& top, double v, unsigned count_after) {
  while ((count_after & 1u) == 0u) {
    v = stk[--top] + v;
    count_after >>= 1;
  }
  stk[top++] = v;
}

// Level A of the streaming tree (gram.cu) per group entry {leaf0, count <= 16}.
__global__ void gram_nodes_a_kernel(const double* __restrict__ partial, int np, int n, const int* __restrict__ tab,
                                    double* __restrict__ gsum, const DevStatus* st) {
  if (failed(st)) return;
  const int i = blockIdx.y;
  const int xb = (n + 127) / 128;
  const int grp = blockIdx.x / xb;
  const int j = i + (blockIdx.x - grp * xb) * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const long long stride = (long long)np * np;
  const int l0 = tab[2 * grp], cnt = tab[2 * grp + 1];
  const double* p = partial + (long long)i * np + j;
  double v[16];
#pragma unroll
  for (int u = 0; u < 16; ++u) v[u] = u < cnt ? __ldg(p + (long long)(l0 + u) * stride) : 0.0;
  double stk[8];
  int top = 0;
#pragma unroll
  for (int u = 0; u < 16; ++u)
    if (u < cnt) push_merge(stk, top, v[u], (unsigned)(u + 1));
  double acc = stk[top - 1];
  for (int k = top - 2; k >= 0; --k) acc = stk[k] + acc;
  gsum[(long long)grp * stride + (long long)i * np + j] = acc;
}

// Level B per node {g0, full, has_partial} -> slot (n x n, upper).
__global__ void gram_nodes_b_kernel(const double* __restrict__ gsum, int np, int n, const int* __restrict__ tab,
                                    double* __restrict__ slots, const DevStatus* st) {
  if (failed(st)) return;
  const int node = blockIdx.z;
  const int i = blockIdx.y;
  const int j = i + blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const int g0 = tab[3 * node], full = tab[3 * node + 1], part = tab[3 * node + 2];
  const long long stride = (long long)np * np;
  const double* p = gsum + (long long)g0 * stride + (long long)i * np + j;
  double stk[40];
  int top = 0;
  for (int k = 0; k < full; ++k) push_merge(stk, top, __ldg(p + (long long)k * stride), (unsigned)(k + 1));
  if (part) stk[top++] = __ldg(p + (long long)full * stride);
  double acc = stk[top - 1];
  for (int k = top - 2; k >= 0; --k) acc = stk[k] + acc;
  slots[(long long)node * n * n + (long long)i * n + j] = acc;
}

// The top of the tree: postfix program over the gathered node slots.
__global__ void gram_program_kernel(const double* __restrict__ slots, int n, const int* __restrict__ prog, int len,
                                    double* __restrict__ g, const DevStatus* st) {
  if (failed(st)) return;
  const int i = blockIdx.y;
  const int j = i + blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  double stk[48];
  int top = 0;
  for (int t = 0; t < len; ++t) {
    const int op = __ldg(prog + t);
    if (op >= 0) {
      stk[top++] = __ldg(slots + (long long)op * n * n + (long long)i * n + j);
    } else {
      const double r = stk[--top];
      stk[top - 1] = stk[top - 1] + r;
    }
  }
  g[(long long)i * n + j] = stk[0];
  g[(long long)j * n + i] = stk[0];
}

}  // namespace

cudaError_t launch_gram_chain(const double* x, long long ldx, long long rows, int n, int np, const double* init,
                              double* out, int check, DevStatus* st, cudaStream_t s) {
  dim3 grid((unsigned)((n + 127) / 128), (unsigned)n);
  gram_chain_kernel<<<grid, 128, 0, s>>>(x, ldx, (int)rows, n, np, init, out, check, st);
  return cudaGetLastError();
}

size_t gram_nodes_tables(const ShardGram& g, std::vector<int>& ta, std::vector<int>& tb) {
  ta.clear();
  tb.clear();
  for (size_t k = 0; k < g.node_start.size(); ++k) {
    const int l0 = (int)(g.node_start[k] - g.lo), cnt = (int)g.node_count[k];
    const int g0 = (int)(ta.size() / 2);
    for (int u = 0; u < cnt; u += 16) {
      ta.push_back(l0 + u);
      ta.push_back(std::min(16, cnt - u));
    }
    tb.push_back(g0);
    tb.push_back(cnt / 16);
    tb.push_back(cnt % 16 != 0 ? 1 : 0);
  }
  return ta.size() / 2;
}

cudaError_t launch_gram_nodes(const double* partial, int np, int n, const int* ta_dev, int groups, const int* tb_dev,
                              int nodes, double* gsum, double* slots, const DevStatus* st, cudaStream_t s) {
  if (nodes <= 0) return cudaSuccess;
  dim3 ga((unsigned)(((n + 127) / 128) * groups), (unsigned)n);
  gram_nodes_a_kernel<<<ga, 128, 0, s>>>(partial, np, n, ta_dev, gsum, st);
  dim3 gb((unsigned)((n + 127) / 128), (unsigned)n, (unsigned)nodes);
  gram_nodes_b_kernel<<<gb, 128, 0, s>>>(gsum, np, n, tb_dev, slots, st);
  return cudaGetLastError();
}

cudaError_t launch_gram_program(const double* slots, int n, const int* prog_dev, int len, double* g,
                                const DevStatus* st, cudaStream_t s) {
  dim3 grid((unsigned)((n + 127) / 128), (unsigned)n);
  gram_program_kernel<<<grid, 128, 0, s>>>(slots, n, prog_dev, len, g, st);
  return cudaGetLastError();
}

}  // namespace cqr

// ---- C-ABI: the plan, for the host-side tests ----------------------------------------
extern "C" int cqr_gram_shard_plan(int64_t m, int p, int b, cqr_gram_shard* out) {
  if (!out || m < 1 || p < 1 || b < 0 || b >= p) return CQR_INVALID_ARGUMENT;
  const cqr::ShardGram g = cqr::shard_gram_plan(m, p, b);
  if (g.node_start.size() > 64) return CQR_INVALID_ARGUMENT;
  out->row0 = g.r0;
  out->row1 = g.r1;
  out->head = g.head;
  out->tail = g.tail;
  out->span = g.span;
  out->head_end = g.head_end;
  out->tail_start = g.tail_start;
  out->full0 = g.full0;
  out->full1 = g.full1;
  out->lo = g.lo;
  out->hi = g.hi;
  out->nodes = (int)g.node_start.size();
  for (int k = 0; k < out->nodes; ++k) {
    out->node_start[k] = g.node_start[k];
    out->node_count[k] = g.node_count[k];
  }
  return CQR_OK;
}

extern "C" int cqr_gram_tree_program(int64_t m, int p, int* prog, int cap, int* slots_per_rank) {
  if (m < 1 || p < 1) return -1;
  const std::vector<int> v = cqr::tree_program(m, p, slots_per_rank);
  if ((int)v.size() > cap || !prog) return -(int)v.size();
  std::copy(v.begin(), v.end(), prog);
  return (int)v.size();
}
