// engine.cu — host orchestration and the C-ABI (include/cqr.h).
//
// Restates the reference's execution engine (proj/src/engine.cpp:78-305) for
// one process per GPU: the tall matrix stays in HBM, every stage is a
// stream-ordered launch of the sm_100a kernels, failures are a device status
// word (so an attempt needs ONE host synchronisation, at its end), the retry
// loop mirrors engine.cpp:137-209 (sizes llround(l*growth^a), seeds
// derive(seed, a)), and the reference's simulated workers (engine.cpp:12-39,
// parexec.cpp) become row-block shards on separate GPUs whose s x n sketch and
// n x n Gram partials are summed with NCCL all-reduce over NVLink.

#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <string>
#include <unordered_set>
#include <vector>
#include <mutex>
#include <set>

#include "../../include/cqr.h"
#include "common.cuh"
#include "gram_shard.h"
#include "kernels.h"

using cqr::DevStatus;

namespace {

constexpr double kU = 2.220446049250313e-16;  // types.hpp:31

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
};

struct StageEv {
  int stage;
  cudaEvent_t a, b;
};

}  // namespace

struct cqr_ctx {
  int device = 0;
  int num_sms = 148;
  cudaStream_t stream = nullptr;
  std::string err;
  DevBuf bufs[32];
  DevStatus* status = nullptr;   // device
  DevStatus* status_h = nullptr;  // pinned host
  double* scal_h = nullptr;       // pinned host scalars
  double* r_pin = nullptr;        // pinned host R staging (the early R copy)
  size_t r_pin_n = 0;
  ncclComm_t comm = nullptr;
  cqr_host_comm hcomm{};     // caller-owned host transport (cqr_attach_host_comm)
  bool has_hcomm = false;
  void* stage_h = nullptr;   // pinned staging for the host transport
  size_t stage_bytes = 0;
  int rank = 0, world = 1;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
  std::vector<StageEv> stage_evs;
  long long launches = 0;
  int tiles_key[2] = {-1, -1};  // gram tile tables currently on the device
  int local_only = 0;  // temporarily treat an attached communicator as absent (replicated small work)
  cudaStream_t cstream = nullptr;  // copy stream of the host-buffer pipeline
  std::vector<cudaEvent_t> pipe_ev;
  cudaEvent_t order_ev = nullptr;  // cqr_order_after
};

namespace {

enum BufId {
  B_A1 = 0, B_SKPART, B_GPART, B_GTILES, B_G, B_RT, B_RH, B_R, B_RTMP, B_SGN, B_PACK1, B_PACK2, B_WORK,
  B_IDX, B_HA, B_HQ, B_SCAL, B_DIAG, B_X, B_SYN, B_SYNV, B_SHPART, B_SHSLOT, B_SHALL, B_SHTAB, B_SHHT, B_HHW,
  B_HHPART, B_HHRED, B_HHTAU, B_SKEXP
};

struct Fail {
  int code;
  long long index;
  std::string msg;
};

void* buf(cqr_ctx* c, int id, size_t bytes) {
  DevBuf& b = c->bufs[id];
  if (bytes == 0) bytes = 8;
  if (b.bytes < bytes) {
    if (b.p) cudaFree(b.p);
    b.p = nullptr;
    b.bytes = 0;
    if (cudaMalloc(&b.p, bytes) != cudaSuccess) {
      cudaGetLastError();
      throw Fail{CQR_OUT_OF_MEMORY, -1, "cudaMalloc of " + std::to_string(bytes) + " bytes failed"};
    }
    b.bytes = bytes;
  }
  return b.p;
}

template <typename T>
T* dbuf(cqr_ctx* c, int id, size_t count) {
  return static_cast<T*>(buf(c, id, count * sizeof(T)));
}

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw Fail{CQR_CUDA_ERROR, -1, std::string(what) + ": " + cudaGetErrorString(e)};
}

void ckn(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw Fail{CQR_NCCL_ERROR, -1, std::string(what) + ": " + ncclGetErrorString(r)};
}

// ---- the rank exchanges: NCCL on the library's stream, or the caller's host transport ----
bool attached(const cqr_ctx* c) { return c->comm != nullptr || c->has_hcomm; }
bool multi(const cqr_ctx* c) { return attached(c) && !c->local_only; }

void* host_stage(cqr_ctx* c, size_t bytes) {
  if (c->stage_bytes < bytes) {
    if (c->stage_h) cudaFreeHost(c->stage_h);
    c->stage_h = nullptr;
    c->stage_bytes = 0;
    ck(cudaMallocHost(&c->stage_h, bytes), "cudaMallocHost (comm staging)");
    c->stage_bytes = bytes;
  }
  return c->stage_h;
}

void hcheck(int rc, const char* what) {
  if (rc != 0) throw Fail{CQR_NCCL_ERROR, -1, std::string("host transport: ") + what + " failed"};
}

// in-place all-reduce of a device buffer: doubles summed, or int32 max
void coll_allreduce(cqr_ctx* c, void* p, size_t count, int dtype) {
  if (!multi(c)) return;
  const size_t esz = dtype == CQR_COMM_F64_SUM ? sizeof(double) : sizeof(int32_t);
  if (c->comm) {
    ckn(ncclAllReduce(p, p, count, dtype == CQR_COMM_F64_SUM ? ncclDouble : ncclInt32,
                      dtype == CQR_COMM_F64_SUM ? ncclSum : ncclMax, c->comm, c->stream),
        "ncclAllReduce");
    return;
  }
  void* h = host_stage(c, count * esz);
  ck(cudaMemcpyAsync(h, p, count * esz, cudaMemcpyDeviceToHost, c->stream), "comm D2H");
  ck(cudaStreamSynchronize(c->stream), "comm sync");
  hcheck(c->hcomm.allreduce(c->hcomm.user, h, (int64_t)count, dtype), "allreduce");
  ck(cudaMemcpyAsync(p, h, count * esz, cudaMemcpyHostToDevice, c->stream), "comm H2D");
  ck(cudaStreamSynchronize(c->stream), "comm sync");
}

// send `count` doubles to dst and receive `count` from src, concurrently (either side may be absent: -1)
void coll_sendrecv(cqr_ctx* c, const double* send, int dst, double* recv, int src, size_t count) {
  if (dst < 0 && src < 0) return;
  if (c->comm) {
    ckn(ncclGroupStart(), "group");
    if (dst >= 0) ckn(ncclSend(send, count, ncclDouble, dst, c->comm, c->stream), "ncclSend");
    if (src >= 0) ckn(ncclRecv(recv, count, ncclDouble, src, c->comm, c->stream), "ncclRecv");
    ckn(ncclGroupEnd(), "group");
    return;
  }
  double* h = static_cast<double*>(host_stage(c, 2 * count * sizeof(double)));
  if (dst >= 0) {
    ck(cudaMemcpyAsync(h, send, count * sizeof(double), cudaMemcpyDeviceToHost, c->stream), "comm D2H");
    ck(cudaStreamSynchronize(c->stream), "comm sync");
  }
  hcheck(c->hcomm.sendrecv(c->hcomm.user, dst >= 0 ? h : nullptr, dst, src >= 0 ? h + count : nullptr, src,
                           (int64_t)count),
         "sendrecv");
  if (src >= 0) {
    ck(cudaMemcpyAsync(recv, h + count, count * sizeof(double), cudaMemcpyHostToDevice, c->stream), "comm H2D");
    ck(cudaStreamSynchronize(c->stream), "comm sync");
  }
}

// every rank's `count` doubles, in rank order
void coll_allgather(cqr_ctx* c, const double* send, double* recv, size_t count) {
  if (c->comm) {
    ckn(ncclAllGather(send, recv, count, ncclDouble, c->comm, c->stream), "ncclAllGather");
    return;
  }
  double* h = static_cast<double*>(host_stage(c, (size_t)(c->world + 1) * count * sizeof(double)));
  ck(cudaMemcpyAsync(h, send, count * sizeof(double), cudaMemcpyDeviceToHost, c->stream), "comm D2H");
  ck(cudaStreamSynchronize(c->stream), "comm sync");
  hcheck(c->hcomm.allgather(c->hcomm.user, h, h + count, (int64_t)count), "allgather");
  ck(cudaMemcpyAsync(recv, h + count, (size_t)c->world * count * sizeof(double), cudaMemcpyHostToDevice, c->stream),
     "comm H2D");
  ck(cudaStreamSynchronize(c->stream), "comm sync");
}

#define LAUNCH(c, expr)          \
  do {                           \
    ck((expr), #expr);           \
    ++(c)->launches;             \
  } while (0)

// Copies that the host waits for, ordered on the library's stream. (A plain cudaMemcpy runs on the
// legacy stream, which the non-blocking library stream is not ordered against, and a pageable H2D
// cudaMemcpy may return before its DMA lands -- a kernel queued next on the library stream could
// read the old bytes.)
void copy_sync(cqr_ctx* c, void* dst, const void* src, size_t bytes, cudaMemcpyKind kind, const char* what);

void require(bool cond, const char* msg) {
  if (!cond) throw Fail{CQR_INVALID_ARGUMENT, -1, msg};
}

bool vec_ok(const void* p, long long ld, int n) {
  return (ld % 2 == 0) && (n % 2 == 0) && ((reinterpret_cast<uintptr_t>(p) & 15) == 0);
}

// ---- rng on the host (rng.hpp:22-42) -----------------------------------------------
uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
uint64_t derive(uint64_t seed, uint64_t salt) { return mix64(seed ^ mix64(salt + 0x51ED270B8A5EC473ull)); }
double unit_at(uint64_t seed, uint64_t k) {
  return static_cast<double>(mix64(seed + (k + 1) * 0x9E3779B97F4A7C15ull) >> 11) * 0x1.0p-53;
}

long long resolved_size(const cqr_sketch_cfg& cfg, long long m, long long n) {  // sketch.cpp:20-23
  long long l = cfg.size > 0 ? cfg.size : static_cast<long long>(std::ceil(cfg.rate * static_cast<double>(n)));
  return std::clamp(l, n, m);
}

cqr_sketch_cfg default_cfg() {
  cqr_sketch_cfg c{};
  c.strategy = CQR_UNIFORM;
  c.rate = 2.0;
  c.max_retries = 2;
  c.retry_growth = 2.0;
  return c;
}

cqr_options default_opts() {
  cqr_options o{};
  o.shift_kind = CQR_SHIFT_THEORY;
  o.workers = 1;
  return o;
}

// ---- stage timing (StageClock, engine.hpp:14-41, with CUDA events) -----------------
cudaEvent_t next_event(cqr_ctx* c) {
  if (c->ev_used == c->ev_pool.size()) {
    cudaEvent_t e;
    ck(cudaEventCreate(&e), "cudaEventCreate");
    c->ev_pool.push_back(e);
  }
  return c->ev_pool[c->ev_used++];
}

struct StageScope {
  cqr_ctx* c;
  StageEv ev;
  cudaStream_t strm;
  StageScope(cqr_ctx* c_, int stage, cudaStream_t on = nullptr) : c(c_), strm(on ? on : c_->stream) {
    ev.stage = stage;
    ev.a = next_event(c);
    ev.b = next_event(c);
    ck(cudaEventRecord(ev.a, strm), "cudaEventRecord");
  }
  ~StageScope() {
    cudaEventRecord(ev.b, strm);
    c->stage_evs.push_back(ev);
  }
};

struct Report {
  std::vector<cqr_stage_info> stages;
  long long sketch_rows = 0;
};

void push_stage(Report& r, int stage, int retries = 0, bool has_shift = false, double shift = 0.0,
                bool has_cond = false, double cond = 0.0) {
  cqr_stage_info s{};
  s.stage = stage;
  s.retries = retries;
  s.has_shift = has_shift ? 1 : 0;
  s.shift = shift;
  s.has_cond_x = has_cond ? 1 : 0;
  s.cond_x = cond;
  r.stages.push_back(s);
}

// ---- engine ---------------------------------------------------------------------------
struct Job {
  cqr_ctx* c;
  int method;
  const double* a;  // device, this rank's shard
  long long m_local, m_global, row0;
  int n;
  long long lda;
  double* q;  // device
  long long ldq;
  cqr_sketch_cfg cfg;
  cqr_options opts;
  cqr_precond_fn precond = nullptr;
  void* user = nullptr;
  int check_first = 0;  // fuse the non-finite check into the first tall kernel
  // host-buffer pipeline (cqr_factor): A arrives in row chunks on the copy
  // stream, the first tall pass consumes them as they land, and the final solve
  // streams Q back chunk by chunk
  const double* a_host = nullptr;
  long long lda_host = 0;
  double* q_host = nullptr;
  long long ldq_host = 0;
  std::vector<long long> bounds;  // chunk row boundaries, bounds.front() = 0, bounds.back() = m
  int waited = 0;                 // H2D chunks the compute stream already waits on
  int det = 0;  // every rank holds its standard row block: the rank-count-independent Gram (gram_shard.cu)
  bool want_r = false;     // the caller takes R back to the host
  bool r_copied = false;   // R already on its way to c->r_pin on the copy stream (overlapping the last solve)
};

bool pipelined(const Job& j) { return j.a_host != nullptr; }

// make the compute stream wait for every H2D chunk that starts below row `rows_end`
void wait_rows(Job& j, long long rows_end) {
  cqr_ctx* c = j.c;
  while (pipelined(j) && j.waited + 1 < (int)j.bounds.size() && j.bounds[j.waited] < rows_end) {
    ck(cudaStreamWaitEvent(c->stream, c->pipe_ev[j.waited], 0), "wait H2D");
    ++j.waited;
  }
}
void wait_all(Job& j) { wait_rows(j, std::numeric_limits<long long>::max()); }

void allreduce(cqr_ctx* c, double* p, size_t count) { coll_allreduce(c, p, count, CQR_COMM_F64_SUM); }

// slot 0: the main plan's table; slot 1: the last-wave table of the split launch (gram_dev)
const int32_t* gram_tiles_dev(cqr_ctx* c, const cqr::GramPlan& p, int slot = 0) {
  int32_t* tiles = dbuf<int32_t>(c, B_GTILES, 8192) + 4096 * slot;
  const int key = p.np * 1000000 + p.wpc * 10000 + p.parts * 100 + p.maxt + (p.tma ? 5000 : 0);
  if (c->tiles_key[slot] != key) {  // the table depends on (np, parts, maxt) only: upload once
    std::vector<int32_t> ht(p.tiles_bytes / sizeof(int32_t));
    cqr::gram_tiles(p, ht.data());
    // ordered on the library's stream (kernels already queued may still read the old table: the
    // copy waits for them, and the kernels queued after it see the new one)
    ck(cudaMemcpyAsync(tiles, ht.data(), p.tiles_bytes, cudaMemcpyHostToDevice, c->stream), "tiles H2D");
    ck(cudaStreamSynchronize(c->stream), "sync");  // ht is a stack buffer
    c->tiles_key[slot] = key;
  }
  return tiles;
}

// ---- the Gaussian sketch: the integer tensor-core kernel (sketch_i8.cu) when A is TMA-addressable,
// else the DMMA kernels (sketch.cu) ------------------------------------------------------------
struct SketchRun {
  cqr::SketchPlan p;
  double* part = nullptr;
};

SketchRun sketch_setup(cqr_ctx* c, const double* a, long long lda, long long m_local, long long m_global,
                       long long row0, int n, int l, int splits) {
  SketchRun r;
  const bool i8 = cqr::sketch_i8_ok(a, lda, m_global, row0, n);
  r.p = cqr::sketch_plan(m_local, n, l, c->num_sms, cqr::sketch_ws_ok(a, lda, m_global, row0, n), splits);
  if (i8) cqr::sketch_i8_plan(r.p, m_local, n, l, c->num_sms, splits);
  r.part = dbuf<double>(c, B_SKPART, std::max<size_t>(r.p.partial_doubles, 1));
  return r;
}

cudaError_t sketch_launch(cqr_ctx* c, const SketchRun& r, const double* a, long long lda, long long m_global,
                          long long row0, uint64_t seed, int vec, int check, int y0 = 0, int y1 = -1) {
  if (r.p.i8) {
    return cqr::launch_sketch_i8(r.p, a, lda, m_global, row0, seed, r.part, c->status, c->stream, y0, y1);
  }
  return cqr::launch_sketch_gaussian(r.p, a, lda, m_global, row0, seed, r.part, vec, check, c->status, c->stream, y0,
                                     y1);
}

// ---- rank-count-independent sharded Gram (gram_shard.cu) ------------------------------
struct ShardWs {
  double *part, *gsum, *slots, *all, *ht;  // ht: 3 np x np chain buffers (head in, tail out, spare)
  int* tab;
  int np, K;
};

ShardWs shard_ws(cqr_ctx* c, long long m, int p, int n, int K) {
  ShardWs w;
  w.np = cqr::gram_plan(1024, n).np;
  w.K = K;
  long long owned = 0;
  for (int b = 0; b < p; ++b) {
    const cqr::ShardGram g = cqr::shard_gram_plan(m, p, b);
    owned = std::max(owned, g.hi - g.lo);
  }
  const size_t np2 = (size_t)w.np * w.np;
  const size_t groups = (size_t)(owned + 15) / 16 + (size_t)K;
  w.part = dbuf<double>(c, B_SHPART, (size_t)(owned + 1) * np2 + groups * np2);
  w.gsum = w.part + (size_t)(owned + 1) * np2;
  w.slots = dbuf<double>(c, B_SHSLOT, (size_t)K * n * n);
  w.all = dbuf<double>(c, B_SHALL, (size_t)p * K * n * n);
  w.ht = dbuf<double>(c, B_SHHT, 3 * np2);
  w.tab = dbuf<int>(c, B_SHTAB, 65536);
  return w;
}

// tail rows -> out (a chain from +0), unless the rank lies inside one leaf
void shard_tail(cqr_ctx* c, const cqr::ShardGram& sg, const double* x, long long ldx, int n, int np, double* out,
                int check) {
  if (sg.tail && !sg.span)
    LAUNCH(c, cqr::launch_gram_chain(x + (sg.tail_start - sg.r0) * ldx, ldx, sg.r1 - sg.tail_start, n, np, nullptr,
                                     out, check, c->status, c->stream));
}

// the head chain (continued from head_in), the complete leaves, and the owned nodes -> slots
void shard_body(cqr_ctx* c, const cqr::ShardGram& sg, const double* x, long long ldx, int n, const ShardWs& w,
                const double* head_in, double* span_out, double* slots, int check) {
  const size_t np2 = (size_t)w.np * w.np;
  if (sg.span) {
    LAUNCH(c, cqr::launch_gram_chain(x, ldx, sg.r1 - sg.r0, n, w.np, head_in, span_out, check, c->status,
                                     c->stream));
    return;
  }
  if (sg.head)
    LAUNCH(c, cqr::launch_gram_chain(x, ldx, sg.head_end - sg.r0, n, w.np, head_in, w.part, check, c->status,
                                     c->stream));
  if (sg.full1 > sg.full0) {
    const double* xf = x + (sg.full0 - sg.r0) * ldx;
    const long long mf = sg.full1 - sg.full0;
    cqr::GramPlan p = cqr::gram_plan(mf, n, cqr::gram_tma_ok(xf, ldx, mf, n));
    const int32_t* tiles = gram_tiles_dev(c, p);
    LAUNCH(c, cqr::launch_gram_leaves(p, xf, ldx, tiles, w.part + (sg.head ? np2 : 0), vec_ok(xf, ldx, n) ? 1 : 0,
                                      check, c->status, c->stream, 0, -1, c->num_sms));
  }
  std::vector<int> ta, tb;
  const int groups = (int)cqr::gram_nodes_tables(sg, ta, tb);
  const int nodes = (int)tb.size() / 3;
  if (nodes == 0) return;
  ta.insert(ta.end(), tb.begin(), tb.end());
  if (ta.size() > 65536) throw Fail{CQR_INVALID_ARGUMENT, -1, "sharded Gram: node table too large"};
  ck(cudaMemcpyAsync(w.tab, ta.data(), ta.size() * sizeof(int), cudaMemcpyHostToDevice, c->stream), "node table");
  LAUNCH(c, cqr::launch_gram_nodes(w.part, w.np, n, w.tab, groups, w.tab + 2 * groups, nodes, w.gsum, slots,
                                   c->status, c->stream));
}

void shard_top(cqr_ctx* c, long long m, int p, int n, const ShardWs& w, double* g) {
  int K = 0;
  const std::vector<int> prog = cqr::tree_program(m, p, &K);
  if (prog.size() > 65536) throw Fail{CQR_INVALID_ARGUMENT, -1, "sharded Gram: program too large"};
  ck(cudaMemcpyAsync(w.tab, prog.data(), prog.size() * sizeof(int), cudaMemcpyHostToDevice, c->stream), "program");
  LAUNCH(c, cqr::launch_gram_program(w.all, n, w.tab, (int)prog.size(), g, c->status, c->stream));
}

int shard_slots(long long m, int p) {
  int K = 0;
  cqr::tree_program(m, p, &K);
  return K;
}

// This rank's part over NCCL: tails to the next rank, heads from the previous, nodes all-gathered.
void gram_det(cqr_ctx* c, const double* x, long long ldx, int n, long long m, double* g, int check) {
  const int p = c->world, b = c->rank;
  const cqr::ShardGram sg = cqr::shard_gram_plan(m, p, b);
  const int K = shard_slots(m, p);
  ShardWs w = shard_ws(c, m, p, n, K);
  const size_t np2 = (size_t)w.np * w.np;
  double* head_in = w.ht;
  double* tail_out = w.ht + np2;
  shard_tail(c, sg, x, ldx, n, w.np, tail_out, check);
  // tails to the next rank, heads from the previous (one group)
  coll_sendrecv(c, tail_out, (sg.tail && !sg.span) ? b + 1 : -1, head_in, sg.head ? b - 1 : -1, np2);
  ck(cudaMemsetAsync(w.slots, 0, sizeof(double) * K * n * n, c->stream), "slots");
  shard_body(c, sg, x, ldx, n, w, head_in, tail_out, w.slots, check);
  if (sg.span) coll_sendrecv(c, tail_out, b + 1, nullptr, -1, np2);  // forward the continued chain
  coll_allgather(c, w.slots, w.all, (size_t)K * n * n);
  shard_top(c, m, p, n, w, g);
}

// The same protocol for p virtual ranks on this device, rank after rank: cqr_gram_sharded_sim.
// The hand-offs between ranks are device copies, or -- with an attached one-rank communicator --
// the NCCL calls of gram_det itself (ncclSend/ncclRecv to self in a group, ncclAllGather of the
// node slots), so the exchange code runs on a one-GPU box.
void gram_det_sim(cqr_ctx* c, const double* x, long long ldx, int n, long long m, int p, double* g) {
  const int K = shard_slots(m, p);
  ShardWs w = shard_ws(c, m, p, n, K);
  const size_t np2 = (size_t)w.np * w.np;
  const bool nccl = c->comm && !c->local_only && c->world == 1;
  ck(cudaMemsetAsync(w.all, 0, sizeof(double) * p * K * n * n, c->stream), "slots");
  double* in = w.ht;         // the chain arriving from the previous rank
  double* out = w.ht + np2;  // this rank's tail (or forwarded span)
  for (int b = 0; b < p; ++b) {
    const cqr::ShardGram sg = cqr::shard_gram_plan(m, p, b);
    const double* xb = x + sg.r0 * ldx;
    double* slots = nccl ? w.slots : w.all + (size_t)b * K * n * n;
    if (nccl) ck(cudaMemsetAsync(w.slots, 0, sizeof(double) * K * n * n, c->stream), "slots");
    shard_tail(c, sg, xb, ldx, n, w.np, out, 1);
    shard_body(c, sg, xb, ldx, n, w, in, out, slots, 1);
    if (nccl) {
      ckn(ncclAllGather(w.slots, w.all + (size_t)b * K * n * n, (size_t)K * n * n, ncclDouble, c->comm, c->stream),
          "allgather nodes");
      if (sg.tail) {
        ckn(ncclGroupStart(), "group");
        ckn(ncclSend(out, np2, ncclDouble, 0, c->comm, c->stream), "send tail");
        ckn(ncclRecv(in, np2, ncclDouble, 0, c->comm, c->stream), "recv head");
        ckn(ncclGroupEnd(), "group");
      }
    } else if (sg.tail) {
      ck(cudaMemcpyAsync(in, out, sizeof(double) * np2, cudaMemcpyDeviceToDevice, c->stream), "hand-off");
    }
  }
  shard_top(c, m, p, n, w, g);
}

// Gram of a device tall matrix (this rank's rows) -> g (n x n, mirrored), summed over ranks.
void gram_dev(cqr_ctx* c, const double* x, long long m, int n, long long ldx, double* g, int check = 0,
              Job* pj = nullptr) {
  if (pj && pj->det && multi(c)) {
    wait_all(*pj);
    gram_det(c, x, ldx, n, pj->m_global, g, check);
    return;
  }
  cqr::GramPlan p = cqr::gram_plan(m, n, cqr::gram_tma_ok(x, ldx, m, n));
  double* part = dbuf<double>(c, B_GPART, std::max<size_t>(p.workspace_doubles, 1));
  const int32_t* tiles = gram_tiles_dev(c, p);
  if (m > 0) {
    if (pj && pipelined(*pj) && pj->waited + 1 < (int)pj->bounds.size()) {
      // leaves as their rows land (whole leaves per launch: the partials are per leaf, so identical)
      int leaf = 0;
      for (size_t i = 1; i < pj->bounds.size() && leaf < p.leaves; ++i) {
        wait_rows(*pj, pj->bounds[i]);
        const int leaf1 = (i + 1 == pj->bounds.size()) ? p.leaves : (int)(pj->bounds[i] / 1024);
        if (leaf1 > leaf)
          LAUNCH(c, cqr::launch_gram_leaves(p, x, ldx, tiles, part, vec_ok(x, ldx, n) ? 1 : 0, check, c->status,
                                            c->stream, leaf, leaf1, c->num_sms));
        leaf = std::max(leaf, leaf1);
      }
    } else {
      if (pj) wait_all(*pj);
      // n in (64, 128], one CTA per leaf: the leaves past the last whole wave of CTAs run as a second launch
      // with each leaf's 36 macro tiles split over 3 CTAs (same tiles, same k order: identical partials), so
      // the last wave takes 1/3 leaf-times per round instead of a full leaf with most SMs idle
      const int waves = p.leaves / c->num_sms, split = waves * c->num_sms, rem = p.leaves - split;
      if (p.tma && p.np == 128 && p.parts == 1 && waves >= 1 && rem > 0 && 3 * rem <= 2 * (c->num_sms / 3) * 3) {
        cqr::GramPlan p3 = p;
        p3.parts = 3;
        p3.maxt = 1;
        p3.tiles_bytes = (size_t)p3.parts * p3.wpc * p3.maxt * sizeof(int32_t);
        const int32_t* tiles3 = gram_tiles_dev(c, p3, 1);
        LAUNCH(c, cqr::launch_gram_leaves(p, x, ldx, tiles, part, vec_ok(x, ldx, n) ? 1 : 0, check, c->status,
                                          c->stream, 0, split, c->num_sms));
        LAUNCH(c, cqr::launch_gram_leaves(p3, x, ldx, tiles3, part, vec_ok(x, ldx, n) ? 1 : 0, check, c->status,
                                          c->stream, split, p.leaves, c->num_sms));
      } else {
        LAUNCH(c, cqr::launch_gram_leaves(p, x, ldx, tiles, part, vec_ok(x, ldx, n) ? 1 : 0, check, c->status,
                                          c->stream, 0, -1, c->num_sms));
      }
    }
    LAUNCH(c, cqr::launch_gram_combine(p, part, g, multi(c) ? 0 : 1, c->status, c->stream));
    ++c->launches;
  } else {
    ck(cudaMemsetAsync(g, 0, sizeof(double) * n * n, c->stream), "memset");
  }
  if (multi(c)) {
    allreduce(c, g, (size_t)n * n);
    LAUNCH(c, cqr::launch_mirror_upper(g, n, c->status, c->stream));
  }
}

// X R = A on device rows; in may alias out.
void trisolve_dev(cqr_ctx* c, const double* in, long long ldi, double* out, long long ldo, long long m, int n,
                  const double* pack) {
  if (m <= 0) return;
  cqr::TrisolveArgs t{};
  t.in = in;
  t.ldi = ldi;
  t.out = out;
  t.ldo = ldo;
  t.m = m;
  t.n = n;
  t.pack = pack;
  t.vec16 = (vec_ok(in, ldi, n) && vec_ok(out, ldo, n)) ? 1 : 0;
  t.num_sms = c->num_sms;
  t.status = c->status;
  static const int variant = [] {  // CQR_TRISOLVE_VARIANT=1 forces the register kernel (A/B runs)
    const char* v = std::getenv("CQR_TRISOLVE_VARIANT");
    return v ? std::atoi(v) : 0;
  }();
  t.variant = variant;
  LAUNCH(c, cqr::launch_trisolve(t, c->stream));
}

const char* status_msg(int code) {
  switch (code) {
    case CQR_CHOLESKY_BREAKDOWN: return "cholesky breakdown";
    case CQR_SINGULAR_TRIANGULAR: return "singular triangular factor";
    case CQR_INVALID_ARGUMENT: return "A has non-finite entries";
    default: return "device failure";
  }
}

void copy_sync(cqr_ctx* c, void* dst, const void* src, size_t bytes, cudaMemcpyKind kind, const char* what) {
  ck(cudaMemcpyAsync(dst, src, bytes, kind, c->stream), what);
  ck(cudaStreamSynchronize(c->stream), what);
}

void reset_status(cqr_ctx* c) { ck(cudaMemsetAsync(c->status, 0, sizeof(DevStatus), c->stream), "status reset"); }

DevStatus read_status(cqr_ctx* c) {
  ck(cudaMemcpyAsync(c->status_h, c->status, sizeof(DevStatus), cudaMemcpyDeviceToHost, c->stream), "status D2H");
  ck(cudaStreamSynchronize(c->stream), "cudaStreamSynchronize");
  return *c->status_h;
}

void check_finite(cqr_ctx* c, const double* a, long long m, int n, long long lda);

// One CholeskyQR pass (engine.cpp:78-92): G = X^T X (+shift I), R = chol(G),
// X <- X R^{-1} (in -> out). shift_mode 0/1/2 as launch_cholesky.
void final_solve(Job& j, const double* in, long long ldi, const double* pack);

void cholesky_pass(Job& j, const double* in, long long ldi, Report& rep, double* r_out, int shift_mode,
                   double shift_value, const double* sgn_for_solve = nullptr, bool defer_solve = false,
                   int check = 0, bool last = false) {
  cqr_ctx* c = j.c;
  const int n = j.n;
  double* g = dbuf<double>(c, B_G, (size_t)n * n);
  {
    StageScope t(c, CQR_STAGE_GRAM);
    gram_dev(c, in, j.m_local, n, ldi, g, check, &j);
  }
  push_stage(rep, CQR_STAGE_GRAM);
  double* work = dbuf<double>(c, B_WORK, (size_t)n * n);
  double* shift_d = dbuf<double>(c, B_SCAL, 4);
  {
    StageScope t(c, CQR_STAGE_CHOLESKY);
    const double coef =
        11.0 * ((double)j.m_global * (double)n + (double)n * (double)(n + 1)) * kU;  // cholqr.cpp:21-26
    LAUNCH(c, cqr::launch_cholesky(g, n, r_out, work, shift_mode, shift_value, coef, shift_d, c->status, c->stream));
  }
  // the theory shift is resolved on the device; its value is patched into the
  // report after the attempt's single synchronisation
  push_stage(rep, CQR_STAGE_CHOLESKY, 0, shift_mode != 0, shift_value);
  if (defer_solve) return;
  double* pack = dbuf<double>(c, B_PACK2, cqr::trisolve_pack_doubles(n));
  {
    StageScope t(c, CQR_STAGE_TRISOLVE);
    LAUNCH(c, cqr::launch_pack_r(r_out, n, n, pack, 0, c->status, c->stream, sgn_for_solve));
    if (last)
      final_solve(j, in, ldi, pack);
    else
      trisolve_dev(c, in, ldi, j.q, j.ldq, j.m_local, n, pack);
  }
  push_stage(rep, CQR_STAGE_TRISOLVE);
}

// The last solve of a factorization; with the host pipeline each row chunk of Q
// is copied back as soon as it is solved (rows are independent, so the chunked
// solve is bit-identical).
void final_solve(Job& j, const double* in, long long ldi, const double* pack) {
  cqr_ctx* c = j.c;
  if (!pipelined(j)) {
    trisolve_dev(c, in, ldi, j.q, j.ldq, j.m_local, j.n, pack);
    return;
  }
  for (size_t i = 0; i + 1 < j.bounds.size(); ++i) {
    const long long r0 = j.bounds[i], r1 = j.bounds[i + 1];
    trisolve_dev(c, in + r0 * ldi, ldi, j.q + r0 * j.ldq, j.ldq, r1 - r0, j.n, pack);
    cudaEvent_t e = c->pipe_ev[j.bounds.size() - 1 + i];
    ck(cudaEventRecord(e, c->stream), "record");
    ck(cudaStreamWaitEvent(c->cstream, e, 0), "wait solve");
    ck(cudaMemcpy2DAsync(j.q_host + r0 * j.ldq_host, sizeof(double) * j.ldq_host, j.q + r0 * j.ldq,
                         sizeof(double) * j.ldq, sizeof(double) * j.n, r1 - r0, cudaMemcpyDeviceToHost, c->cstream),
       "Q D2H");
  }
}

struct Outcome {
  Report rep;
  bool has_r = false;
  const double* r_dev = nullptr;
};

// ---- tall Householder QR (householder.cu) -----------------------------------------------
// In place on this rank's rows of the m_global x n matrix W: R (n x n, replicated, unnormalised signs)
// and tau (n); the reflectors stay below W's diagonal. Each column: one reduction pass, summed over
// ranks (engine collectives), the reflector, one update pass.
struct HhWs {
  double *partial, *red, *coef, *tau;
  int blocks;
};

HhWs hh_ws(cqr_ctx* c, long long m_local, int n) {
  HhWs w;
  w.blocks = cqr::hh_blocks(m_local, c->num_sms);
  w.partial = dbuf<double>(c, B_HHPART, (size_t)w.blocks * n);
  w.red = dbuf<double>(c, B_HHRED, (size_t)3 * n);
  w.coef = w.red + 2 * n;
  w.tau = dbuf<double>(c, B_HHTAU, (size_t)n);
  return w;
}

void hh_factor(cqr_ctx* c, double* W, long long ldw, long long m_local, long long row0, int n, double* R,
               const HhWs& w) {
  ck(cudaMemsetAsync(R, 0, sizeof(double) * n * n, c->stream), "memset R");
  for (int col = 0; col < n; ++col) {
    LAUNCH(c, cqr::launch_hh_reduce(W, ldw, W, ldw, m_local, row0, col, n, w.blocks, w.partial, w.red, c->stream));
    allreduce(c, w.red, (size_t)2 * (n - col));
    LAUNCH(c, cqr::launch_hh_reflect_update(W, ldw, m_local, row0, col, n, w.red, w.coef, R, w.tau, c->num_sms,
                                            c->stream));
  }
}

// Q = H_0 ... H_{n-1} [I; 0] on this rank's rows from the reflectors of hh_factor
void hh_form_q(cqr_ctx* c, const double* W, long long ldw, double* Q, long long ldq, long long m_local,
               long long row0, int n, const HhWs& w) {
  LAUNCH(c, cqr::launch_hh_qinit(Q, ldq, m_local, row0, n, c->num_sms, c->stream));
  for (int col = n - 1; col >= 0; --col) {
    LAUNCH(c, cqr::launch_hh_reduce(W, ldw, Q, ldq, m_local, row0, col, n, w.blocks, w.partial, w.red, c->stream));
    allreduce(c, w.red, (size_t)2 * (n - col));
    LAUNCH(c, cqr::launch_hh_qstep(W, ldw, Q, ldq, m_local, row0, col, n, w.red, w.tau, w.coef, c->num_sms,
                                   c->stream));
  }
}

// householder_qr_thin (kernels.hpp:192-209) for Method::HouseholderQr (engine.cpp:227-239): Q and R with
// the R diagonal made non-negative (rows of R, columns of Q flipped).
Outcome run_householder(Job& j) {
  cqr_ctx* c = j.c;
  const int n = j.n;
  Outcome o;
  {
    StageScope t(c, CQR_STAGE_HOUSEHOLDER);
    double* W = dbuf<double>(c, B_HHW, (size_t)std::max<long long>(j.m_local, 1) * n);
    wait_all(j);
    if (j.m_local > 0)
      ck(cudaMemcpy2DAsync(W, sizeof(double) * n, j.a, sizeof(double) * j.lda, sizeof(double) * n, j.m_local,
                           cudaMemcpyDeviceToDevice, c->stream),
         "A copy");
    HhWs w = hh_ws(c, j.m_local, n);
    double* r = dbuf<double>(c, B_R, (size_t)n * n);
    double* sgn = dbuf<double>(c, B_SGN, (size_t)n);
    hh_factor(c, W, n, j.m_local, j.row0, n, r, w);
    hh_form_q(c, W, n, j.q, j.ldq, j.m_local, j.row0, n, w);
    LAUNCH(c, cqr::launch_normalize_sign(r, n, sgn, c->status, c->stream));
    LAUNCH(c, cqr::launch_col_sign(j.q, j.ldq, j.m_local, n, sgn, c->num_sms, c->stream));
    if (pipelined(j))  // Q back to the host
      for (size_t i = 0; i + 1 < j.bounds.size(); ++i) {
        const long long r0 = j.bounds[i], r1 = j.bounds[i + 1];
        cudaEvent_t e = c->pipe_ev[j.bounds.size() - 1 + i];
        ck(cudaEventRecord(e, c->stream), "record");
        ck(cudaStreamWaitEvent(c->cstream, e, 0), "wait");
        ck(cudaMemcpy2DAsync(j.q_host + r0 * j.ldq_host, sizeof(double) * j.ldq_host, j.q + r0 * j.ldq,
                             sizeof(double) * j.ldq, sizeof(double) * n, r1 - r0, cudaMemcpyDeviceToHost, c->cstream),
           "Q D2H");
      }
    o.r_dev = r;
  }
  push_stage(o.rep, CQR_STAGE_HOUSEHOLDER);
  DevStatus s = read_status(c);
  if (s.code != 0) throw Fail{s.code, s.index, status_msg(s.code)};
  o.has_r = j.opts.r_less == 0;
  return o;
}

// engine.cpp:241-284
Outcome run_cholqr_family(Job& j) {
  cqr_ctx* c = j.c;
  const int n = j.n;
  Outcome o;
  double* r1 = dbuf<double>(c, B_RT, (size_t)n * n);
  double* r2 = dbuf<double>(c, B_RH, (size_t)n * n);
  double* r3 = dbuf<double>(c, B_RTMP, (size_t)n * n);
  double* r = dbuf<double>(c, B_R, (size_t)n * n);
  const bool r_less = j.opts.r_less != 0;
  const int chk = j.check_first;
  if (j.method == CQR_CHOLQR) {
    cholesky_pass(j, j.a, j.lda, o.rep, r1, 0, 0.0, nullptr, false, chk, true);
    o.has_r = !r_less;
    o.r_dev = r1;
  } else if (j.method == CQR_CHOLQR2) {
    cholesky_pass(j, j.a, j.lda, o.rep, r1, 0, 0.0, nullptr, false, chk);
    cholesky_pass(j, j.q, j.ldq, o.rep, r2, 0, 0.0, nullptr, false, 0, true);
    if (!r_less) {
      StageScope t(c, CQR_STAGE_RECOVER);
      LAUNCH(c, cqr::launch_triangular_product(r2, r1, n, r, c->status, c->stream));
    }
    if (!r_less) push_stage(o.rep, CQR_STAGE_RECOVER);
    o.has_r = !r_less;
    o.r_dev = r;
  } else {  // CQR_SCHOLQR3
    const int mode = j.opts.shift_kind == CQR_SHIFT_FIXED ? 1 : 2;
    cholesky_pass(j, j.a, j.lda, o.rep, r1, mode, j.opts.shift_value, nullptr, false, chk);
    cholesky_pass(j, j.q, j.ldq, o.rep, r2, 0, 0.0);
    double* r3b = dbuf<double>(c, B_X, (size_t)n * n);
    cholesky_pass(j, j.q, j.ldq, o.rep, r3b, 0, 0.0, nullptr, false, 0, true);
    if (!r_less) {
      StageScope t(c, CQR_STAGE_RECOVER);
      LAUNCH(c, cqr::launch_triangular_product(r2, r1, n, r3, c->status, c->stream));
      LAUNCH(c, cqr::launch_triangular_product(r3b, r3, n, r, c->status, c->stream));
    }
    if (!r_less) push_stage(o.rep, CQR_STAGE_RECOVER);
    o.has_r = !r_less;
    o.r_dev = r;
  }
  DevStatus s = read_status(c);
  if (s.code != 0) throw Fail{s.code, s.index, status_msg(s.code)};
  if (j.method == CQR_SCHOLQR3 && j.opts.shift_kind != CQR_SHIFT_FIXED) {
    copy_sync(c, c->scal_h, dbuf<double>(c, B_SCAL, 4), sizeof(double), cudaMemcpyDeviceToHost, "shift D2H");
    for (auto& st : o.rep.stages)
      if (st.has_shift) {
        st.shift = c->scal_h[0];
        break;
      }
  }
  return o;
}

// engine.cpp:137-209 with the device pipeline.
Outcome run_precond(Job& j) {
  cqr_ctx* c = j.c;
  const int n = j.n;
  const long long m = j.m_global;
  const long long base_l = resolved_size(j.cfg, m, n);
  const bool r_less = j.opts.r_less != 0;
  if (j.cfg.strategy == CQR_LEVERAGE)
    throw Fail{CQR_INVALID_ARGUMENT, -1, "leverage sampling needs an oracle Q; call sample_rows_leverage directly"};
  for (int attempt = 0;; ++attempt) {
    cqr_sketch_cfg try_cfg = j.cfg;
    try_cfg.size = std::min<long long>(
        m, static_cast<long long>(std::llround(static_cast<double>(base_l) * std::pow(j.cfg.retry_growth, attempt))));
    const uint64_t seed = attempt == 0 ? j.cfg.seed : derive(j.cfg.seed, static_cast<uint64_t>(attempt));
    const bool last = attempt >= j.cfg.max_retries;
    const long long l = resolved_size(try_cfg, m, n);
    Outcome o;
    if (attempt > 0) reset_status(c);
    double* a1 = dbuf<double>(c, B_A1, (size_t)l * n);
    // ---- Sketch (sketch.cpp:94-127)
    {
      StageScope t(c, CQR_STAGE_SKETCH);
      if (try_cfg.strategy == CQR_GAUSSIAN) {
        const SketchRun sr = sketch_setup(c, j.a, j.lda, j.m_local, m, j.row0, n, (int)l,
                                          pipelined(j) ? (int)j.bounds.size() - 1 : 1);
        const cqr::SketchPlan& sp = sr.p;
        if (j.m_local > 0) {
          const int vec = vec_ok(j.a, j.lda, n) ? 1 : 0, chk = attempt == 0 ? j.check_first : 0;
          if (pipelined(j) && j.waited + 1 < (int)j.bounds.size()) {
            // k-chunks as their rows land (whole k-chunks per launch: identical partials)
            int y = 0;
            for (size_t i = 1; i < j.bounds.size() && y < sp.kchunks; ++i) {
              wait_rows(j, j.bounds[i]);
              const int y1 = (i + 1 == j.bounds.size()) ? sp.kchunks : (int)(j.bounds[i] / sp.rows_per_chunk);
              if (y1 > y) LAUNCH(c, sketch_launch(c, sr, j.a, j.lda, m, j.row0, seed, vec, chk, y, y1));
              y = std::max(y, y1);
            }
          } else {
            wait_all(j);
            LAUNCH(c, sketch_launch(c, sr, j.a, j.lda, m, j.row0, seed, vec, chk));
          }
          LAUNCH(c, cqr::launch_sketch_reduce(sp, sr.part, a1, c->status, c->stream));
        } else {
          ck(cudaMemsetAsync(a1, 0, sizeof(double) * l * n, c->stream), "memset");
        }
      } else {  // Uniform (sketch.cpp:27-55)
        long long* idx = nullptr;
        if (try_cfg.without_replacement) {
          std::vector<long long> h;
          std::unordered_set<long long> seen;
          uint64_t pos = 0;
          while ((long long)h.size() < l) {
            const long long i = (long long)(unit_at(seed, pos++) * (double)m);
            if (seen.insert(i).second) h.push_back(i);
          }
          idx = dbuf<long long>(c, B_IDX, (size_t)l);
          ck(cudaMemcpyAsync(idx, h.data(), sizeof(long long) * l, cudaMemcpyHostToDevice, c->stream), "idx H2D");
          ck(cudaStreamSynchronize(c->stream), "sync");
        }
        wait_all(j);
        LAUNCH(c, cqr::launch_gather_rows(j.a, j.lda, j.m_local, m, j.row0, n, (int)l, seed, idx, a1, nullptr,
                                          c->status, c->stream));
      }
      allreduce(c, a1, (size_t)l * n);
    }
    // ---- Precondition: R~ = QR/LU of A1 (kernels.hpp:175-257)
    double* rt = dbuf<double>(c, B_RT, (size_t)n * n);
    double* work = dbuf<double>(c, B_WORK, std::max<size_t>(cqr::qr_work_doubles((int)l, n), (size_t)n * n));
    double* pack1 = dbuf<double>(c, B_PACK1, cqr::trisolve_pack_doubles(n));
    {
      StageScope t(c, CQR_STAGE_PRECONDITION);
      if (j.precond) {
        std::vector<double> ha((size_t)l * n), hr((size_t)n * n, 0.0);
        ck(cudaMemcpyAsync(ha.data(), a1, sizeof(double) * l * n, cudaMemcpyDeviceToHost, c->stream), "a1 D2H");
        ck(cudaStreamSynchronize(c->stream), "sync");
        int64_t idx = -1;
        const int st = j.precond(j.user, ha.data(), l, n, hr.data(), &idx);
        if (st == CQR_SINGULAR_TRIANGULAR) {
          if (last) throw Fail{CQR_SINGULAR_TRIANGULAR, idx, "preconditioner: singular triangular factor"};
          continue;
        }
        if (st != CQR_OK) throw Fail{st, idx, "preconditioner failed"};
        ck(cudaMemcpyAsync(rt, hr.data(), sizeof(double) * n * n, cudaMemcpyHostToDevice, c->stream), "rt H2D");
        ck(cudaStreamSynchronize(c->stream), "sync");
      } else if (j.method == CQR_RLU) {
        LAUNCH(c, cqr::launch_lu_u(a1, (int)l, n, rt, work, c->status, c->stream));
      } else {
        LAUNCH(c, cqr::launch_qr_r(a1, (int)l, n, rt, work, c->status, c->stream));
      }
      // degenerate_diagonal (engine.cpp:118-127) + packing for the solve
      LAUNCH(c, cqr::launch_pack_r(rt, n, n, pack1, 1, c->status, c->stream));
    }
    push_stage(o.rep, CQR_STAGE_SKETCH, attempt);
    // ---- X = A R~^{-1} (A -> Q buffer; A stays intact for a retry)
    {
      StageScope t(c, CQR_STAGE_TRISOLVE);
      wait_all(j);
      trisolve_dev(c, j.a, j.lda, j.q, j.ldq, j.m_local, n, pack1);
    }
    const bool diag = j.opts.diagnostics != 0;
    // ---- CholeskyQR on X (Gram, Cholesky; the solve is deferred past Recover so
    // the sign normalisation of engine.cpp:109-116 can be fused into it)
    double* rh = dbuf<double>(c, B_RH, (size_t)n * n);
    Report pass;
    cholesky_pass(j, j.q, j.ldq, pass, rh, 0, 0.0, nullptr, true);
    double cond = 0.0;
    if (diag) {  // cond(X) = cond(R^) (engine.cpp:94-100) by a device Jacobi sweep; inf when the pass fails
      DevStatus s = read_status(c);
      if (s.code == 0) {
        double* cw = dbuf<double>(c, B_DIAG, (size_t)n * n + 2);
        LAUNCH(c, cqr::launch_jacobi_cond(rh, n, cw, cw + (size_t)n * n, c->stream));
        copy_sync(c, c->scal_h, cw + (size_t)n * n, sizeof(double), cudaMemcpyDeviceToHost, "cond D2H");
        cond = c->scal_h[0];
      } else {
        cond = std::numeric_limits<double>::infinity();
      }
    }
    push_stage(o.rep, CQR_STAGE_PRECONDITION, 0, false, 0.0, diag, cond);
    for (auto& s : pass.stages) o.rep.stages.push_back(s);
    double* r = dbuf<double>(c, B_R, (size_t)n * n);
    double* sgn = dbuf<double>(c, B_SGN, (size_t)n);
    cudaEvent_t ev_r = nullptr;
    if (!r_less) {
      // (a side stream for this step measured no better: the last solve's persistent CTAs hold every SM)
      StageScope t(c, CQR_STAGE_RECOVER);
      LAUNCH(c, cqr::launch_triangular_product(rh, rt, n, r, c->status, c->stream));
      LAUNCH(c, cqr::launch_normalize_sign(r, n, sgn, c->status, c->stream));
    }
    if (!r_less && j.want_r) {
      ev_r = next_event(c);
      ck(cudaEventRecord(ev_r, c->stream), "record R");  // R is final: its copy overlaps the last solve
    }
    double* pack2 = dbuf<double>(c, B_PACK2, cqr::trisolve_pack_doubles(n));
    {
      StageScope t(c, CQR_STAGE_TRISOLVE);
      LAUNCH(c, cqr::launch_pack_r(rh, n, n, pack2, 0, c->status, c->stream, r_less ? nullptr : sgn));
      final_solve(j, j.q, j.ldq, pack2);  // the column signs are folded into the pack
    }
    if (!r_less && j.want_r) {  // R is final: bring it to pinned host memory while the last solve runs
      if (c->r_pin_n < (size_t)n * n) {
        if (c->r_pin) cudaFreeHost(c->r_pin);
        c->r_pin = nullptr;
        c->r_pin_n = 0;
        ck(cudaMallocHost(&c->r_pin, sizeof(double) * n * n), "cudaMallocHost (R staging)");
        c->r_pin_n = (size_t)n * n;
      }
      if (!c->cstream) ck(cudaStreamCreateWithFlags(&c->cstream, cudaStreamNonBlocking), "copy stream");
      ck(cudaStreamWaitEvent(c->cstream, ev_r, 0), "wait R");
      ck(cudaMemcpyAsync(c->r_pin, r, sizeof(double) * n * n, cudaMemcpyDeviceToHost, c->cstream), "R D2H");
      j.r_copied = true;
    }
    push_stage(o.rep, CQR_STAGE_TRISOLVE);
    if (!r_less) push_stage(o.rep, CQR_STAGE_RECOVER);
    DevStatus s = read_status(c);
    if (s.code == 0) {
      o.has_r = !r_less;
      o.r_dev = r;
      o.rep.sketch_rows = l;
      return o;
    }
    if ((s.code == CQR_CHOLESKY_BREAKDOWN || s.code == CQR_SINGULAR_TRIANGULAR) && !last) continue;
    throw Fail{s.code, s.code == CQR_INVALID_ARGUMENT ? -1 : s.index, status_msg(s.code)};
  }
}

void fill_report(cqr_ctx* c, cqr_report* rep, const Outcome* o, int status, long long index, bool r_less,
                 int method, long long n, long long l, int workers) {
  // stage times from the recorded events (accumulated across attempts)
  double ms[CQR_STAGE_COUNT] = {0};
  for (auto& e : c->stage_evs) {
    float t = 0.f;
    if (cudaEventElapsedTime(&t, e.a, e.b) == cudaSuccess) ms[e.stage] += t;  // the stream is synchronised
  }
  cudaGetLastError();
  c->stage_evs.clear();
  c->ev_used = 0;
  if (!rep) return;
  std::memset(rep, 0, sizeof(*rep));
  rep->status = status;
  rep->index = index;
  rep->r_less = r_less ? 1 : 0;
  double tot = 0.0;
  for (int s = 0; s < CQR_STAGE_COUNT; ++s) {
    rep->stage_ms[s] = ms[s];
    tot += ms[s];
  }
  rep->total_ms = tot;
  if (o) {
    rep->n_stages = (int)std::min<size_t>(o->rep.stages.size(), CQR_MAX_STAGE_INFOS);
    for (int i = 0; i < rep->n_stages; ++i) rep->stages[i] = o->rep.stages[i];
    rep->sketch_rows = o->rep.sketch_rows;
  }
  int rmin, rmax;
  double vmin, vmax;
  // parexec.cpp:64-75: the model of the p that ran -- the ranks of an attached communicator, else
  // the simulated worker count of the options (run_parallel on one process)
  const int p = attached(c) ? c->world : std::max(1, workers);
  cqr_comm_model(method, p, n, l, &rmin, &rmax, &vmin, &vmax);
  rep->comm_rounds = rmax;
  rep->comm_volume = vmax;
}

template <typename F>
int guarded(cqr_ctx* c, F&& f) {
  try {
    f();
    return CQR_OK;
  } catch (const Fail& e) {
    if (c) c->err = e.msg;
    return e.code;
  }
}

// device-side finiteness check (engine.cpp:222, errors.hpp:89-93): one pass
// over A with 16-byte loads; a warp vote keeps the flag write rare.
__global__ void finite_kernel(const double* __restrict__ a, long long lda, long long m, int n, int vec,
                              DevStatus* st) {
  bool bad = false;
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long t0 = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (lda == n && vec) {
    const double2* p = reinterpret_cast<const double2*>(a);
    const long long total = m * n / 2;
    for (long long e = t0; e < total; e += stride) {
      const double2 v = __ldg(p + e);
      bad |= !isfinite(v.x) || !isfinite(v.y);
    }
    if (t0 == 0 && (m * n) % 2) bad |= !isfinite(a[m * n - 1]);
  } else {
    for (long long i = t0 / 32; i < m; i += stride / 32)
      for (int j = (int)(t0 & 31); j < n; j += 32) bad |= !isfinite(a[i * lda + j]);
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) cqr::set_status(st, CQR_INVALID_ARGUMENT, -1);
}

void check_finite(cqr_ctx* c, const double* a, long long m, int n, long long lda) {
  if (m <= 0) return;
  const int vec = (reinterpret_cast<uintptr_t>(a) & 15) == 0;
  finite_kernel<<<c->num_sms * 8, 256, 0, c->stream>>>(a, lda, m, n, vec, c->status);
  ck(cudaGetLastError(), "finite_kernel");
  ++c->launches;
}

// CQR_TRACE=1: host timeline of one call (us since entry) and the device gap before the first stage
struct CallTrace {
  bool on = false;
  std::chrono::steady_clock::time_point t0;
  cudaEvent_t e0 = nullptr;
  std::vector<std::pair<const char*, double>> marks;
  void mark(const char* what) {
    if (on)
      marks.push_back({what, std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count()});
  }
};

int factor_dev_impl(cqr_ctx* c, Job& j, double* r_host, long long ldr, cqr_report* report) {
  static const bool trace = std::getenv("CQR_TRACE") != nullptr;
  CallTrace tr;
  tr.on = trace;
  if (tr.on) {
    tr.t0 = std::chrono::steady_clock::now();
    cudaEventCreate(&tr.e0);
    cudaEventRecord(tr.e0, c->stream);
  }
  Outcome o;
  long long index = -1;
  const bool r_less = j.opts.r_less != 0;
  j.want_r = r_host != nullptr;
  const long long l =
      (j.m_global >= j.n && j.n >= 1) ? resolved_size(j.cfg, j.m_global, j.n) : 0;
  c->stage_evs.clear();
  c->ev_used = 0;
  int st = CQR_OK;
  try {
    require(j.n >= 1 && j.m_global >= j.n, "need m >= n >= 1");
    require(j.lda >= j.n && j.ldq >= j.n, "leading dimension must be >= n");
    require(j.m_local >= 0 && j.row0 >= 0 && j.row0 + j.m_local <= j.m_global, "bad shard");
    require(j.n <= 512, "n > 512 is not supported by the device kernels");
    // engine.cpp:224: p in [1, m] (0 = a zero-initialised options struct: one worker)
    require(j.opts.workers >= 0 && j.opts.workers <= j.m_global, "worker count must be in [1, m]");
    ck(cudaSetDevice(c->device), "cudaSetDevice");
    // non-finite input is rejected up front (engine.cpp:222). One process: the
    // check only sets the status word (read with the attempt's single sync);
    // several ranks agree on it first so they take the same path.
    reset_status(c);
    const bool gaussian = j.method == CQR_RQR_GAUSSIAN || j.cfg.strategy == CQR_GAUSSIAN;
    const bool family = j.method == CQR_CHOLQR || j.method == CQR_CHOLQR2 || j.method == CQR_SCHOLQR3;
    j.check_first = (!attached(c) && !j.precond && (family || gaussian)) ? 1 : 0;
    if (!j.check_first) {
      wait_all(j);
      check_finite(c, j.a, j.m_local, j.n, j.lda);
    }
    if (attached(c)) {  // every rank takes the same path
      DevStatus s0 = read_status(c);
      // flags[1]: this rank's rows are not its standard block (parexec.cpp:13-15); then
      // every rank sums plain Gram partials instead of the rank-count-independent tree
      int flags[2] = {s0.code != 0, j.row0 != cqr::shard_offset(j.m_global, c->world, c->rank) ||
                                        j.row0 + j.m_local != cqr::shard_offset(j.m_global, c->world, c->rank + 1)};
      {
        int* flag = dbuf<int>(c, B_DIAG, 2);
        ck(cudaMemcpyAsync(flag, flags, sizeof(flags), cudaMemcpyHostToDevice, c->stream), "flag");
        coll_allreduce(c, flag, 2, CQR_COMM_I32_MAX);
        ck(cudaMemcpyAsync(flags, flag, sizeof(flags), cudaMemcpyDeviceToHost, c->stream), "flag");
        ck(cudaStreamSynchronize(c->stream), "sync");
      }
      if (flags[0]) throw Fail{CQR_INVALID_ARGUMENT, -1, "A has non-finite entries"};
      j.det = flags[1] ? 0 : 1;
    }
    switch (j.method) {
      case CQR_CHOLQR:
      case CQR_CHOLQR2:
      case CQR_SCHOLQR3:
        o = run_cholqr_family(j);
        break;
      case CQR_RQR:
      case CQR_RLU:
        o = run_precond(j);
        break;
      case CQR_RQR_GAUSSIAN:
        j.cfg.strategy = CQR_GAUSSIAN;
        o = run_precond(j);
        break;
      case CQR_HOUSEHOLDER:
        o = run_householder(j);
        break;
      default:
        throw Fail{CQR_INVALID_ARGUMENT, -1, "unknown method"};
    }
    tr.mark("attempts done (status read)");
    if (o.has_r && r_host && j.r_copied) {
      ck(cudaStreamSynchronize(c->cstream), "sync R");
      for (int i = 0; i < j.n; ++i) std::memcpy(r_host + (size_t)i * ldr, c->r_pin + (size_t)i * j.n, sizeof(double) * j.n);
    } else if (o.has_r && r_host) {
      ck(cudaMemcpy2DAsync(r_host, sizeof(double) * ldr, o.r_dev, sizeof(double) * j.n, sizeof(double) * j.n, j.n,
                           cudaMemcpyDeviceToHost, c->stream),
         "R D2H");
      ck(cudaStreamSynchronize(c->stream), "sync");
    }
    tr.mark("R D2H");
  } catch (const Fail& e) {
    st = e.code;
    index = e.index;
    c->err = e.msg;
    cudaStreamSynchronize(c->stream);
    cudaGetLastError();
  }
  fill_report(c, report, st == CQR_OK ? &o : nullptr, st, index, r_less, j.method, j.n, l, j.opts.workers);
  tr.mark("report");
  if (tr.on) {
    float gap = 0.f, span = 0.f;
    if (!c->stage_evs.empty()) {
      cudaEventElapsedTime(&gap, tr.e0, c->stage_evs.front().a);
      cudaEventElapsedTime(&span, c->stage_evs.front().a, c->stage_evs.back().b);
    }
    std::fprintf(stderr, "CQR_TRACE device: entry->first stage %.1f us, first->last stage %.1f us; host:", gap * 1e3,
                 span * 1e3);
    for (auto& m : tr.marks) std::fprintf(stderr, " %s %.1f", m.first, m.second);
    std::fprintf(stderr, "\n");
    cudaEventDestroy(tr.e0);
  }
  return st;
}

}  // namespace

namespace cqr {
cudaError_t allow_max_smem_impl(const void* kernel) {
  static std::mutex mu;
  static std::set<std::pair<int, const void*>> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> g(mu);
  if (done.count({dev, kernel})) return cudaSuccess;
  int optin = 0;
  e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (e != cudaSuccess) return e;
  cudaFuncAttributes fa;
  e = cudaFuncGetAttributes(&fa, kernel);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - (int)fa.sharedSizeBytes);
  if (e == cudaSuccess) done.insert({dev, kernel});
  return e;
}
}  // namespace cqr

// =============================== C ABI ===========================================
extern "C" {

int cqr_abi_version(void) { return CQR_ABI_VERSION; }

void cqr_sketch_cfg_default(cqr_sketch_cfg* cfg) {
  if (cfg) *cfg = default_cfg();
}

void cqr_options_default(cqr_options* opts) {
  if (opts) *opts = default_opts();
}

int64_t cqr_resolved_size(const cqr_sketch_cfg* cfg, int64_t m, int64_t n) {
  return resolved_size(cfg ? *cfg : default_cfg(), m, n);
}

int cqr_create(cqr_ctx** out, int device) {
  if (!out) return CQR_INVALID_ARGUMENT;
  *out = nullptr;
  cqr_ctx* c = new cqr_ctx();
  c->device = device;
  const int st = guarded(c, [&] {
    ck(cudaSetDevice(device), "cudaSetDevice");
    ck(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device), "attr");
    ck(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking), "stream");
    ck(cudaMalloc(&c->status, sizeof(DevStatus)), "status");
    ck(cudaMallocHost(&c->status_h, sizeof(DevStatus)), "status_h");
    ck(cudaMallocHost(&c->scal_h, 8 * sizeof(double)), "scal_h");
  });
  if (st != CQR_OK) {
    std::fprintf(stderr, "cqr_create: %s\n", c->err.c_str());
    delete c;
    return st;
  }
  *out = c;
  return CQR_OK;
}

int cqr_destroy(cqr_ctx* c) {
  if (!c) return CQR_OK;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  for (auto& b : c->bufs)
    if (b.p) cudaFree(b.p);
  for (auto e : c->ev_pool) cudaEventDestroy(e);
  if (c->comm) ncclCommDestroy(c->comm);
  if (c->status) cudaFree(c->status);
  if (c->status_h) cudaFreeHost(c->status_h);
  if (c->scal_h) cudaFreeHost(c->scal_h);
  if (c->r_pin) cudaFreeHost(c->r_pin);
  if (c->stage_h) cudaFreeHost(c->stage_h);
  if (c->stream) cudaStreamDestroy(c->stream);
  if (c->cstream) cudaStreamDestroy(c->cstream);
  for (auto e : c->pipe_ev) cudaEventDestroy(e);
  if (c->order_ev) cudaEventDestroy(c->order_ev);
  delete c;
  return CQR_OK;
}

const char* cqr_last_error(const cqr_ctx* c) { return c ? c->err.c_str() : "null context"; }

int cqr_comm_id_size(void) { return (int)sizeof(ncclUniqueId); }

int cqr_comm_make_id(void* id) {
  ncclUniqueId u;
  if (ncclGetUniqueId(&u) != ncclSuccess) return CQR_NCCL_ERROR;
  std::memcpy(id, &u, sizeof(u));
  return CQR_OK;
}

int cqr_attach_comm(cqr_ctx* c, int rank, int world, const void* id) {
  if (!c || world < 1 || rank < 0 || rank >= world) return CQR_INVALID_ARGUMENT;
  return guarded(c, [&] {
    ck(cudaSetDevice(c->device), "cudaSetDevice");
    if (c->comm) {
      ncclCommDestroy(c->comm);
      c->comm = nullptr;
    }
    c->has_hcomm = false;
    c->rank = rank;
    c->world = world;
    // an attached communicator switches the collective paths on, also for world == 1
    // (a one-rank NCCL communicator: the exchange steps run as on a multi-GPU job)
    ncclUniqueId u;
    std::memcpy(&u, id, sizeof(u));
    ckn(ncclCommInitRank(&c->comm, world, u, rank), "ncclCommInitRank");
  });
}

int cqr_attach_host_comm(cqr_ctx* c, int rank, int world, const cqr_host_comm* hc) {
  if (!c || world < 1 || rank < 0 || rank >= world) return CQR_INVALID_ARGUMENT;
  if (hc && (!hc->allreduce || !hc->sendrecv || !hc->allgather)) return CQR_INVALID_ARGUMENT;
  if (!hc && world != 1) return CQR_INVALID_ARGUMENT;
  return guarded(c, [&] {
    ck(cudaSetDevice(c->device), "cudaSetDevice");
    if (c->comm) {
      ncclCommDestroy(c->comm);
      c->comm = nullptr;
    }
    c->has_hcomm = hc != nullptr;
    c->hcomm = hc ? *hc : cqr_host_comm{};
    c->rank = hc ? rank : 0;
    c->world = hc ? world : 1;
  });
}

int cqr_stream_handle(cqr_ctx* c, void** stream) {
  if (!c || !stream) return CQR_INVALID_ARGUMENT;
  *stream = (void*)c->stream;
  return CQR_OK;
}

int cqr_order_after(cqr_ctx* c, void* stream) {
  if (!c) return CQR_INVALID_ARGUMENT;
  return guarded(c, [&] {
    if (!c->order_ev) ck(cudaEventCreateWithFlags(&c->order_ev, cudaEventDisableTiming), "event");
    ck(cudaEventRecord(c->order_ev, (cudaStream_t)stream), "record");
    ck(cudaStreamWaitEvent(c->stream, c->order_ev, 0), "wait");
  });
}

int64_t cqr_launch_count(const cqr_ctx* c) { return c ? c->launches : 0; }

int cqr_factor_dev(cqr_ctx* c, int method, const double* a, int64_t m_local, int64_t m_global, int64_t row0,
                   int64_t n, int64_t lda, const cqr_sketch_cfg* cfg, const cqr_options* opts, double* q,
                   int64_t ldq, double* r, int64_t ldr, cqr_report* report) {
  if (!c) return CQR_INVALID_ARGUMENT;
  Job j{};
  j.c = c;
  j.method = method;
  j.a = a;
  j.m_local = m_local;
  j.m_global = m_global;
  j.row0 = row0;
  j.n = (int)n;
  j.lda = lda;
  j.q = q;
  j.ldq = ldq;
  j.cfg = cfg ? *cfg : default_cfg();
  j.opts = opts ? *opts : default_opts();
  if (c->world <= 1 && (m_local != m_global || row0 != 0)) {
    c->err = "sharded call without an attached communicator";
    return CQR_INVALID_ARGUMENT;
  }
  return factor_dev_impl(c, j, r, ldr, report);
}

// Host buffers: this rank's rows [row0, row0 + m) of an m_global-row matrix
// (m_global == m, row0 == 0 for the unsharded calls).
static int factor_host(cqr_ctx* c, int method, const double* a, int64_t m, int64_t m_global, int64_t row0, int64_t n,
                       int64_t lda, const cqr_sketch_cfg* cfg, const cqr_options* opts, double* q, int64_t ldq,
                       double* r, int64_t ldr, cqr_report* report, cqr_precond_fn fn, void* user) {
  if (!c) return CQR_INVALID_ARGUMENT;
  const bool sharded = m != m_global || row0 != 0;
  if (m < 1 || n < 1 || lda < n || ldq < n || (r && ldr < n) || row0 < 0 || row0 + m > m_global ||
      (sharded && !attached(c)) || (!sharded && c->world > 1)) {
    c->err = sharded && !attached(c) ? "sharded call without an attached communicator"
             : !sharded && c->world > 1 ? "a multi-rank context takes its shard through cqr_factor_sharded"
                                        : "bad shape";
    if (report) {
      std::memset(report, 0, sizeof(*report));
      report->status = CQR_INVALID_ARGUMENT;
      report->index = -1;
    }
    return CQR_INVALID_ARGUMENT;
  }
  int st = guarded(c, [&] {
    ck(cudaSetDevice(c->device), "cudaSetDevice");
    double* da = dbuf<double>(c, B_HA, (size_t)m * n);
    double* dq = dbuf<double>(c, B_HQ, (size_t)m * n);
    Job j{};
    // chunked H2D on the copy stream (8 chunks of >= 8 MB), consumed as it lands
    if (!c->cstream) ck(cudaStreamCreateWithFlags(&c->cstream, cudaStreamNonBlocking), "copy stream");
    int nch = (int)std::min<long long>(8, std::max<long long>(1, (m * n * 8) / (8 << 20)));
    j.bounds.clear();
    for (int i = 0; i <= nch; ++i) j.bounds.push_back(m * i / nch);
    while ((int)c->pipe_ev.size() < 2 * nch) {
      cudaEvent_t e;
      ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
      c->pipe_ev.push_back(e);
    }
    ck(cudaEventRecord(c->pipe_ev[0], c->stream), "record");  // previous work on the compute stream done
    ck(cudaStreamWaitEvent(c->cstream, c->pipe_ev[0], 0), "wait");
    for (int i = 0; i < nch; ++i) {
      const long long r0 = j.bounds[i], r1 = j.bounds[i + 1];
      ck(cudaMemcpy2DAsync(da + r0 * n, sizeof(double) * n, a + r0 * lda, sizeof(double) * lda, sizeof(double) * n,
                           r1 - r0, cudaMemcpyHostToDevice, c->cstream),
         "A H2D");
      ck(cudaEventRecord(c->pipe_ev[i], c->cstream), "record");
    }
    j.a_host = a;
    j.lda_host = lda;
    j.q_host = q;
    j.ldq_host = ldq;
    j.c = c;
    j.method = method;
    j.a = da;
    j.m_local = m;
    j.m_global = m_global;
    j.row0 = row0;
    j.n = (int)n;
    j.lda = n;
    j.q = dq;
    j.ldq = n;
    j.cfg = cfg ? *cfg : default_cfg();
    j.opts = opts ? *opts : default_opts();
    j.precond = fn;
    j.user = user;
    const int s = factor_dev_impl(c, j, r, ldr, report);
    ck(cudaStreamSynchronize(c->cstream), "sync copies");
    if (s != CQR_OK) throw Fail{s, report ? report->index : -1, c->err};
    ck(cudaStreamSynchronize(c->stream), "sync");
  });
  return st;
}

int cqr_factor(cqr_ctx* c, int method, const double* a, int64_t m, int64_t n, int64_t lda,
               const cqr_sketch_cfg* cfg, const cqr_options* opts, double* q, int64_t ldq, double* r, int64_t ldr,
               cqr_report* report) {
  return factor_host(c, method, a, m, m, 0, n, lda, cfg, opts, q, ldq, r, ldr, report, nullptr, nullptr);
}

int cqr_factor_sharded(cqr_ctx* c, int method, const double* a, int64_t m_local, int64_t m_global, int64_t row0,
                       int64_t n, int64_t lda, const cqr_sketch_cfg* cfg, const cqr_options* opts, double* q,
                       int64_t ldq, double* r, int64_t ldr, cqr_report* report) {
  return factor_host(c, method, a, m_local, m_global, row0, n, lda, cfg, opts, q, ldq, r, ldr, report, nullptr,
                     nullptr);
}

int cqr_precond_factor(cqr_ctx* c, const double* a, int64_t m, int64_t n, int64_t lda, cqr_precond_fn precond,
                       void* user, const cqr_sketch_cfg* cfg, const cqr_options* opts, double* q, int64_t ldq,
                       double* r, int64_t ldr, cqr_report* report) {
  if (!precond) return CQR_INVALID_ARGUMENT;
  return factor_host(c, CQR_RQR, a, m, m, 0, n, lda, cfg, opts, q, ldq, r, ldr, report, precond, user);
}

// ---- kernel-level entry points -------------------------------------------------------
int cqr_gram_dev(cqr_ctx* c, const double* x, int64_t m, int64_t n, int64_t ldx, double* g) {
  if (!c || m < n || n < 1 || ldx < n || n > 512) return CQR_INVALID_ARGUMENT;  // kernels.hpp:65
  return guarded(c, [&] {
    ck(cudaSetDevice(c->device), "cudaSetDevice");
    reset_status(c);
    gram_dev(c, x, m, (int)n, ldx, g);
    ck(cudaStreamSynchronize(c->stream), "sync");
  });
}

int cqr_gram_sharded_sim(cqr_ctx* c, const double* x, int64_t m, int64_t n, int64_t ldx, int p, double* g) {
  if (!c || m < n || n < 1 || ldx < n || n > 512 || p < 1 || p > m) return CQR_INVALID_ARGUMENT;
  return guarded(c, [&] {
    ck(cudaSetDevice(c->device), "cudaSetDevice");
    reset_status(c);
    gram_det_sim(c, x, ldx, (int)n, m, p, g);
    DevStatus s = read_status(c);
    if (s.code) throw Fail{s.code, s.index, status_msg(s.code)};
  });
}

int cqr_gram(cqr_ctx* c, const double* x, int64_t m, int64_t n, int64_t ldx, double* g) {
  if (!c || m < n || n < 1 || ldx < n || n > 512) return CQR_INVALID_ARGUMENT;
  return guarded(c, [&] {
    ck(cudaSetDevice(c->device), "cudaSetDevice");
    double* dx = dbuf<double>(c, B_HA, (size_t)m * n);
    double* dg = dbuf<double>(c, B_G, (size_t)n * n);
    ck(cudaMemcpy2DAsync(dx, sizeof(double) * n, x, sizeof(double) * ldx, sizeof(double) * n, m,
                         cudaMemcpyHostToDevice, c->stream),
       "X H2D");
    reset_status(c);
    gram_dev(c, dx, m, (int)n, n, dg);
    ck(cudaMemcpyAsync(g, dg, sizeof(double) * n * n, cudaMemcpyDeviceToHost, c->stream), "G D2H");
    ck(cudaStreamSynchronize(c->stream), "sync");
  });
}

int cqr_cholesky_upper(cqr_ctx* c, const double* g, int64_t n, double* r, int64_t* pivot) {
  if (!c || n < 1 || n > 4096) return CQR_INVALID_ARGUMENT;
  if (pivot) *pivot = -1;
  long long idx = -1;
  int st = guarded(c, [&] {
    ck(cudaSetDevice(c->device), "cudaSetDevice");
    double* dg = dbuf<double>(c, B_G, (size_t)n * n);
    double* dr = dbuf<double>(c, B_RH, (size_t)n * n);
    double* work = dbuf<double>(c, B_WORK, (size_t)n * n);
    ck(cudaMemcpyAsync(dg, g, sizeof(double) * n * n, cudaMemcpyHostToDevice, c->stream), "G H2D");
    reset_status(c);
    LAUNCH(c, cqr::launch_cholesky(dg, (int)n, dr, work, 0, 0.0, 0.0, nullptr, c->status, c->stream));
    DevStatus s = read_status(c);
    if (s.code) {
      idx = s.index;
      throw Fail{s.code, s.index, "cholesky breakdown"};
    }
    copy_sync(c, r, dr, sizeof(double) * n * n, cudaMemcpyDeviceToHost, "R D2H");
  });
  if (pivot) *pivot = idx;
  return st;
}

int cqr_trisolve_inplace_dev(cqr_ctx* c, double* x, int64_t m, int64_t n, int64_t ldx, const double* r_dev,
                             int64_t* index) {
  if (!c || n < 1 || n > 512 || ldx < n || m < 0) return CQR_INVALID_ARGUMENT;
  if (index) *index = -1;
  long long idx = -1;
  int st = guarded(c, [&] {
    ck(cudaSetDevice(c->device), "cudaSetDevice");
    double* pack = dbuf<double>(c, B_PACK1, cqr::trisolve_pack_doubles((int)n));
    reset_status(c);
    LAUNCH(c, cqr::launch_pack_r(r_dev, (int)n, (int)n, pack, 0, c->status, c->stream));
    trisolve_dev(c, x, ldx, x, ldx, m, (int)n, pack);
    DevStatus s = read_status(c);
    if (s.code) {
      idx = s.index;
      throw Fail{s.code, s.index, "singular triangular factor"};
    }
  });
  if (index) *index = idx;
  return st;
}

int cqr_trisolve_inplace(cqr_ctx* c, double* x, int64_t m, int64_t n, int64_t ldx, const double* r,
                         int64_t* index) {
  if (!c || n < 1 || n > 512 || ldx < n || m < 0) return CQR_INVALID_ARGUMENT;
  if (index) *index = -1;
  for (int64_t j = 0; j < n; ++j)  // kernels.hpp:106-107: checked before X is touched
    if (r[j * n + j] == 0.0) {
      if (index) *index = j;
      c->err = "singular triangular factor";
      return CQR_SINGULAR_TRIANGULAR;
    }
  return guarded(c, [&] {
    ck(cudaSetDevice(c->device), "cudaSetDevice");
    double* dx = dbuf<double>(c, B_HA, (size_t)std::max<int64_t>(m, 1) * n);
    double* dr = dbuf<double>(c, B_RT, (size_t)n * n);
    double* pack = dbuf<double>(c, B_PACK1, cqr::trisolve_pack_doubles((int)n));
    ck(cudaMemcpyAsync(dr, r, sizeof(double) * n * n, cudaMemcpyHostToDevice, c->stream), "R H2D");
    if (m > 0)
      ck(cudaMemcpy2DAsync(dx, sizeof(double) * n, x, sizeof(double) * ldx, sizeof(double) * n, m,
                           cudaMemcpyHostToDevice, c->stream),
         "X H2D");
    reset_status(c);
    LAUNCH(c, cqr::launch_pack_r(dr, (int)n, (int)n, pack, 0, c->status, c->stream));
    trisolve_dev(c, dx, n, dx, n, m, (int)n, pack);
    DevStatus s = read_status(c);
    if (s.code) throw Fail{s.code, s.index, "singular triangular factor"};
    if (m > 0)
      ck(cudaMemcpy2DAsync(x, sizeof(double) * ldx, dx, sizeof(double) * n, sizeof(double) * n, m,
                           cudaMemcpyDeviceToHost, c->stream),
         "X D2H");
    ck(cudaStreamSynchronize(c->stream), "sync");
  });
}

static int small_factor(cqr_ctx* c, const double* a1, int64_t l, int64_t n, double* out, int64_t* index, bool lu) {
  if (!c || n < 1 || l < n || n > 512) return CQR_INVALID_ARGUMENT;  // kernels.hpp:176, 218
  if (index) *index = -1;
  long long idx = -1;
  int st = guarded(c, [&] {
    ck(cudaSetDevice(c->device), "cudaSetDevice");
    double* da = dbuf<double>(c, B_A1, (size_t)l * n);
    double* dr = dbuf<double>(c, B_RT, (size_t)n * n);
    double* work = dbuf<double>(c, B_WORK, cqr::qr_work_doubles((int)l, (int)n));
    ck(cudaMemcpyAsync(da, a1, sizeof(double) * l * n, cudaMemcpyHostToDevice, c->stream), "A1 H2D");
    reset_status(c);
    if (lu)
      LAUNCH(c, cqr::launch_lu_u(da, (int)l, (int)n, dr, work, c->status, c->stream));
    else
      LAUNCH(c, cqr::launch_qr_r(da, (int)l, (int)n, dr, work, c->status, c->stream));
    DevStatus s = read_status(c);
    if (s.code) {
      idx = s.index;
      throw Fail{s.code, s.index, "singular triangular factor"};
    }
    copy_sync(c, out, dr, sizeof(double) * n * n, cudaMemcpyDeviceToHost, "R D2H");
  });
  if (index) *index = idx;
  return st;
}

int cqr_qr_r_factor(cqr_ctx* c, const double* a1, int64_t l, int64_t n, double* r) {
  return small_factor(c, a1, l, n, r, nullptr, false);
}

int cqr_lu_u_factor(cqr_ctx* c, const double* a1, int64_t l, int64_t n, double* u, int64_t* index) {
  return small_factor(c, a1, l, n, u, index, true);
}

int cqr_sketch_gaussian_dev(cqr_ctx* c, const double* a, int64_t m_local, int64_t m_global, int64_t row0, int64_t n,
                            int64_t lda, int64_t l, uint64_t seed, double* a1_dev) {
  if (!c || n < 1 || n > 512 || l < 1 || lda < n || m_local < 0 || row0 + m_local > m_global)
    return CQR_INVALID_ARGUMENT;
  return guarded(c, [&] {
    ck(cudaSetDevice(c->device), "cudaSetDevice");
    reset_status(c);
    const SketchRun sr = sketch_setup(c, a, lda, m_local, m_global, row0, (int)n, (int)l, 1);
    if (m_local > 0) {
      LAUNCH(c, sketch_launch(c, sr, a, lda, m_global, row0, seed, vec_ok(a, lda, (int)n) ? 1 : 0, 0));
      LAUNCH(c, cqr::launch_sketch_reduce(sr.p, sr.part, a1_dev, c->status, c->stream));
    } else {
      ck(cudaMemsetAsync(a1_dev, 0, sizeof(double) * l * n, c->stream), "memset");
    }
    allreduce(c, a1_dev, (size_t)l * n);
    ck(cudaStreamSynchronize(c->stream), "sync");
  });
}

int cqr_sketch_gaussian(cqr_ctx* c, const double* a, int64_t m, int64_t n, int64_t lda, int64_t l, uint64_t seed,
                        double* a1) {
  if (!c || n < 1 || n > 512 || l < 1 || lda < n || m < 1) return CQR_INVALID_ARGUMENT;
  return guarded(c, [&] {
    ck(cudaSetDevice(c->device), "cudaSetDevice");
    double* da = dbuf<double>(c, B_HA, (size_t)m * n);
    double* d1 = dbuf<double>(c, B_A1, (size_t)l * n);
    ck(cudaMemcpy2DAsync(da, sizeof(double) * n, a, sizeof(double) * lda, sizeof(double) * n, m,
                         cudaMemcpyHostToDevice, c->stream),
       "A H2D");
    reset_status(c);
    const SketchRun sr = sketch_setup(c, da, n, m, m, 0, (int)n, (int)l, 1);
    LAUNCH(c, sketch_launch(c, sr, da, n, m, 0, seed, vec_ok(da, n, (int)n) ? 1 : 0, 0));
    LAUNCH(c, cqr::launch_sketch_reduce(sr.p, sr.part, d1, c->status, c->stream));
    ck(cudaMemcpyAsync(a1, d1, sizeof(double) * l * n, cudaMemcpyDeviceToHost, c->stream), "A1 D2H");
    ck(cudaStreamSynchronize(c->stream), "sync");
  });
}

int cqr_sample_rows_uniform(cqr_ctx* c, const double* a, int64_t m, int64_t n, int64_t lda, int64_t l, uint64_t seed,
                            int without_replacement, double* a1, int64_t* idx) {
  if (!c || n < 1 || l < 1 || lda < n || m < 1) return CQR_INVALID_ARGUMENT;
  return guarded(c, [&] {
    ck(cudaSetDevice(c->device), "cudaSetDevice");
    double* da = dbuf<double>(c, B_HA, (size_t)m * n);
    double* d1 = dbuf<double>(c, B_A1, (size_t)l * n);
    long long* didx = dbuf<long long>(c, B_IDX, (size_t)l);
    long long* dio = dbuf<long long>(c, B_X, (size_t)l);
    ck(cudaMemcpy2DAsync(da, sizeof(double) * n, a, sizeof(double) * lda, sizeof(double) * n, m,
                         cudaMemcpyHostToDevice, c->stream),
       "A H2D");
    const long long* in = nullptr;
    std::vector<long long> h;
    if (without_replacement) {
      require(l <= m, "without replacement needs l <= m");
      std::unordered_set<long long> seen;
      uint64_t pos = 0;
      while ((long long)h.size() < l) {
        const long long i = (long long)(unit_at(seed, pos++) * (double)m);
        if (seen.insert(i).second) h.push_back(i);
      }
      ck(cudaMemcpyAsync(didx, h.data(), sizeof(long long) * l, cudaMemcpyHostToDevice, c->stream), "idx H2D");
      in = didx;
    }
    reset_status(c);
    LAUNCH(c, cqr::launch_gather_rows(da, n, m, m, 0, (int)n, (int)l, seed, in, d1, dio, c->status, c->stream));
    ck(cudaMemcpyAsync(a1, d1, sizeof(double) * l * n, cudaMemcpyDeviceToHost, c->stream), "A1 D2H");
    if (idx) ck(cudaMemcpyAsync(idx, dio, sizeof(long long) * l, cudaMemcpyDeviceToHost, c->stream), "idx D2H");
    ck(cudaStreamSynchronize(c->stream), "sync");
  });
}

int cqr_rng_bits(cqr_ctx* c, uint64_t seed, uint64_t k0, int64_t count, uint64_t* out) {
  if (!c || count < 0) return CQR_INVALID_ARGUMENT;
  return guarded(c, [&] {
    ck(cudaSetDevice(c->device), "cudaSetDevice");
    uint64_t* d = dbuf<uint64_t>(c, B_X, (size_t)std::max<int64_t>(count, 1));
    LAUNCH(c, cqr::launch_rng_bits(seed, k0, count, d, c->stream));
    ck(cudaMemcpyAsync(out, d, sizeof(uint64_t) * count, cudaMemcpyDeviceToHost, c->stream), "D2H");
    ck(cudaStreamSynchronize(c->stream), "sync");
  });
}

int cqr_rng_gaussian(cqr_ctx* c, uint64_t seed, uint64_t k0, int64_t count, double* out) {
  if (!c || count < 0) return CQR_INVALID_ARGUMENT;
  return guarded(c, [&] {
    ck(cudaSetDevice(c->device), "cudaSetDevice");
    double* d = dbuf<double>(c, B_X, (size_t)std::max<int64_t>(count, 1));
    LAUNCH(c, cqr::launch_rng_gaussian(seed, k0, count, d, c->stream));
    ck(cudaMemcpyAsync(out, d, sizeof(double) * count, cudaMemcpyDeviceToHost, c->stream), "D2H");
    ck(cudaStreamSynchronize(c->stream), "sync");
  });
}

int cqr_box_muller_bits(cqr_ctx* c, const uint64_t* bits, int64_t pairs, double* out) {
  if (!c || pairs < 0 || (pairs > 0 && (!bits || !out))) return CQR_INVALID_ARGUMENT;
  return guarded(c, [&] {
    ck(cudaSetDevice(c->device), "cudaSetDevice");
    const size_t cnt = (size_t)std::max<int64_t>(2 * pairs, 1);
    uint64_t* db = dbuf<uint64_t>(c, B_SYN, cnt);
    double* d = dbuf<double>(c, B_X, cnt);
    ck(cudaMemcpyAsync(db, bits, sizeof(uint64_t) * 2 * pairs, cudaMemcpyHostToDevice, c->stream), "H2D");
    LAUNCH(c, cqr::launch_box_muller_bits(db, pairs, d, c->stream));
    ck(cudaMemcpyAsync(out, d, sizeof(double) * 2 * pairs, cudaMemcpyDeviceToHost, c->stream), "D2H");
    ck(cudaStreamSynchronize(c->stream), "sync");
  });
}

int cqr_orthogonality_error_dev(cqr_ctx* c, const double* q, int64_t m, int64_t n, int64_t ldq, double* out) {
  if (!c || m < n || n < 1 || n > 512) return CQR_INVALID_ARGUMENT;
  return guarded(c, [&] {
    ck(cudaSetDevice(c->device), "cudaSetDevice");
    reset_status(c);
    double* g = dbuf<double>(c, B_DIAG, (size_t)n * n + 2);
    gram_dev(c, q, m, (int)n, ldq, g);
    double* o = g + (size_t)n * n;
    LAUNCH(c, cqr::launch_orth_from_gram(g, (int)n, o, c->stream));
    ck(cudaMemcpyAsync(c->scal_h, o, sizeof(double), cudaMemcpyDeviceToHost, c->stream), "D2H");
    ck(cudaStreamSynchronize(c->stream), "sync");
    *out = c->scal_h[0];
  });
}

int cqr_residual_error_dev(cqr_ctx* c, const double* a, int64_t lda, const double* q, int64_t ldq,
                           const double* r_host, int64_t m, int64_t n, double* out) {
  if (!c || m < 1 || n < 1) return CQR_INVALID_ARGUMENT;
  return guarded(c, [&] {
    ck(cudaSetDevice(c->device), "cudaSetDevice");
    const int nb = c->num_sms * 4;
    double* dr = dbuf<double>(c, B_DIAG, (size_t)n * n + 2 * nb + 2);
    double* part = dr + (size_t)n * n;
    double* o = part + 2 * nb;
    ck(cudaMemcpyAsync(dr, r_host, sizeof(double) * n * n, cudaMemcpyHostToDevice, c->stream), "R H2D");
    LAUNCH(c, cqr::launch_residual(a, lda, q, ldq, dr, m, (int)n, part, nb, o, c->stream));
    ++c->launches;
    allreduce(c, o, 2);
    ck(cudaMemcpyAsync(c->scal_h, o, 2 * sizeof(double), cudaMemcpyDeviceToHost, c->stream), "D2H");
    ck(cudaStreamSynchronize(c->stream), "sync");
    *out = std::sqrt(c->scal_h[0]) / std::sqrt(c->scal_h[1]);
  });
}

// matgen.cpp:21-46 on the device: A = U diag(sigma) V^T with U = random_orthogonal(m, n,
// derive(seed, 0)) rows [row0, row0 + m_local) and V = random_orthogonal(n, n, derive(seed, 1)), where
// random_orthogonal (matgen.cpp:12-19) is the thin Householder Q of gaussian_matrix(rows, cols, seed) with
// the signs Householder leaves (global counters; the tall Householder's column reductions are summed over
// the ranks when a communicator is attached). The same matrix as the reference's synthesize up to rounding.
int cqr_synthesize_dev(cqr_ctx* c, int64_t m_local, int64_t m_global, int64_t row0, int64_t n, const double* sigma,
                       uint64_t seed, double* a, int64_t lda) {
  if (!c || n < 1 || n > 512 || m_global < n || m_local < 0 || row0 + m_local > m_global || lda < n || !sigma)
    return CQR_INVALID_ARGUMENT;
  if (!attached(c) && (m_local != m_global || row0 != 0)) {
    c->err = "sharded call without an attached communicator";
    return CQR_INVALID_ARGUMENT;
  }
  return guarded(c, [&] {
    ck(cudaSetDevice(c->device), "cudaSetDevice");
    reset_status(c);
    const size_t rows = (size_t)std::max<int64_t>(m_local, 1);
    double* g = dbuf<double>(c, B_SYN, rows * n);    // the Gaussian, then its reflectors
    double* u = dbuf<double>(c, B_HHW, rows * n);    // U
    double* v = dbuf<double>(c, B_SYNV, (size_t)n * n * 4);
    double* gv = v + (size_t)n * n;
    double* rr = gv + (size_t)n * n;                  // R of the factorizations (not used)
    // U (matgen.cpp:41): rows [row0, row0 + m_local) of gaussian_matrix(m, n, derive(seed, 0))
    if (m_local > 0)
      LAUNCH(c, cqr::launch_rng_gaussian(derive(seed, 0), (uint64_t)row0 * n, m_local * n, g, c->stream));
    HhWs w = hh_ws(c, m_local, (int)n);
    hh_factor(c, g, n, m_local, row0, (int)n, rr, w);
    hh_form_q(c, g, n, u, n, m_local, row0, (int)n, w);
    // V (matgen.cpp:35): n x n, replicated on every rank
    LAUNCH(c, cqr::launch_rng_gaussian(derive(seed, 1), 0, n * n, gv, c->stream));
    c->local_only = 1;
    try {
      HhWs wv = hh_ws(c, n, (int)n);
      hh_factor(c, gv, n, n, 0, (int)n, rr, wv);
      hh_form_q(c, gv, n, v, n, n, 0, (int)n, wv);
    } catch (...) {
      c->local_only = 0;
      throw;
    }
    c->local_only = 0;
    std::vector<double> hv((size_t)n * n), svt((size_t)n * n);
    copy_sync(c, hv.data(), v, sizeof(double) * n * n, cudaMemcpyDeviceToHost, "V D2H");
    for (int64_t i = 0; i < n; ++i)  // svt = diag(sigma) V^T (matgen.cpp:36)
      for (int64_t jj = 0; jj < n; ++jj) svt[(size_t)(i * n + jj)] = sigma[i] * hv[(size_t)(jj * n + i)];
    double* b = v + (size_t)3 * n * n;
    copy_sync(c, b, svt.data(), sizeof(double) * n * n, cudaMemcpyHostToDevice, "SVt H2D");
    if (m_local > 0) LAUNCH(c, cqr::launch_gemm_tall(u, n, b, a, lda, m_local, (int)n, c->num_sms, c->stream));
    DevStatus s = read_status(c);
    if (s.code) throw Fail{s.code, s.index, "matgen failed"};
    c->stage_evs.clear();
    c->ev_used = 0;
  });
}

int64_t cqr_block_offset(int64_t m, int p, int b) {  // parexec.cpp:13-15
  if (b <= 0) return 0;
  if (b >= p) return m;
  return (static_cast<int64_t>(b) * m + p - 1) / p;
}

int cqr_comm_model(int method, int p, int64_t n, int64_t l, int* rounds_min, int* rounds_max, double* volume_min,
                   double* volume_max) {  // parexec.cpp:44-62
  const double pn2 = (double)p * (double)n * (double)n;
  const double nl = (double)n * (double)l;
  int a = 0, b = 0;
  double x = 0, y = 0;
  switch (method) {
    case CQR_CHOLQR: a = b = 2; x = y = pn2; break;
    case CQR_CHOLQR2: a = b = 4; x = y = 2 * pn2; break;
    case CQR_SCHOLQR3: a = b = 6; x = y = 3 * pn2; break;
    case CQR_RLU:
    case CQR_RQR:
    case CQR_RQR_GAUSSIAN: a = 3; b = 4; x = 1.5 * pn2; y = 1.5 * pn2 + nl; break;
    case CQR_HOUSEHOLDER: break;
    default: return CQR_INVALID_ARGUMENT;
  }
  if (rounds_min) *rounds_min = a;
  if (rounds_max) *rounds_max = b;
  if (volume_min) *volume_min = x;
  if (volume_max) *volume_max = y;
  return CQR_OK;
}

}  // extern "C"
