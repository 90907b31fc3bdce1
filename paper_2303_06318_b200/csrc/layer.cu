// layer.cu -- one rank's TED MoE layer: the B200-native MoeRank MoE branch.
//
// Forward  (MoeRank::forward_layer, moe.cpp:435-563):
//   gate -> capacity scan -> [DTD chunk] dispatch -> EP all-to-all + [DTD TP all-gather]
//   -> GEMM1+bias+GELU -> GEMM2+bias -> [TP all-reduce] + return all-to-all + [DTD home
//   all-gather] -> combine.  On more than one GPU the bracketed collectives are NVLink
//   peer-memory kernels (peer_kernels.cu: one scatter, one pull that also sums the TP
//   partials) ordered by plane barriers; the exchange plan is built on the device, so the
//   step has no host round trip and ted_layer_step replays it as a CUDA graph.
//   TED_EXCHANGE=nccl keeps the NCCL send/recv + all-gather + all-reduce version.
// Backward (MoeRank::backward_layer, moe.cpp:582-686): the mirror image, with dgrad
//   GEMMs (dGELU and the db1 column sums fused), wgrad GEMMs written straight into the
//   flat expert family -- or, when the optimizer step follows and the family is
//   unsharded, with AdamW fused into their epilogues -- bias column sums, gate backward.
// Optimizer (run_grad_sync / family_optimizer_step, moe.cpp:699-741): DP all-reduce of
//   each family, AdamW over the ZeRO-1 owned range, completion all-gather.
// Communicators: one per TED group family (ncclCommSplit of the world communicator,
// colours from topology.cpp:56-93) plus the EP x TP plane of each data replica.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <chrono>
#include <cmath>
#include <cstdio>
#include <thread>
#include <cstdlib>
#include <cstring>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/ted.h"
#include "ted_host.h"
#include "ted_internal.h"
#include "ted_plan.h"

namespace ted {


}  // namespace ted

using namespace ted;

struct ted_layer {
  // configuration
  ted_model_cfg model{};
  ted_topo_cfg topo{};
  ted_flags flags{};
  ted_adam_cfg adam{};
  ted_tile_cfg tiles{};
  double cf = 0.0;
  int shard_opt = 1;
  int rank = 0, world = 1;
  int T = 1, P = 1, D = 1;  // tensor, expert-parallel, expert-data degrees
  int t = 0, ep = 0, d = 0;
  int n = 0, h = 0, E = 0, f = 0, fT = 0, Eloc = 1, Tc = 1;
  // Shapes below the tensor-core tiles (the reference's own verify sweep runs hidden = 8):
  // the layer computes on h and fT zero-padded to multiples of 256 (padded weight rows /
  // columns, biases and optimizer state stay exactly zero, so every result is the
  // unpadded one); hu / fTu are the reference's shapes, io_h the width of the caller's
  // token buffers (hu for ted_layer_create, the padded h inside a padded model stack).
  int hu = 0, fTu = 0, io_h = 0;
  DevBuf<bf16> pad_a, pad_y, pad_dy, pad_da;  // [n][h] staging when io_h != h
  bool dtd = false, local = true;
  int64_t cap = 0;
  int my_chunk = -1;
  int nblk = 0;
  int64_t R_max = 0;

  // comms
  ncclComm_t world_c = nullptr, tp_c = nullptr, ep_c = nullptr, expdp_c = nullptr,
             nonexpdp_c = nullptr, plane_c = nullptr;  // plane = TP x EP ranks of one d

  // peer-memory exchange: IPC mappings of every plane rank's assembled buffers
  bool direct = false;
  int plane_rank = 0, plane_size = 1;
  DevBuf<unsigned long long> peer_tab;  // [5][plane]: x_asm, dfe_asm, fe_asm, dx_asm, flags
  std::vector<void*> ipc_opened;
  DevBuf<long long> disp_base;  // [E] dispatch rows, then [Tc][E] pull rows
  HostBuf<long long> h_tabs;
  DevBuf<int> bar;
  DevBuf<unsigned> bar_flags;  // plane barrier: slot r written by plane member r (IPC-mapped)
  DevBuf<unsigned> bar_epoch;  // device barrier epoch (advances on graph replays too)
  bool nccl_barrier = false;
  // failure detection (TrainerOptions::collective_timeout, moe.hpp:96; Fabric's
  // TimeoutError, fabric.cpp:65-96): the plane barrier records a missing member in a
  // host-mapped word instead of trapping; host-side waits poll it and NCCL's async errors
  // and abort the communicators on timeout.  A faulted layer fails every later call.
  int* fault_h = nullptr;  // host view (mapped pinned memory)
  int* fault_d = nullptr;  // device view
  double timeout_s = 120.0;
  std::string poisoned;
  // the reference's CommLedger (ledger.hpp:46-77) of this rank: [phase][op][calls, bytes],
  // phases Forward, Recompute, Backward, GradSync, Optim, ops AllReduce, AllGather,
  // AllToAll (types.hpp:32-40).  The routing-dependent MoE entries accumulate on the
  // device (one tiny kernel per pass, graph-safe), the static ones on the host.
  DevBuf<unsigned long long> led;
  unsigned long long led_host[5][3][2] = {};
  int ledger_phase = 0;  // Forward, or Recompute while a model stack recomputes
  // peer exchange with the plan built on the device (no host round trip per step, so the
  // multi-GPU step is graph-capturable); the host plan is rebuilt lazily for statistics
  bool devplan = false;
  // push return (device plan only): GEMM2 / dgrad1 epilogues store their TP-partial output
  // rows straight into the home ranks' receive slots (ret: [T][n][h], IPC-mapped, peer
  // table 5) over NVLink, overlapped with the GEMM; the combine / gate-dx then read and sum
  // the T slots locally.  row_home / row_src map assembled rows to home rows / shards.
  bool push = false;
  DevBuf<bf16> ret;
  DevBuf<int> row_home, row_src;

  // parameters: expert family (local experts: w1,b1,w2,b2 each) + non-expert (gate)
  Family fam_exp, fam_non;
  int64_t per_expert = 0, off_w1 = 0, off_b1 = 0, off_w2 = 0, off_b2 = 0;

  // routing
  DevBuf<float> logits, probs, prob, loss_part, dlogits, gate_part, col_part;
  DevBuf<bf16> wgT;  // the gate weight transposed for the L1-resident gate kernel
  DevBuf<int> expert, slot, pos_send, pos_home, blk_hist, blk_prefix, chunk_prefix, kc, kc_all,
      send_base, home_base, seg_off;
  int* seg_valid_view = nullptr;  // [Eloc] view inside seg_off's allocation
  DevBuf<double> loss;
  DevBuf<int> verdict;  // placement verdict: [0] last forward, [1] sticky (moe.cpp:537-556)
  HostBuf<int> h_kc_all, h_seg;
  HostBuf<double> h_loss;
  // activations
  DevBuf<bf16> x_asm, z, hbuf, fe_asm, xsend, fhome, dfe_send, dfe_asm, dx_home, dx_asm;
  ted_layer* share = nullptr;     // activation buffers borrowed from this layer (ckpt)
  int fwd_mode = FWD_LIVE;        // LIVE / RECORD / REPLAY (CAC)
  DevBuf<bf16> stash_x, stash_f;  // CAC stash: assembled rows, combined home rows
  int64_t stash_rows = 0;
  const bf16* last_a = nullptr;
  const bf16* last_y = nullptr;
  LayerPlan plan;
  int64_t last_dropped = 0;
  bool have_forward = false;

  // the stream ted_layer_step forks onto (and captures its CUDA graph on)
  cudaStream_t hs = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  // step_follows: the optimizer step follows this backward (ted_layer_step / a model step),
  // so the expert family's AdamW may run inside the wgrad epilogues (exp_done_fused)
  bool step_follows = false, exp_done_fused = false;
  bool fuse_ok = false;  // expert family unsharded, no DP sync: AdamW may fuse into wgrad
  // the fused epilogues write the updated parameters; the bf16 expert weight gradients are
  // stored too only with keep_grads (ted_layer_keep_grads), else get_grad of w1/w2 fails
  // until the next unfused backward (grads_stale)
  bool keep_grads = false, grads_stale = false;

  // CUDA graph of the whole single-rank training step (ted_layer_step): the step has no
  // host synchronisation, so it is captured once and replayed (removes ~45 launches and
  // 24 tensor-map encodes of host work per step).
  bool use_graph = true, capturing = false;
  struct Graph {
    cudaGraphExec_t exec = nullptr;
    const void *a = nullptr, *y = nullptr, *da = nullptr;
    unsigned long long launches = 0;
    std::vector<cudaEvent_t> evs;  // timing event nodes (timed graph only)
    std::vector<const char*> names;
    unsigned long long used = 0;  // last use (LRU among the cached graphs)
  };
  // one graph per (input, output, input-gradient) buffer triple, so callers that double
  // buffer their inputs (H2D of step i+1 under step i) replay without re-capturing
  static constexpr int kGraphs = 4;
  Graph graphs[kGraphs];
  unsigned long long graph_clock = 0;

  // live per-stage timing (CUDA events on the launching stream)
  bool timing = false;
  std::vector<cudaEvent_t> evs;
  std::vector<const char*> ev_names;
  size_t ev_used = 0;
  std::map<std::string, double> stage_ms;
  std::map<std::string, int64_t> stage_cnt;

  void mark(const char* name, cudaStream_t s) {
    if (!timing) return;
    if (ev_used == evs.size()) {
      cudaEvent_t e;
      CU(cudaEventCreate(&e));
      evs.push_back(e);
      ev_names.push_back(nullptr);
    }
    CU(cudaEventRecord(evs[ev_used], s));
    ev_names[ev_used] = name;
    ++ev_used;
  }
};

namespace {
void graph_reset(ted_layer::Graph& g);
}

namespace ted {
thread_local std::string g_err;
void set_error(const std::string& m) { g_err = m; }
const char* last_error() { return g_err.c_str(); }
}  // namespace ted

namespace {


// --------------------------------------------------------------- parameters
struct ParamLoc {
  Family* fam;
  int64_t off;       // element offset of the local shard in the family
  int64_t rows, cols;  // local shard shape (rows=1 for vectors), the reference's shape
  int64_t full_rows, full_cols;
  int axis;  // 0 none, 1 column, 2 row
  double scale;
  int64_t ld;  // row stride in the family (>= cols: zero-padded columns)
};

bool lookup(ted_layer* L, const std::string& name, ParamLoc& out) {
  if (name == "layer0.gate.w") {
    out = {&L->fam_non, 0, L->hu, L->E, L->hu, L->E, 0, 1.0 / std::sqrt(double(L->hu)), L->E};
    return true;
  }
  const std::string pre = "layer0.expert";
  if (name.compare(0, pre.size(), pre) != 0) return false;
  size_t dot = name.find('.', pre.size());
  if (dot == std::string::npos) return false;
  const int e = std::stoi(name.substr(pre.size(), dot - pre.size()));
  const std::string leaf = name.substr(dot + 1);
  if (e < 0 || e >= L->E) return false;
  if (e / L->Eloc != L->ep) return false;  // not housed on this rank
  const int le = e % L->Eloc;
  const int64_t base = int64_t(le) * L->per_expert;
  const double sin = 1.0 / std::sqrt(double(L->hu)), sout = 1.0 / std::sqrt(double(L->f));
  const int hu = L->hu, fTu = L->fTu;
  if (leaf == "w1") out = {&L->fam_exp, base + L->off_w1, hu, fTu, hu, L->f, 1, sin, L->fT};
  else if (leaf == "b1") out = {&L->fam_exp, base + L->off_b1, 1, fTu, 1, L->f, 1, 0.1, L->fT};
  else if (leaf == "w2") out = {&L->fam_exp, base + L->off_w2, fTu, hu, L->f, hu, 2, sout, L->h};
  else if (leaf == "b2") out = {&L->fam_exp, base + L->off_b2, 1, hu, 1, hu, 0, 0.1, L->h};
  else return false;
  return true;
}

// expert weight matrices whose optimizer state uses the blk_off layout
bool state_blocked(const ted_layer* L, const ParamLoc& pl) {
  return L->fam_exp.blocked && pl.fam == &L->fam_exp && pl.rows > 1;
}


__global__ void init_family_kernel(bf16* param, float* master, int64_t begin, int64_t end,
                                   int64_t off, int64_t rows, int64_t cols, int64_t ld,
                                   int64_t full_cols, int64_t col0, uint64_t seed, float scale,
                                   int blocked) {
  const int64_t n = rows * cols;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = i / cols, c = i % cols;
    uint64_t z = seed + 0x9E3779B97F4A7C15ULL * uint64_t(r * full_cols + col0 + c + 1);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    z ^= z >> 31;
    const float u = float(z >> 40) * (1.0f / 16777216.0f);
    const float v = (2.f * u - 1.f) * scale;
    const int64_t fi = off + r * ld + c;  // padded columns (c >= cols) stay zero
    param[fi] = __float2bfloat16(v);
    if (blocked) master[off + blk_off(r, c, ld)] = v;  // unsharded family (begin == 0)
    else if (fi >= begin && fi < end) master[fi - begin] = v;
  }
}

void setup_family(ted_layer* L, Family& F, int64_t elems, ncclComm_t dp, int group, int pos) {
  F.elems = elems;
  F.group = L->shard_opt ? group : 1;
  F.pos = L->shard_opt ? pos : 0;
  F.dp = dp;
  F.begin = shard_lo(elems, F.group, F.pos);
  F.end = shard_lo(elems, F.group, F.pos + 1);
  F.chunk = (elems + F.group - 1) / F.group;
  // 8-element padding keeps every vector access aligned
  F.param.alloc(size_t(elems + 8));
  F.param.zero();
  F.grad.alloc(size_t(elems + 8));
  F.grad.zero();
  const size_t owned = size_t(F.end - F.begin);
  F.master.alloc(owned + 4);
  F.master.zero();
  F.m1.alloc(owned + 4);
  F.m1.zero();
  F.m2.alloc(owned + 4);
  F.m2.zero();
  if (F.group > 1) F.gather.alloc(size_t(F.chunk) * F.group + 8);
  F.dstep.alloc(1);
  F.dstep.zero();
  F.dcoef.alloc(2);
}

// --------------------------------------------------------------- NCCL helpers
void grouped_p2p(const std::vector<PeerXfer>& sends, const bf16* sbuf,
                 const std::vector<PeerXfer>& recvs, bf16* rbuf, int64_t h, ncclComm_t comm,
                 cudaStream_t s) {
  if (sends.empty() && recvs.empty()) return;
  NC(ncclGroupStart());
  for (const auto& x : sends)
    NC(ncclSend(sbuf + x.row * h, size_t(x.rows * h), ncclBfloat16, x.peer, comm, s));
  for (const auto& x : recvs)
    NC(ncclRecv(rbuf + x.row * h, size_t(x.rows * h), ncclBfloat16, x.peer, comm, s));
  NC(ncclGroupEnd());
}

// send-side rows (home layout, my chunk) <-> assembled rows, both directions.
void a2a_dispatch(ted_layer* L, const bf16* send_rows, bf16* asm_rows, cudaStream_t s) {
  grouped_p2p(L->plan.a2a_send, send_rows, L->plan.a2a_recv, asm_rows, L->h, L->ep_c, s);
}
void a2a_return(ted_layer* L, const bf16* asm_rows, bf16* home_rows, cudaStream_t s) {
  // the inverse exchange: what I received goes back to its source, into my home chunk
  std::vector<PeerXfer> recv = L->plan.a2a_send;
  const int64_t base = L->plan.chunk_row[L->dtd ? L->t : 0];
  for (auto& x : recv) x.row += base;
  grouped_p2p(L->plan.a2a_recv, asm_rows, recv, home_rows, L->h, L->ep_c, s);
}

// stream-ordered barrier over the TP x EP plane (all writers' kernels are fenced)
void plane_barrier(ted_layer* L, cudaStream_t s) {
  if (L->nccl_barrier) {  // TED_BARRIER=nccl: stream-ordered 1-int all-reduce
    NC(ncclAllReduce(L->bar.p, L->bar.p, 1, ncclInt32, ncclSum, L->plane_c, s));
    return;
  }
  check(plane_barrier_peer(L->peer_tab.p + size_t(4) * L->plane_size, L->plane_size,
                           L->plane_rank, L->bar_epoch.p, L->fault_d,
                           (unsigned long long)(L->timeout_s * 1e9), s),
        "plane_barrier_peer");
}

void abort_comms(ted_layer* L) {
  for (ncclComm_t* c : {&L->tp_c, &L->ep_c, &L->expdp_c, &L->nonexpdp_c, &L->plane_c,
                        &L->world_c})
    if (*c) {
      ncclCommAbort(*c);
      *c = nullptr;
    }
}

[[noreturn]] void poison(ted_layer* L, const std::string& why) {
  L->poisoned = why;
  abort_comms(L);
  throw RuntimeError(why);
}

// the layer's failure state: a faulted earlier call, a plane-barrier timeout recorded by
// the device, or an asynchronous NCCL error
void check_fault(ted_layer* L) {
  if (!L->poisoned.empty()) throw RuntimeError(L->poisoned + " (layer unusable after the failure)");
  const int f = L->fault_h ? *reinterpret_cast<volatile int*>(L->fault_h) : 0;
  if (f != 0) {
    char buf[256];
    std::snprintf(buf, sizeof(buf),
                  "TimeoutError: plane barrier of rank %d: member %d of the EP x TP plane did not "
                  "arrive within %.1f s (collective_timeout)",
                  L->rank, f - 1, L->timeout_s);
    poison(L, buf);
  }
  for (ncclComm_t c : {L->tp_c, L->ep_c, L->expdp_c, L->nonexpdp_c, L->plane_c, L->world_c}) {
    if (!c) continue;
    ncclResult_t r = ncclSuccess;
    if (ncclCommGetAsyncError(c, &r) == ncclSuccess && r != ncclSuccess && r != ncclInProgress)
      poison(L, std::string("NCCL asynchronous error: ") + ncclGetErrorString(r));
  }
}

// stream synchronisation that cannot hang: polls the stream, the fault word and NCCL's
// async errors; past the timeout the communicators are aborted (TimeoutError, status 1)
void wait_stream(ted_layer* L, cudaStream_t s) {
  const auto t0 = std::chrono::steady_clock::now();
  for (;;) {
    const cudaError_t q = cudaStreamQuery(s);
    if (q == cudaSuccess) break;
    if (q != cudaErrorNotReady) CU(q);
    check_fault(L);
    const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (L->timeout_s > 0 && el > L->timeout_s && L->world > 1)
      poison(L, "TimeoutError: rank " + std::to_string(L->rank) + ": the step did not complete within " +
                    std::to_string(L->timeout_s) + " s (a peer is stalled or gone; collective_timeout)");
    std::this_thread::sleep_for(std::chrono::microseconds(50));
  }
  check_fault(L);
}

// ledger entries of this pass's MoE collectives (see ledger_moe_pass_kernel)
void ledger_pass(ted_layer* L, int phase, cudaStream_t s) {
  if (L->local) return;
  check(ledger_moe_pass(L->led.p, phase, L->P, L->T, L->dtd ? 1 : 0, L->Tc, L->E, L->Eloc, L->t,
                        L->ep, L->kc.p, L->kc_all.p, L->direct ? L->T : 1, L->seg_valid_view,
                        L->hu, s),
        "ledger_moe_pass");
}

// grad sync + ZeRO-1 completion entries (static sizes, moe.cpp:699-734)
void ledger_host_optim(ted_layer* L) {
  // the reference's family sizes (zero padding of small shapes excluded)
  const int64_t exp_u = int64_t(L->Eloc) * (2 * int64_t(L->hu) * L->fTu + L->fTu + L->hu);
  const int64_t non_u = int64_t(L->hu) * L->E;
  auto add = [&](int phase, int op, int64_t elems) {
    L->led_host[phase][op][0] += 1;
    L->led_host[phase][op][1] += uint64_t(elems) * 2;
  };
  if (L->D > 1) add(3, 0, exp_u);
  if (L->P * L->D > 1) add(3, 0, non_u);
  if (L->fam_exp.group > 1) add(4, 1, (exp_u + L->fam_exp.group - 1) / L->fam_exp.group);
  if (L->fam_non.group > 1) add(4, 1, (non_u + L->fam_non.group - 1) / L->fam_non.group);
}

const unsigned long long* peer_table(ted_layer* L, int which) {
  return L->peer_tab.p + size_t(which) * L->plane_size;
}

// Destination / source row bases of this rank's blocks inside every expert rank's
// assembled buffer (all ranks hold all counts, so every rank can lay out every peer).
void build_peer_tables(ted_layer* L, const int* cnt) {
  const int E = L->E, Tc = L->Tc, P = L->P, Eloc = L->Eloc;
  const int my_c = L->dtd ? L->t : 0;
  long long* tab = L->h_tabs.p;  // [E] disp, then [Tc][E] pull
  for (int ep2 = 0; ep2 < P; ++ep2) {
    const LayerPlan pl = build_plan(P, L->T, E, L->dtd, ep2, 0, cnt);
    for (int le = 0; le < Eloc; ++le) {
      const int e = ep2 * Eloc + le;
      tab[e] = pl.blk_row[(size_t(le) * Tc + my_c) * P + L->ep];
      for (int c = 0; c < Tc; ++c)
        tab[E + c * E + e] = pl.blk_row[(size_t(le) * Tc + c) * P + L->ep];
    }
  }
}

// rows the assembled buffers span this step (the device-plan path does not know them on
// the host: the whole workspace, the GEMMs schedule tiles from the device segments)
int64_t asm_rows_bound(const ted_layer* L) {
  return (L->direct && L->devplan) ? L->R_max : std::max<int64_t>(L->plan.asm_rows, 128);
}

void zero_asm_pads(ted_layer* L, bf16* buf, cudaStream_t s) {
  int maxpad = 0;
  if (L->direct && L->devplan) maxpad = kPad - 1;
  else
    for (int le = 0; le < L->Eloc; ++le)
      maxpad = std::max(maxpad, L->plan.seg_off[le + 1] - L->plan.seg_off[le] - L->plan.seg_rows[le]);
  if (maxpad > 0)
    check(zero_pad_rows(buf, L->h, L->h, L->seg_off.p, L->seg_valid_view, L->Eloc, maxpad, s),
          "zero_pad_rows");
}


// corrupt_drop on the peer exchange: my rows go to my slot's blocks, sized for my slot's
// chunk, not for the chunk the fault hook dispatches
const int* peer_clamp(const ted_layer* L) {
  return (L->dtd && L->flags.corrupt_drop) ? L->kc.p + size_t(L->t) * L->E : nullptr;
}

// push return: the epilogue's destination (receive slots of the home shard's TP members)
void set_push(ted_layer* L, GemmParams& g) {
  g.push_peers = peer_table(L, 5);
  g.row_home = L->row_home.p;
  g.row_src = L->row_src.p;
  g.push_T = L->T;
  g.push_slot = L->t;
  g.push_slot_stride = int64_t(L->n) * L->h;
}

// the T pushed partial rows of every token, in this rank's receive slots
RowSrc ret_src(ted_layer* L) {
  RowSrc r;
  r.local = L->ret.p;
  r.pos_home = L->pos_home.p;
  r.slot_stride = int64_t(L->n) * L->h;
  r.nsum = L->T;
  return r;
}

RowSrc pull_src(ted_layer* L, int which) {
  RowSrc r;
  r.pos_home = L->pos_home.p;
  r.peers = peer_table(L, which);
  r.pull_base = L->disp_base.p + L->E;
  r.home_base = L->home_base.p;
  r.expert = L->expert.p;
  r.chunk_len = L->n / L->Tc;
  r.Tc = L->Tc;
  r.E = L->E;
  r.Eloc = L->Eloc;
  r.Tp = L->T;
  r.my_t = L->t;
  return r;
}

// --------------------------------------------------------------- forward
// Z = X W1 + b1, H = gelu(Z) over the assembled rows (column_parallel_forward + gelu,
// parallel_linear.cpp:8-11, nn.cpp:108-112); leaves g / o set up for GEMM2
void expert_gemm1(ted_layer* L, int64_t rows, cudaStream_t s, GemmParams& g, GemmOperands& o) {
  bf16* P = L->fam_exp.param.p;
  g = GemmParams{};
  g.mode = GEMM_ROWS;
  g.groups = L->Eloc;
  g.seg_off = L->seg_off.p;
  o = GemmOperands{};
  o.A = L->x_asm.p;
  o.lda = L->h;
  o.a_mn = false;
  o.B = P + L->off_w1;
  o.ldb = L->fT;
  o.b_group_stride = L->per_expert;
  o.b_mn = true;
  L->mark("gemm1_fwd", s);
  g.epi = EPI_BIAS_GELU;
  g.M = 0;
  g.N = L->fT;
  g.K = L->h;
  g.C = L->z.p;
  g.ldc = L->fT;
  g.bias = P + L->off_b1;
  g.bias_group_stride = L->per_expert;
  g.aux = L->hbuf.p;
  g.ld_aux = L->fT;
  run_gemm(o, g, rows, s);
}

void stash_alloc(ted_layer* L) {
  if (L->stash_x.n == 0) {
    L->stash_x.alloc(size_t(L->R_max) * L->h);
    L->stash_f.alloc(size_t(L->n) * L->h);
  }
}

// CAC recompute (Mode::Replay, channel.cpp:37-51): the routing state of the recorded
// forward is still in place; the collectives' outputs come from the stash, so only the
// local math the backward reads (Z and H of GEMM1) is recomputed
void layer_forward_replay(ted_layer* L, const bf16* a, cudaStream_t s) {
  require(L->stash_x.n != 0, "CAC replay without a recorded forward");
  L->last_a = a;
  const int64_t rows = L->stash_rows;
  check(cudaMemcpyAsync(L->x_asm.p, L->stash_x.p, sizeof(bf16) * size_t(rows) * L->h,
                        cudaMemcpyDeviceToDevice, s),
        "replay");
  GemmParams g{};
  GemmOperands o{};
  expert_gemm1(L, rows, s, g, o);
  check(cudaMemcpyAsync(L->fhome.p, L->stash_f.p, sizeof(bf16) * size_t(L->n) * L->h,
                        cudaMemcpyDeviceToDevice, s),
        "replay");
  L->mark("_end", s);
  L->have_forward = true;
}

void layer_forward_impl(ted_layer* L, const bf16* a, bf16* y, cudaStream_t s) {
  if (L->fwd_mode == FWD_REPLAY && !L->local) {
    layer_forward_replay(L, a, s);
    return;
  }
  const int h = L->h, E = L->E;
  L->last_a = a;
  L->last_y = y;
  const bf16* wg = L->fam_non.param.p;
  L->mark("gate", s);
  check(gate_forward(a, wg, L->n, h, E, L->logits.p, L->probs.p, L->expert.p, L->prob.p,
                     L->blk_hist.p, L->wgT.n ? L->wgT.p : nullptr, s),
        "gate_forward");
  L->mark("route_dispatch", s);
  RouteScanArgs ra{};
  ra.n = L->n;
  ra.E = E;
  ra.T = L->Tc;
  ra.my_chunk = L->my_chunk;
  ra.cap = L->cap;
  ra.local = L->local ? 1 : 0;
  ra.expert = L->expert.p;
  ra.blk_hist = L->blk_hist.p;
  ra.blk_prefix = L->blk_prefix.p;
  ra.chunk_prefix = L->chunk_prefix.p;
  ra.kc = L->kc.p;
  ra.send_base = L->send_base.p;
  ra.home_base = L->home_base.p;
  ra.seg_off = L->seg_off.p;
  check(route_scan(ra, s), "route_scan");
  bf16* xs = L->local ? L->x_asm.p : (L->direct ? nullptr : L->xsend.p);
  check(dispatch_rows(a, L->n, h, E, L->Tc, L->my_chunk, L->cap, L->expert.p, L->blk_prefix.p,
                      L->chunk_prefix.p, L->send_base.p, L->home_base.p, L->slot.p,
                      L->pos_send.p, L->pos_home.p, xs, s),
        "dispatch_rows");
  // the DTD round trip's placement verdict, from the rows the dispatch actually selected
  check(placement_verdict(L->pos_send.p, L->pos_home.p, L->n, L->Tc, L->dtd ? L->t : -1,
                          L->verdict.p, s),
        "placement_verdict");

  int64_t rows = 0;  // rows spanned by the assembled buffer
  if (L->local) {
    // device-resident segment table; valid counts = kc row 0
    check(cudaMemcpyAsync(L->seg_valid_view, L->kc.p, sizeof(int) * E, cudaMemcpyDeviceToDevice, s),
          "memcpy");
    // pad rows: at most 127 per expert
    check(zero_pad_rows(L->x_asm.p, h, h, L->seg_off.p, L->seg_valid_view, E, kPad, s), "zero_pad");
    rows = L->R_max;
  } else if (L->direct && L->devplan) {
    L->mark("count_exchange", s);
    // chunk counts over the plane (the reference's A2A metadata, fabric.cpp:282-285; also
    // orders this step's peer writes after every peer's previous-step reads), then the
    // exchange plan on the device
    const size_t nc = size_t(L->Tc) * E;
    NC(ncclAllGather(L->kc.p, L->kc_all.p, nc, ncclInt32, L->plane_c, s));
    check(plan_peer(L->kc_all.p, L->T, L->P, E, L->Tc, L->ep, L->dtd ? L->t : 0, L->seg_off.p,
                    L->disp_base.p, L->disp_base.p + E, s),
          "plan_peer");
    if (L->push)
      check(push_map(L->kc_all.p, L->T, L->P, E, L->Tc, L->ep, L->seg_off.p, L->row_home.p,
                     L->row_src.p, s),
            "push_map");
    PeerDst pd;
    pd.peers = peer_table(L, 0);
    pd.disp_base = L->disp_base.p;
    pd.send_base = L->send_base.p;
    pd.Eloc = L->Eloc;
    pd.Tp = L->T;
    pd.my_t = L->t;
    pd.all_replicas = L->dtd ? 1 : 0;
    pd.clamp_rows = peer_clamp(L);
    if (L->timing) {
      // timed pass: the fused scatter as two launches, the reference's all-to-all (rows to
      // replica my_t of each expert rank) and, with DTD, its TP all-gather (the other
      // replicas), so their times are reported separately
      L->mark("dispatch_a2a", s);
      pd.part = 1;
      check(scatter_rows_peer(a, L->pos_send.p, L->expert.p, L->n, h, pd, nullptr, false, s),
            "scatter_rows_peer");
      if (L->dtd) {
        L->mark("dispatch_ag", s);
        pd.part = 2;
        check(scatter_rows_peer(a, L->pos_send.p, L->expert.p, L->n, h, pd, nullptr, false, s),
              "scatter_rows_peer");
      }
    } else {
      L->mark("dispatch_peer", s);
      check(scatter_rows_peer(a, L->pos_send.p, L->expert.p, L->n, h, pd, nullptr, false, s),
            "scatter_rows_peer");
    }
    L->mark("barrier", s);
    plane_barrier(L, s);
    L->mark("zero_pad", s);
    zero_asm_pads(L, L->x_asm.p, s);
    rows = asm_rows_bound(L);
  } else {
    L->mark("count_exchange", s);
    // count exchange over EP (the reference's A2A metadata, fabric.cpp:282-285)
    const size_t nc = size_t(L->Tc) * E;
    std::vector<int> cnt(nc * L->P);
    if (L->direct) {
      // over the whole plane: also orders this step's peer writes after every peer's
      // previous-step reads of its buffers
      NC(ncclAllGather(L->kc.p, L->kc_all.p, nc, ncclInt32, L->plane_c, s));
      check(cudaMemcpyAsync(L->h_kc_all.p, L->kc_all.p, nc * L->plane_size * sizeof(int),
                            cudaMemcpyDeviceToHost, s),
            "memcpy");
      wait_stream(L, s);
      for (int src = 0; src < L->P; ++src)  // TP peers hold identical counts: take t = 0
        std::memcpy(cnt.data() + size_t(src) * nc, L->h_kc_all.p + size_t(L->T * src) * nc,
                    nc * sizeof(int));
    } else {
      if (L->P > 1) {
        NC(ncclAllGather(L->kc.p, L->kc_all.p, nc, ncclInt32, L->ep_c, s));
      } else {
        check(cudaMemcpyAsync(L->kc_all.p, L->kc.p, nc * sizeof(int), cudaMemcpyDeviceToDevice, s),
              "memcpy");
      }
      check(cudaMemcpyAsync(L->h_kc_all.p, L->kc_all.p, nc * L->P * sizeof(int),
                            cudaMemcpyDeviceToHost, s),
            "memcpy");
      wait_stream(L, s);
      std::memcpy(cnt.data(), L->h_kc_all.p, nc * L->P * sizeof(int));
    }
    L->plan = build_plan(L->P, L->T, E, L->dtd, L->ep, L->t, cnt.data());
    if (L->plan.asm_rows > L->R_max) throw RuntimeError("assembled rows exceed workspace");
    int* hs = L->h_seg.p;
    for (int i = 0; i <= L->Eloc; ++i) hs[i] = L->plan.seg_off[i];
    for (int i = 0; i < L->Eloc; ++i) hs[L->Eloc + 1 + i] = L->plan.seg_rows[i];
    check(cudaMemcpyAsync(L->seg_off.p, hs, sizeof(int) * (2 * L->Eloc + 1),
                          cudaMemcpyHostToDevice, s),
          "memcpy");
    if (L->direct) {
      build_peer_tables(L, cnt.data());
      check(cudaMemcpyAsync(L->disp_base.p, L->h_tabs.p, sizeof(long long) * E * (1 + L->Tc),
                            cudaMemcpyHostToDevice, s),
            "memcpy");
      // the all-to-all (and, with DTD, the expert-side all-gather) as one NVLink scatter
      L->mark("dispatch_peer", s);
      PeerDst pd;
      pd.peers = peer_table(L, 0);
      pd.disp_base = L->disp_base.p;
      pd.send_base = L->send_base.p;
      pd.Eloc = L->Eloc;
      pd.Tp = L->T;
      pd.my_t = L->t;
      pd.all_replicas = L->dtd ? 1 : 0;
    pd.clamp_rows = peer_clamp(L);
      check(scatter_rows_peer(a, L->pos_send.p, L->expert.p, L->n, h, pd, nullptr, false, s),
            "scatter_rows_peer");
      L->mark("barrier", s);
      plane_barrier(L, s);
    } else {
      L->mark("a2a_fwd", s);
      a2a_dispatch(L, L->xsend.p, L->x_asm.p, s);
      if (L->dtd) {
        L->mark("ag_fwd", s);
        grouped_p2p(L->plan.ag_asm_send, L->x_asm.p, L->plan.ag_asm_recv, L->x_asm.p, h,
                    L->tp_c, s);
      }
    }
    L->mark("zero_pad", s);
    zero_asm_pads(L, L->x_asm.p, s);
    rows = asm_rows_bound(L);
  }

  ledger_pass(L, L->ledger_phase, s);
  if (L->fwd_mode == FWD_RECORD && !L->local) {  // CAC: stash the exchanged expert rows
    stash_alloc(L);
    L->stash_rows = rows;
    check(cudaMemcpyAsync(L->stash_x.p, L->x_asm.p, sizeof(bf16) * size_t(rows) * h,
                          cudaMemcpyDeviceToDevice, s),
          "stash");
  }
  // expert FFN (tensor cores): Z = X W1 + b1, H = gelu(Z); Fe = H W2 (+ b2 on TP rank 0)
  bf16* P = L->fam_exp.param.p;
  GemmParams g{};
  GemmOperands o{};
  expert_gemm1(L, rows, s, g, o);

  L->mark("gemm2_fwd", s);
  o.A = L->hbuf.p;
  o.lda = L->fT;
  o.B = P + L->off_w2;
  o.ldb = h;
  g.epi = EPI_BIAS;
  g.N = h;
  g.K = L->fT;
  g.C = L->fe_asm.p;
  g.ldc = h;
  g.bias = (L->t == 0) ? P + L->off_b2 : nullptr;  // bias after the reduce (parallel_linear.cpp:29)
  g.aux = nullptr;
  if (L->push) set_push(L, g);  // the return trip inside the epilogue
  run_gemm(o, g, rows, s);

  const bf16* fh;
  const double nglob = double(L->n) * L->P * L->D;
  if (L->direct) {
    L->mark("barrier", s);
    plane_barrier(L, s);
    // return trip + DTD home gather + TP reduction (row-parallel GEMM2 partial sums,
    // parallel_linear.cpp:28) + combine: every token pulls and sums its expert's T partial
    // rows straight from the replicas' buffers
    L->mark("combine_pull", s);
    RowSrc src = L->push ? ret_src(L) : pull_src(L, 2);
    src.nsum = L->T;
    check(combine_pull(src, L->prob.p, L->n, h, y, L->fhome.p, L->loss_part.p, s),
          "combine_pull");
    check(loss_finalize(L->loss_part.p, L->nblk, 1.0 / (2.0 * nglob), L->loss.p, s), "loss");
    if (L->fwd_mode == FWD_RECORD)  // CAC: stash the combined (returned + reduced) rows
      check(cudaMemcpyAsync(L->stash_f.p, L->fhome.p, sizeof(bf16) * size_t(L->n) * h,
                            cudaMemcpyDeviceToDevice, s),
            "stash");
    L->mark("_end", s);
    L->have_forward = true;
    return;
  }
  if (L->local) {
    fh = L->fe_asm.p;
  } else {
    L->mark("tp_allreduce_fwd", s);
    if (L->T > 1 && L->plan.asm_rows > 0)
      NC(ncclAllReduce(L->fe_asm.p, L->fe_asm.p, size_t(L->plan.asm_rows) * h, ncclBfloat16,
                       ncclSum, L->tp_c, s));
    L->mark("a2a_ret_fwd", s);
    a2a_return(L, L->fe_asm.p, L->fhome.p, s);
    if (L->dtd) {
      L->mark("ag_home_fwd", s);
      grouped_p2p(L->plan.ag_home_send, L->fhome.p, L->plan.ag_home_recv, L->fhome.p, h,
                  L->tp_c, s);
    }
    fh = L->fhome.p;
    if (L->fwd_mode == FWD_RECORD)
      check(cudaMemcpyAsync(L->stash_f.p, L->fhome.p, sizeof(bf16) * size_t(L->n) * h,
                            cudaMemcpyDeviceToDevice, s),
            "stash");
  }
  L->mark("combine_fwd", s);
  check(combine_forward(fh, L->pos_home.p, L->prob.p, L->n, h, y, L->loss_part.p, s),
        "combine_forward");
  check(loss_finalize(L->loss_part.p, L->nblk, 1.0 / (2.0 * nglob), L->loss.p, s), "loss");
  L->mark("_end", s);
  L->have_forward = true;
}

}  // namespace

namespace {

// [n][w_src] -> [n][w_dst] rows (the zero-padded staging of small shapes)
void copy_rows_2d(bf16* dst, int w_dst, const bf16* src, int w_src, int64_t n, cudaStream_t s) {
  check(cudaMemcpy2DAsync(dst, size_t(w_dst) * 2, src, size_t(w_src) * 2,
                          size_t(std::min(w_dst, w_src)) * 2, size_t(n), cudaMemcpyDeviceToDevice, s),
        "pad copy");
}

void layer_forward(ted_layer* L, const bf16* a, bf16* y, cudaStream_t s) {
  if (L->io_h == L->h) {
    layer_forward_impl(L, a, y, s);
    return;
  }
  copy_rows_2d(L->pad_a.p, L->h, a, L->io_h, L->n, s);
  layer_forward_impl(L, L->pad_a.p, L->pad_y.p, s);
  if (L->fwd_mode != FWD_REPLAY || L->local) copy_rows_2d(y, L->io_h, L->pad_y.p, L->h, L->n, s);
}

// set_param resets the family's optimizer state (reset_master, optimizer.cpp:46-56)
void family_reset_if_needed(Family& F, cudaStream_t s) {
  if (!F.reset) return;
  CU(cudaMemsetAsync(F.m1.p, 0, sizeof(float) * F.m1.n, s));
  CU(cudaMemsetAsync(F.m2.p, 0, sizeof(float) * F.m2.n, s));
  CU(cudaMemsetAsync(F.dstep.p, 0, sizeof(long long), s));
  F.steps = 0;
  F.reset = false;
}

// steps_done += 1 and the bias corrections, both on the device (optimizer.cpp:68-70)
void family_begin(ted_layer* L, Family& F, cudaStream_t s) {
  family_reset_if_needed(F, s);
  if (!L->capturing) F.steps += 1;  // host mirror (replays add it themselves)
  check(adam_prep(F.dstep.p, F.dcoef.p, L->adam.beta1, L->adam.beta2, s), "adam_prep");
}

// AdamW over one bias kind (b1 or b2) of every local expert, after its column sum.
void bias_adam(ted_layer* L, int64_t off, int64_t len, cudaStream_t s) {
  Family& F = L->fam_exp;
  check(adam_segments(F.master.p, F.m1.p, F.m2.p, F.param.p, F.grad.p, L->Eloc, L->per_expert,
                      off, len, float(L->adam.lr), float(L->adam.beta1), float(L->adam.beta2),
                      float(1.0 - L->adam.beta1), float(1.0 - L->adam.beta2),
                      float(L->adam.eps), float(L->adam.weight_decay), 1.f, 1.f, F.dcoef.p,
                      sm_count(), s),
        "adam_segments");
}

// wgrad GEMM params for the fused-AdamW epilogue (the gradient tile updates the parameter
// block in place; the bf16 parameter is the GEMM output)
void set_adam_epilogue(ted_layer* L, GemmParams& g, int64_t off) {
  Family& F = L->fam_exp;
  g.epi = EPI_ADAM;
  g.adam_grad = L->keep_grads ? g.C : nullptr;  // g.C = the gradient slot of this weight
  g.C = F.param.p + off;
  g.adam_master = F.master.p + off;
  g.adam_m1 = F.m1.p + off;
  g.adam_m2 = F.m2.p + off;
  g.adam_coef = F.dcoef.p;
  g.adam = AdamK{float(L->adam.lr), float(L->adam.beta1), float(L->adam.beta2),
                 float(1.0 - L->adam.beta1), float(1.0 - L->adam.beta2), float(L->adam.eps),
                 float(L->adam.weight_decay)};
}

// --------------------------------------------------------------- backward
void layer_backward_impl(ted_layer* L, const bf16* dy, bf16* da, cudaStream_t s);
void layer_backward(ted_layer* L, const bf16* dy, bf16* da, cudaStream_t s) {
  if (L->io_h == L->h) {
    layer_backward_impl(L, dy, da, s);
    return;
  }
  if (dy) copy_rows_2d(L->pad_dy.p, L->h, dy, L->io_h, L->n, s);
  layer_backward_impl(L, dy ? L->pad_dy.p : nullptr, L->pad_da.p, s);
  copy_rows_2d(da, L->io_h, L->pad_da.p, L->h, L->n, s);
}

void layer_backward_impl(ted_layer* L, const bf16* dy, bf16* da, cudaStream_t s) {
  if (!L->have_forward) throw ConfigError("backward called before forward");
  const int h = L->h, E = L->E;
  const double nglob = double(L->n) * L->P * L->D;
  const bf16* fh = L->local ? L->fe_asm.p : L->fhome.p;
  bf16* dfe_t = L->local ? L->dfe_asm.p : L->dfe_send.p;
  L->mark("combine_bwd", s);
  // combine backward + dlogits (moe.cpp:587-597, :197-203)
  if (L->direct) {  // p*dy rows go straight into the experts' dFe buffers (moe.cpp:603-632)
    PeerDst pd;
    pd.peers = peer_table(L, 1);
    pd.disp_base = L->disp_base.p;
    pd.send_base = L->send_base.p;
    pd.Eloc = L->Eloc;
    pd.Tp = L->T;
    pd.my_t = L->t;
    pd.all_replicas = L->dtd ? 1 : 0;
    pd.clamp_rows = peer_clamp(L);
    check(combine_backward_peer(L->fhome.p, L->pos_home.p, L->pos_send.p, L->prob.p, L->probs.p,
                                L->expert.p, L->n, h, E, dy, L->last_y, float(1.0 / nglob), pd,
                                L->dlogits.p, s),
          "combine_backward_peer");
  } else
  check(combine_backward(fh, L->pos_home.p, L->pos_send.p, L->prob.p, L->probs.p, L->expert.p,
                         L->n, h, E, dy, L->last_y, float(1.0 / nglob), dfe_t, L->dlogits.p, s),
        "combine_backward");
  L->mark("gate_dw", s);
  // dWg = a^T dlogits (moe.cpp:205)
  check(gate_backward_weight(L->last_a, L->dlogits.p, L->n, h, E, L->gate_part.p,
                             L->fam_non.grad.p, s),
        "gate_backward_weight");
  int64_t rows;
  L->mark(L->local ? "zero_pad" : "a2a_bwd", s);
  if (L->local) {
    check(zero_pad_rows(L->dfe_asm.p, h, h, L->seg_off.p, L->seg_valid_view, E, kPad, s),
          "zero_pad");
    rows = L->R_max;
  } else if (L->direct) {
    L->mark("barrier", s);
    plane_barrier(L, s);
    L->mark("zero_pad", s);
    zero_asm_pads(L, L->dfe_asm.p, s);
    rows = asm_rows_bound(L);
  } else {
    a2a_dispatch(L, L->dfe_send.p, L->dfe_asm.p, s);  // moe.cpp:614
    if (L->dtd) {
      L->mark("ag_bwd", s);
      grouped_p2p(L->plan.ag_asm_send, L->dfe_asm.p, L->plan.ag_asm_recv, L->dfe_asm.p, h,
                  L->tp_c, s);  // moe.cpp:626
    }
    L->mark("zero_pad", s);
    zero_asm_pads(L, L->dfe_asm.p, s);
    rows = asm_rows_bound(L);
  }
  ledger_pass(L, 2, s);
  bf16* P = L->fam_exp.param.p;
  bf16* G = L->fam_exp.grad.p;
  GemmOperands o{};
  GemmParams g{};
  g.groups = L->Eloc;
  g.seg_off = L->seg_off.p;
  L->mark("dgrad2", s);
  // dgrad of GEMM2 with the GELU backward fused: dZ = (dFe W2^T) * gelu'(Z)   (in place)
  g.mode = GEMM_ROWS;
  g.epi = EPI_DGELU;
  g.N = L->fT;
  g.K = h;
  g.C = L->z.p;
  g.ldc = L->fT;
  g.aux = L->z.p;
  g.ld_aux = L->fT;
  o.A = L->dfe_asm.p;
  o.lda = h;
  o.a_mn = false;
  o.B = P + L->off_w2;
  o.ldb = h;
  o.b_group_stride = L->per_expert;
  o.b_mn = false;
  g.colsum_part = L->col_part.p;  // db1 partials straight from the epilogue's dZ
  run_gemm(o, g, rows, s);
  L->mark("colsum", s);
  check(colsum_finish(L->col_part.p, L->fT, L->seg_off.p, L->Eloc, G + L->off_b1,
                      L->per_expert, s),
        "colsum db1");
  L->mark("wgrad2", s);
  // wgrad of GEMM2: dW2 = H^T dFe  -> expert family grads (row_parallel_backward :36)
  g = GemmParams{};
  g.groups = L->Eloc;
  g.seg_off = L->seg_off.p;
  g.mode = GEMM_KDIM;
  g.epi = EPI_STORE;
  g.M = L->fT;
  g.N = h;
  g.C = G + L->off_w2;
  g.ldc = h;
  g.c_group_stride = L->per_expert;
  // the optimizer follows this backward and the expert family needs no data-parallel sync:
  // AdamW runs inside the wgrad epilogues (W2 is no longer read: dgrad2 ran before)
  const bool fuse_adam = L->step_follows && L->fuse_ok;
  L->grads_stale = fuse_adam && !L->keep_grads;
  if (fuse_adam) {
    family_begin(L, L->fam_exp, s);
    set_adam_epilogue(L, g, L->off_w2);
  }
  o = GemmOperands{};
  o.A = L->hbuf.p;
  o.lda = L->fT;
  o.a_mn = true;
  o.B = L->dfe_asm.p;
  o.ldb = h;
  o.b_mn = true;
  run_gemm(o, g, rows, s);
  L->mark("colsum", s);
  const int maxg = int(std::min<int64_t>(rows, L->R_max));
  check(colsum_groups(L->dfe_asm.p, h, h, L->seg_off.p, L->Eloc, maxg, L->col_part.p,
                      G + L->off_b2, L->per_expert, s),
        "colsum db2");
  if (fuse_adam) bias_adam(L, L->off_b2, h, s);
  L->mark("dgrad1", s);
  // dgrad of GEMM1: dX = dZ W1^T  (column_parallel_backward :16)
  g = GemmParams{};
  g.groups = L->Eloc;
  g.seg_off = L->seg_off.p;
  g.mode = GEMM_ROWS;
  g.epi = EPI_STORE;
  g.N = h;
  g.K = L->fT;
  bf16* dx_asm = L->direct ? L->dx_asm.p : L->fe_asm.p;  // Fe is dead after forward
  g.C = dx_asm;
  g.ldc = h;
  o = GemmOperands{};
  o.A = L->z.p;
  o.lda = L->fT;
  o.a_mn = false;
  o.B = P + L->off_w1;
  o.ldb = L->fT;
  o.b_group_stride = L->per_expert;
  o.b_mn = false;
  if (L->push) set_push(L, g);  // dX partials straight to the home ranks
  run_gemm(o, g, rows, s);
  L->mark("wgrad1", s);
  // wgrad of GEMM1: dW1 = X^T dZ
  g = GemmParams{};
  g.groups = L->Eloc;
  g.seg_off = L->seg_off.p;
  g.mode = GEMM_KDIM;
  g.epi = EPI_STORE;
  g.M = h;
  g.N = L->fT;
  g.C = G + L->off_w1;
  g.ldc = L->fT;
  g.c_group_stride = L->per_expert;
  if (fuse_adam) set_adam_epilogue(L, g, L->off_w1);  // dgrad1 (reads W1) ran before
  o = GemmOperands{};
  o.A = L->x_asm.p;
  o.lda = h;
  o.a_mn = true;
  o.B = L->z.p;
  o.ldb = L->fT;
  o.b_mn = true;
  run_gemm(o, g, rows, s);
  if (fuse_adam) {
    bias_adam(L, L->off_b1, L->fT, s);
    L->exp_done_fused = true;
  }
  const bf16* dxh;
  if (L->direct) {
    L->mark("barrier", s);
    plane_barrier(L, s);
    L->mark("gate_dx", s);
    // return trip of dX pulled from the expert ranks, TP partial sums of the
    // column-parallel dgrad folded in (parallel_linear.cpp:19), + dl Wg^T (moe.cpp:660-685)
    RowSrc src = L->push ? ret_src(L) : pull_src(L, 3);
    src.nsum = L->T;
    check(gate_backward_input(src, L->dlogits.p, L->fam_non.param.p, L->n, h, E, da, s),
          "gate_backward_input");
    L->mark("_end", s);
    return;
  }
  if (L->local) {
    dxh = L->fe_asm.p;
  } else {
    L->mark("tp_allreduce_bwd", s);
    if (L->T > 1 && L->plan.asm_rows > 0)  // parallel_linear.cpp:19
      NC(ncclAllReduce(L->fe_asm.p, L->fe_asm.p, size_t(L->plan.asm_rows) * h, ncclBfloat16,
                       ncclSum, L->tp_c, s));
    L->mark("a2a_ret_bwd", s);
    a2a_return(L, L->fe_asm.p, L->dx_home.p, s);  // moe.cpp:660
    if (L->dtd) {
      L->mark("ag_home_bwd", s);
      grouped_p2p(L->plan.ag_home_send, L->dx_home.p, L->plan.ag_home_recv, L->dx_home.p, h,
                  L->tp_c, s);  // moe.cpp:678
    }
    dxh = L->dx_home.p;
  }
  L->mark("gate_dx", s);
  // da = da_dispatch + dinput_gate (moe.cpp:685)
  RowSrc rs;
  rs.local = dxh;
  rs.pos_home = L->pos_home.p;
  check(gate_backward_input(rs, L->dlogits.p, L->fam_non.param.p, L->n, h, E, da, s),
        "gate_backward_input");
  L->mark("_end", s);
}

// --------------------------------------------------------------- optimizer
void family_step(ted_layer* L, Family& F, cudaStream_t s) {
  if (F.elems == 0) return;
  family_begin(L, F, s);
  const int64_t owned = F.end - F.begin;
  const int64_t one = std::max<int64_t>(owned, 1);
  const int64_t tile = L->tiles.enabled ? std::min<int64_t>(L->tiles.tile_size, one) : one;
  F.upcast_peak = std::max<uint64_t>(F.upcast_peak, owned == 0 ? 0 : uint64_t(tile) * 4);
  if (F.blocked) {  // expert family with blk_off weight state: w1, w2 blocked, biases flat
    const struct {
      int64_t off, len;
      int cols;
    } regions[4] = {{L->off_w1, int64_t(L->h) * L->fT, L->fT},
                    {L->off_b1, L->fT, 0},
                    {L->off_w2, int64_t(L->fT) * L->h, L->h},
                    {L->off_b2, L->h, 0}};
    for (const auto& rg : regions)
      check(adam_segments(F.master.p, F.m1.p, F.m2.p, F.param.p, F.grad.p, L->Eloc,
                          L->per_expert, rg.off, rg.len, float(L->adam.lr),
                          float(L->adam.beta1), float(L->adam.beta2),
                          float(1.0 - L->adam.beta1), float(1.0 - L->adam.beta2),
                          float(L->adam.eps), float(L->adam.weight_decay), 1.f, 1.f, F.dcoef.p,
                          sm_count(), s, rg.cols),
            "adam_segments");
  } else {
    check(adam_step(F.master.p, F.m1.p, F.m2.p, F.param.p, F.grad.p, F.begin, F.end, tile,
                    float(L->adam.lr), float(L->adam.beta1), float(L->adam.beta2),
                    float(1.0 - L->adam.beta1), float(1.0 - L->adam.beta2), float(L->adam.eps),
                    float(L->adam.weight_decay), 1.f, 1.f, F.dcoef.p, s),
          "adam_step");
  }
  if (F.group > 1) {  // ZeRO-1 completion (moe.cpp:718-732), zero-padded equal chunks
    bf16* gbuf = F.gather.p;
    CU(cudaMemsetAsync(gbuf + F.pos * F.chunk, 0, sizeof(bf16) * F.chunk, s));
    CU(cudaMemcpyAsync(gbuf + F.pos * F.chunk, F.param.p + F.begin, sizeof(bf16) * owned,
                       cudaMemcpyDeviceToDevice, s));
    NC(ncclAllGather(gbuf + F.pos * F.chunk, gbuf, size_t(F.chunk), ncclBfloat16, F.dp, s));
    for (int p = 0; p < F.group; ++p) {
      if (p == F.pos) continue;
      const int64_t b = shard_lo(F.elems, F.group, p), e = shard_lo(F.elems, F.group, p + 1);
      if (e > b)
        CU(cudaMemcpyAsync(F.param.p + b, gbuf + p * F.chunk, sizeof(bf16) * (e - b),
                           cudaMemcpyDeviceToDevice, s));
    }
  }
}

void layer_optimizer(ted_layer* L, cudaStream_t s) {
  if (!L->capturing) ledger_host_optim(L);  // graph replays add it per launch
  L->mark("grad_sync", s);
  // run_grad_sync (moe.cpp:699-711): sum over the data groups
  if (L->D > 1)
    NC(ncclAllReduce(L->fam_exp.grad.p, L->fam_exp.grad.p, size_t(L->fam_exp.elems), ncclBfloat16,
                     ncclSum, L->expdp_c, s));
  if (L->P * L->D > 1)
    NC(ncclAllReduce(L->fam_non.grad.p, L->fam_non.grad.p, size_t(L->fam_non.elems),
                     ncclBfloat16, ncclSum, L->nonexpdp_c, s));
  L->mark("adam", s);
  family_step(L, L->fam_non, s);
  if (L->exp_done_fused) {  // already updated inside the backward's wgrad epilogues
    L->exp_done_fused = false;
  } else {
    family_step(L, L->fam_exp, s);
  }
  L->mark("_end", s);
}

uint64_t name_seed(uint64_t seed, const std::string& name) {
  uint64_t hsh = 14695981039346656037ULL;
  for (unsigned char c : name) {
    hsh ^= c;
    hsh *= 1099511628211ULL;
  }
  return seed * 0x9E3779B97F4A7C15ULL + hsh;
}

std::vector<std::string> local_param_names(ted_layer* L) {
  std::vector<std::string> v{"layer0.gate.w"};
  for (int le = 0; le < L->Eloc; ++le) {
    const std::string p = "layer0.expert" + std::to_string(L->ep * L->Eloc + le) + ".";
    for (const char* leaf : {"w1", "b1", "w2", "b2"}) v.push_back(p + leaf);
  }
  return v;
}

// Export the four exchange buffers with CUDA IPC, all-gather the handles over the plane
// and map every peer's buffers (NVLink peer access), giving device tables of base pointers.
void setup_peer_exchange(ted_layer* L) {
  if (L->share) L->dx_asm.view(L->share->dx_asm);
  else L->dx_asm.alloc(size_t(L->R_max) * L->h);
  L->disp_base.alloc(size_t(L->E) * (1 + L->Tc));
  L->h_tabs.alloc(size_t(L->E) * (1 + L->Tc));
  L->bar.alloc(1);
  L->bar.zero();
  L->bar_flags.alloc(size_t(L->plane_size));
  L->bar_flags.zero();
  L->bar_epoch.alloc(1);
  L->bar_epoch.zero();
  const char* dp = std::getenv("TED_DEVPLAN");
  L->devplan = !(dp && std::strcmp(dp, "0") == 0);
  const char* bv = std::getenv("TED_BARRIER");
  L->nccl_barrier = bv && std::strcmp(bv, "nccl") == 0;
  {
    const char* pv = std::getenv("TED_PUSH");
    L->push = L->devplan && !(pv && std::strcmp(pv, "0") == 0);
  }
  if (L->push) {
    L->ret.alloc(size_t(L->T) * L->n * L->h);
    L->row_home.alloc(size_t(L->R_max));
    L->row_src.alloc(size_t(L->R_max));
  } else {
    L->ret.alloc(8);  // (mapped like the others; unused)
  }
  constexpr int NB = 6;  // x_asm, dfe_asm, fe_asm, dx_asm, barrier flags, receive slots
  void* mine[NB] = {L->x_asm.p, L->dfe_asm.p, L->fe_asm.p, L->dx_asm.p, L->bar_flags.p, L->ret.p};
  const int PS = L->plane_size;
  const size_t HB = sizeof(cudaIpcMemHandle_t);
  std::vector<char> hmine(NB * HB), hall(size_t(PS) * NB * HB);
  for (int b = 0; b < NB; ++b)
    CU(cudaIpcGetMemHandle(reinterpret_cast<cudaIpcMemHandle_t*>(hmine.data() + b * HB), mine[b]));
  DevBuf<char> dh;
  dh.alloc(hall.size());
  CU(cudaMemcpy(dh.p + size_t(L->plane_rank) * NB * HB, hmine.data(), NB * HB,
                cudaMemcpyHostToDevice));
  NC(ncclAllGather(dh.p + size_t(L->plane_rank) * NB * HB, dh.p, NB * HB, ncclChar, L->plane_c,
                   nullptr));
  CU(cudaDeviceSynchronize());
  CU(cudaMemcpy(hall.data(), dh.p, hall.size(), cudaMemcpyDeviceToHost));
  std::vector<unsigned long long> tab(size_t(NB) * PS);
  if (L->share) {  // buffers 0-3 are the sharing layer's: reuse its mapped peer addresses
    std::vector<unsigned long long> st(size_t(NB) * PS);
    CU(cudaMemcpy(st.data(), L->share->peer_tab.p, st.size() * sizeof(unsigned long long),
                  cudaMemcpyDeviceToHost));
    std::vector<unsigned long long> tab(size_t(NB) * PS);
    for (int r = 0; r < PS; ++r)
      for (int b = 0; b < NB; ++b) {
        if (b < 4) {  // (the receive slots, 5, stay per layer like the barrier flags)
          tab[size_t(b) * PS + r] = st[size_t(b) * PS + r];
          continue;
        }
        void* ptr = mine[b];
        if (r != L->plane_rank) {
          cudaIpcMemHandle_t hd;
          std::memcpy(&hd, hall.data() + (size_t(r) * NB + b) * HB, HB);
          CU(cudaIpcOpenMemHandle(&ptr, hd, cudaIpcMemLazyEnablePeerAccess));
          L->ipc_opened.push_back(ptr);
        }
        tab[size_t(b) * PS + r] = reinterpret_cast<unsigned long long>(ptr);
      }
    L->peer_tab.alloc(tab.size());
    CU(cudaMemcpy(L->peer_tab.p, tab.data(), tab.size() * sizeof(unsigned long long),
                  cudaMemcpyHostToDevice));
    return;
  }
  for (int r = 0; r < PS; ++r)
    for (int b = 0; b < NB; ++b) {
      void* ptr = mine[b];
      if (r != L->plane_rank) {
        cudaIpcMemHandle_t hd;
        std::memcpy(&hd, hall.data() + (size_t(r) * NB + b) * HB, HB);
        CU(cudaIpcOpenMemHandle(&ptr, hd, cudaIpcMemLazyEnablePeerAccess));
        L->ipc_opened.push_back(ptr);
      }
      tab[size_t(b) * PS + r] = reinterpret_cast<unsigned long long>(ptr);
    }
  L->peer_tab.alloc(tab.size());
  CU(cudaMemcpy(L->peer_tab.p, tab.data(), tab.size() * sizeof(unsigned long long),
                cudaMemcpyHostToDevice));
}

void create_layer(ted_layer* L, const ted_model_cfg* model, const ted_topo_cfg* topo,
                  const ted_flags* flags, const ted_adam_cfg* adam, const ted_tile_cfg* tiles,
                  double cf, int shard_opt, int rank, const void* uid,
                  ncclComm_t parent = nullptr, ted_layer* share = nullptr,
                  bool io_internal = false) {
  require(model && topo && flags && adam && tiles, "null config pointer");
  L->model = *model;
  L->topo = *topo;
  L->flags = *flags;
  L->adam = *adam;
  L->tiles = *tiles;
  L->cf = cf;
  L->shard_opt = shard_opt;
  L->rank = rank;
  require(model->hidden >= 1 && model->experts >= 1 && model->tokens_per_shard >= 1,
          "model: hidden, experts and tokens_per_shard must be >= 1");
  require(flags->cac == 0 && flags->ckpt == 0,
          "flags: ckpt/cac (activation checkpointing, CAC) are not implemented in this build");
  require(model->experts <= 64, "model: at most 64 experts");
  L->hu = model->hidden;
  L->h = (L->hu + 255) / 256 * 256;  // tensor-core N tile; zero-padded beyond hu
  L->io_h = io_internal ? L->h : L->hu;
  L->E = model->experts;
  L->n = model->tokens_per_shard;
  L->f = 4 * L->hu;  // kFfnMultiple (moe.hpp:33)
  L->T = topo->tensor_parallel;
  L->P = topo->experts;
  L->world = topo->world_size;
  require(L->T >= 1 && L->P >= 1 && L->world >= 1, "topology degrees must be >= 1");
  require(L->world % (L->T * L->P) == 0,
          "tensor_parallel * expert_parallel must divide world_size");
  L->D = L->world / (L->T * L->P);
  require(rank >= 0 && rank < L->world, "rank outside [0, world_size)");
  require(L->E % L->P == 0, "experts (" + std::to_string(L->E) +
                                ") must be a multiple of the expert-parallel degree (" +
                                std::to_string(L->P) + ")");
  L->Eloc = L->E / L->P;
  require(L->f % L->T == 0, "tensor_parallel does not divide the block inner width");
  L->fTu = L->f / L->T;
  L->fT = (L->fTu + 255) / 256 * 256;
  L->dtd = flags->dtd && L->T > 1;
  require(!L->dtd || L->n % L->T == 0,
          "token dropping needs tensor_parallel to divide tokens_per_shard (moe.cpp:775-779)");
  L->t = rank % L->T;
  L->ep = (rank / L->T) % L->P;
  L->d = rank / (L->T * L->P);
  L->local = (L->P == 1 && L->T == 1);
  L->Tc = L->dtd ? L->T : 1;
  L->my_chunk = L->dtd ? (flags->corrupt_drop ? (L->t + 1) % L->T : L->t) : -1;
  L->cap = cf > 0 ? std::min<int64_t>(L->n, int64_t(std::ceil(cf * L->n / double(L->E)))) : L->n;
  L->nblk = (L->n + kRouteBlock - 1) / kRouteBlock;
  require_device();
  CU(cudaHostAlloc(reinterpret_cast<void**>(&L->fault_h), sizeof(int),
                   cudaHostAllocMapped | cudaHostAllocPortable));
  *L->fault_h = 0;
  CU(cudaHostGetDevicePointer(reinterpret_cast<void**>(&L->fault_d), L->fault_h, 0));

  // communicators (topology.cpp:56-93 colours; ascending-rank keys)
  if (L->world > 1) {
    if (parent != nullptr) {  // a layer of a model stack: split the model's communicator
      NC(ncclCommSplit(parent, 0, rank, &L->world_c, nullptr));
    } else {
      require(uid != nullptr, "world_size > 1 needs an NCCL unique id");
      ncclUniqueId id;
      std::memcpy(&id, uid, sizeof(id));
      NC(ncclCommInitRank(&L->world_c, L->world, id, rank));
    }
    NC(ncclCommSplit(L->world_c, L->ep + L->P * L->d, L->t, &L->tp_c, nullptr));
    NC(ncclCommSplit(L->world_c, L->t + L->T * L->d, L->ep, &L->ep_c, nullptr));
    NC(ncclCommSplit(L->world_c, L->t + L->T * L->ep, L->d, &L->expdp_c, nullptr));
    NC(ncclCommSplit(L->world_c, L->t, L->ep + L->P * L->d, &L->nonexpdp_c, nullptr));
    NC(ncclCommSplit(L->world_c, L->d, L->t + L->T * L->ep, &L->plane_c, nullptr));
    const char* ex = std::getenv("TED_EXCHANGE");
    L->direct = !L->local && !(ex && std::strcmp(ex, "nccl") == 0);
    L->plane_rank = L->t + L->T * L->ep;
    L->plane_size = L->T * L->P;
  }

  // flat families in enumerate_params order (moe.cpp:115-147, flatten_family :303-312)
  L->off_w1 = 0;
  L->off_b1 = int64_t(L->h) * L->fT;
  L->off_w2 = L->off_b1 + L->fT;
  L->off_b2 = L->off_w2 + int64_t(L->fT) * L->h;
  L->per_expert = L->off_b2 + L->h;
  setup_family(L, L->fam_exp, L->per_expert * L->Eloc, L->expdp_c, L->D, L->d);
  setup_family(L, L->fam_non, int64_t(L->h) * L->E, L->nonexpdp_c, L->P * L->D,
               L->ep + L->P * L->d);

  // workspaces (worst case: every source routes everything here, capped by capacity)
  const int64_t n = L->n, h = L->h, E = L->E;
  const int64_t recv_max = std::min<int64_t>(int64_t(L->P) * n, int64_t(L->Eloc) * L->P * L->cap);
  L->R_max = pad_up(recv_max + int64_t(L->Eloc) * kPad, kPad);
  L->logits.alloc(n * E);
  L->probs.alloc(n * E);
  L->prob.alloc(n);
  L->dlogits.alloc(n * E);
  L->loss_part.alloc(L->nblk + 1);
  L->loss.alloc(1);
  L->loss.zero();
  L->h_loss.alloc(1);
  if (size_t wt = gate_wgt_elems(L->h, L->E)) L->wgT.alloc(wt);
  L->led.alloc(5 * 3 * 2);
  L->led.zero();
  L->verdict.alloc(2);
  {
    const int one[2] = {1, 1};
    CU(cudaMemcpy(L->verdict.p, one, sizeof(one), cudaMemcpyHostToDevice));
  }
  L->expert.alloc(n);
  L->slot.alloc(n);
  L->pos_send.alloc(n);
  L->pos_home.alloc(n);
  L->blk_hist.alloc(size_t(L->nblk) * E);
  L->blk_prefix.alloc(size_t(L->nblk) * E);
  L->chunk_prefix.alloc(size_t(L->Tc + 1) * E);
  L->kc.alloc(size_t(L->Tc) * E);
  L->kc_all.alloc(size_t(L->Tc) * E * L->P * L->T);
  L->send_base.alloc(E);
  L->home_base.alloc(size_t(L->Tc) * E);
  L->seg_off.alloc(size_t(2 * L->Eloc + 2));
  L->seg_off.zero();
  L->h_kc_all.alloc(size_t(L->Tc) * E * L->P * L->T);
  L->h_seg.alloc(size_t(2 * L->Eloc + 2));
  L->gate_part.alloc(gate_dw_part_floats(n, L->h, L->E));
  L->col_part.alloc(std::max(colsum_part_floats(L->fT, L->Eloc, int(L->R_max)),
                             colsum_part_floats(L->h, L->Eloc, int(L->R_max))));
  if (share != nullptr) {  // activation checkpointing: one activation set for the stack
    require(share->R_max == L->R_max && share->local == L->local && share->n == n &&
                share->h == h && share->fT == L->fT,
            "activation sharing needs layers of one shape");
    L->share = share;
    for (auto pr : {std::make_pair(&L->x_asm, &share->x_asm), std::make_pair(&L->z, &share->z),
                    std::make_pair(&L->hbuf, &share->hbuf),
                    std::make_pair(&L->fe_asm, &share->fe_asm),
                    std::make_pair(&L->dfe_asm, &share->dfe_asm),
                    std::make_pair(&L->xsend, &share->xsend),
                    std::make_pair(&L->fhome, &share->fhome),
                    std::make_pair(&L->dfe_send, &share->dfe_send),
                    std::make_pair(&L->dx_home, &share->dx_home)})
      pr.first->view(*pr.second);
  } else {
    L->x_asm.alloc(size_t(L->R_max) * h);
    L->x_asm.zero();
    L->z.alloc(size_t(L->R_max) * L->fT);
    L->hbuf.alloc(size_t(L->R_max) * L->fT);
    L->fe_asm.alloc(size_t(L->R_max) * h);
    L->dfe_asm.alloc(size_t(L->R_max) * h);
    L->dfe_asm.zero();
    if (!L->local) {
      L->xsend.alloc(size_t(n) * h);
      L->xsend.zero();
      L->fhome.alloc(size_t(n) * h);
      L->fhome.zero();
      L->dfe_send.alloc(size_t(n) * h);
      L->dx_home.alloc(size_t(n) * h);
    }
  }
  if (L->io_h != L->h) {  // zero-padded staging of the caller's [n][hu] token buffers
    for (DevBuf<bf16>* b : {&L->pad_a, &L->pad_y, &L->pad_dy, &L->pad_da}) {
      b->alloc(size_t(n) * h);
      b->zero();
    }
  }
  if (L->direct) setup_peer_exchange(L);
  {
    const char* gv = std::getenv("TED_GRAPH");
    L->use_graph = !(gv && std::strcmp(gv, "0") == 0);
  }
  L->fuse_ok = L->D == 1 && L->fam_exp.group == 1 && (L->per_expert % 4) == 0 &&
               (L->off_w2 % 4) == 0 && (L->off_b1 % 4) == 0 && (L->off_b2 % 4) == 0 &&
               L->h % 256 == 0 && L->fT % 256 == 0;
  if (const char* fz = std::getenv("TED_FUSE_ADAM"))  // A/B switch for measurements
    if (std::strcmp(fz, "0") == 0) L->fuse_ok = false;
  L->fam_exp.blocked = L->fuse_ok;
  if (L->fuse_ok) {
    int least = 0, greatest = 0;
    CU(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    CU(cudaStreamCreateWithPriority(&L->hs, cudaStreamNonBlocking, greatest));
    CU(cudaEventCreateWithFlags(&L->ev_fork, cudaEventDisableTiming));
    CU(cudaEventCreateWithFlags(&L->ev_join, cudaEventDisableTiming));
  }
  CU(cudaDeviceSynchronize());
}

// seg_valid lives right after seg_off[Eloc+1] in the same device allocation
void fix_views(ted_layer* L) { L->seg_valid_view = L->seg_off.p + (L->Eloc + 1); }

}  // namespace

// =================================================================== C ABI (layer)
extern "C" {

int ted_nccl_unique_id(void* out128) {
  return guard([&] {
    ncclUniqueId id;
    NC(ncclGetUniqueId(&id));
    std::memcpy(out128, &id, sizeof(id));
  });
}

}  // extern "C"

namespace ted {
int layer_create_child(const ted_model_cfg* model, const ted_topo_cfg* topo,
                       const ted_flags* flags, const ted_adam_cfg* adam,
                       const ted_tile_cfg* tiles, double capacity_factor, int shard_optimizer,
                       int rank, ncclComm_t parent, ted_layer* share, ted_layer** out) {
  return guard([&] {
    require(out != nullptr, "null output pointer");
    auto* L = new ted_layer();
    try {
      // the stack passes its own zero-padded [n][h] buffers: no staging copies
      create_layer(L, model, topo, flags, adam, tiles, capacity_factor, shard_optimizer, rank,
                   nullptr, parent, share, /*io_internal=*/true);
      fix_views(L);
    } catch (...) {
      delete L;
      throw;
    }
    *out = L;
  });
}
void layer_backward_then_step(ted_layer* L, const bf16* dy, bf16* da, cudaStream_t s) {
  L->step_follows = true;  // fuse_ok decides inside: AdamW in the wgrad epilogues
  try {
    layer_backward(L, dy, da, s);
  } catch (...) {
    L->step_follows = false;
    throw;
  }
  L->step_follows = false;
}

void layer_set_forward_mode(ted_layer* L, int mode) {
  L->fwd_mode = mode;
  if (mode == FWD_RECORD && !L->local) stash_alloc(L);
}

void layer_check_fault(ted_layer* L) { check_fault(L); }
void layer_set_ledger_phase(ted_layer* L, int phase) { L->ledger_phase = phase; }
void layer_abort(ted_layer* L, const std::string& why) {
  if (L->poisoned.empty()) L->poisoned = why;
  abort_comms(L);
}

void layer_memory(const ted_layer* L, int64_t* activations, int64_t* params, int64_t* stash) {
  int64_t act = 0;
  for (const DevBuf<bf16>* b : {&L->x_asm, &L->z, &L->hbuf, &L->fe_asm, &L->xsend, &L->fhome,
                                &L->dfe_send, &L->dfe_asm, &L->dx_home, &L->dx_asm})
    act += int64_t(b->bytes());
  for (const DevBuf<float>* b : {&L->logits, &L->probs, &L->prob, &L->dlogits, &L->gate_part,
                                 &L->col_part})
    act += int64_t(b->bytes());
  int64_t par = 0;
  for (const Family* F : {&L->fam_exp, &L->fam_non})
    par += int64_t(F->param.bytes() + F->grad.bytes() + F->gather.bytes() + F->master.bytes() +
                   F->m1.bytes() + F->m2.bytes());
  if (activations) *activations = act;
  if (params) *params = par;
  if (stash) *stash = int64_t(L->stash_x.bytes() + L->stash_f.bytes());
}
}  // namespace ted

extern "C" {

int ted_layer_create(const ted_model_cfg* model, const ted_topo_cfg* topo,
                     const ted_flags* flags, const ted_adam_cfg* adam,
                     const ted_tile_cfg* tiles, double capacity_factor, int shard_optimizer,
                     int rank, const void* nccl_uid, ted_layer** out) {
  return guard([&] {
    require(out != nullptr, "null output pointer");
    auto* L = new ted_layer();
    try {
      create_layer(L, model, topo, flags, adam, tiles, capacity_factor, shard_optimizer, rank,
                   nccl_uid);
      fix_views(L);
    } catch (...) {
      delete L;
      throw;
    }
    *out = L;
  });
}

void ted_layer_destroy(ted_layer* L) {
  if (!L) return;
  cudaDeviceSynchronize();
  for (auto& g : L->graphs) graph_reset(g);
  for (cudaEvent_t e : L->evs) cudaEventDestroy(e);
  for (cudaEvent_t e : {L->ev_fork, L->ev_join})
    if (e) cudaEventDestroy(e);
  if (L->hs) cudaStreamDestroy(L->hs);
  for (void* ptr : L->ipc_opened) cudaIpcCloseMemHandle(ptr);
  L->ipc_opened.clear();
  for (ncclComm_t* c : {&L->tp_c, &L->ep_c, &L->expdp_c, &L->nonexpdp_c, &L->plane_c,
                        &L->world_c})
    if (*c) {
      ncclCommDestroy(*c);
      *c = nullptr;
    }
  if (L->fault_h) cudaFreeHost(L->fault_h);
  delete L;
}

int ted_layer_set_timeout(ted_layer* L, double seconds) {
  return guard([&] {
    require(L != nullptr, "null layer");
    require(seconds >= 0, "timeout must be >= 0 (0 = no limit)");
    CU(cudaDeviceSynchronize());
    L->timeout_s = seconds;
    for (auto& g : L->graphs) graph_reset(g);  // the barrier kernels carry the timeout
  });
}

int ted_layer_set_param(ted_layer* L, const char* name, const float* full) {
  return guard([&] {
    ParamLoc pl;
    require(L && name && full, "null argument");
    require(lookup(L, name, pl), std::string("no parameter named ") + name + " on rank " +
                                     std::to_string(L->rank));
    // the shard in the family's (possibly column-padded) layout: rows x ld, pads zero
    std::vector<float> shard(size_t(pl.rows * pl.ld), 0.f);
    for (int64_t r = 0; r < pl.rows; ++r)
      for (int64_t c = 0; c < pl.cols; ++c) {
        int64_t fr = r, fc = c;
        if (pl.axis == 1) fc = c + int64_t(L->t) * pl.cols;
        if (pl.axis == 2) fr = r + int64_t(L->t) * pl.rows;
        shard[size_t(r * pl.ld + c)] = full[fr * pl.full_cols + fc];
      }
    std::vector<uint16_t> b(shard.size());
    for (size_t i = 0; i < b.size(); ++i) b[i] = f2bf(shard[i]);
    Family& F = *pl.fam;
    CU(cudaDeviceSynchronize());  // a step in flight on a non-blocking stream may still write
    CU(cudaMemcpy(F.param.p + pl.off, b.data(), b.size() * 2, cudaMemcpyHostToDevice));
    const int64_t lo = std::max(pl.off, F.begin), hi = std::min(pl.off + int64_t(b.size()), F.end);
    if (state_blocked(L, pl)) {  // unsharded: the whole tensor, state in the blk_off layout
      const int64_t prow = (pl.rows + 127) / 128 * 128;  // padded rows of the blocked tile grid
      std::vector<float> blk(size_t(std::min<int64_t>(prow, pl.axis == 2 ? L->fT : L->h) * pl.ld),
                             0.f);
      for (int64_t r = 0; r < pl.rows; ++r)
        for (int64_t c = 0; c < pl.cols; ++c)
          blk[size_t(blk_off(r, c, pl.ld))] = shard[size_t(r * pl.ld + c)];
      CU(cudaMemcpy(F.master.p + pl.off, blk.data(), sizeof(float) * blk.size(),
                    cudaMemcpyHostToDevice));
    } else if (hi > lo)
      CU(cudaMemcpy(F.master.p + (lo - F.begin), shard.data() + (lo - pl.off),
                    sizeof(float) * (hi - lo), cudaMemcpyHostToDevice));
    L->fam_exp.reset = true;
    L->fam_non.reset = true;
  });
}

static int get_tensor(ted_layer* L, const char* name, float* out, int64_t* numel, bool grad) {
  return guard([&] {
    ParamLoc pl;
    require(L && name, "null argument");
    require(lookup(L, name, pl), std::string("no parameter named ") + name + " on rank " +
                                     std::to_string(L->rank));
    const int64_t cnt = pl.rows * pl.cols;
    if (numel) *numel = cnt;
    if (!out) return;
    if (grad && L->grads_stale && pl.fam == &L->fam_exp && pl.rows > 1)
      throw RuntimeError(std::string("gradient of ") + name +
                         " was consumed by the AdamW fused into the wgrad GEMM of the last "
                         "step and not stored (ted_layer_keep_grads(L, 1) stores it; a "
                         "separate backward() materialises it)");
    std::vector<uint16_t> b{};
    b.resize(size_t(pl.rows * pl.ld));
    CU(cudaDeviceSynchronize());
    CU(cudaMemcpy(b.data(), (grad ? pl.fam->grad.p : pl.fam->param.p) + pl.off, b.size() * 2,
                  cudaMemcpyDeviceToHost));
    for (int64_t r = 0; r < pl.rows; ++r)
      for (int64_t c = 0; c < pl.cols; ++c) out[r * pl.cols + c] = bf2f(b[size_t(r * pl.ld + c)]);
  });
}

int ted_layer_get_param(ted_layer* L, const char* name, float* out, int64_t* numel) {
  return get_tensor(L, name, out, numel, false);
}
int ted_layer_get_grad(ted_layer* L, const char* name, float* out, int64_t* numel) {
  return get_tensor(L, name, out, numel, true);
}

int ted_layer_init_params(ted_layer* L, uint64_t seed) {
  return guard([&] {
    require(L != nullptr, "null layer");
    CU(cudaDeviceSynchronize());  // after any step still in flight
    for (const std::string& nm : local_param_names(L)) {
      ParamLoc pl;
      lookup(L, nm, pl);
      int64_t col0 = 0;
      if (pl.axis == 1) col0 = int64_t(L->t) * pl.cols;
      if (pl.axis == 2) col0 = int64_t(L->t) * pl.rows * pl.cols;
      Family& F = *pl.fam;
      init_family_kernel<<<sm_count() * 4, 256>>>(F.param.p, F.master.p, F.begin, F.end, pl.off,
                                                  pl.rows, pl.cols, pl.ld, pl.full_cols, col0,
                                                  name_seed(seed, nm), float(pl.scale),
                                                  state_blocked(L, pl) ? 1 : 0);
      CU(cudaGetLastError());
    }
    L->fam_exp.reset = true;
    L->fam_non.reset = true;
    CU(cudaDeviceSynchronize());
  });
}

int ted_layer_forward(ted_layer* L, const uint16_t* a, uint16_t* y, void* stream) {
  return guard([&] {
    require(L && a && y, "null argument");
    check_fault(L);
    layer_forward(L, reinterpret_cast<const bf16*>(a), reinterpret_cast<bf16*>(y), S(stream));
  });
}

int ted_layer_backward(ted_layer* L, const uint16_t* dy, uint16_t* da, void* stream) {
  return guard([&] {
    require(L && da, "null argument");
    check_fault(L);
    layer_backward(L, reinterpret_cast<const bf16*>(dy), reinterpret_cast<bf16*>(da), S(stream));
  });
}

int ted_layer_optimizer_step(ted_layer* L, void* stream) {
  return guard([&] {
    require(L != nullptr, "null layer");
    check_fault(L);
    layer_optimizer(L, S(stream));
  });
}

}  // extern "C"

namespace {

// forward + synthetic loss + backward (AdamW fused into wgrad) + optimizer on stream ms
void step_body(ted_layer* L, const uint16_t* a, uint16_t* y, uint16_t* da, cudaStream_t ms) {
  layer_forward(L, reinterpret_cast<const bf16*>(a), reinterpret_cast<bf16*>(y), ms);
  L->step_follows = true;  // the optimizer follows: fuse AdamW into the wgrad epilogues
  try {
    layer_backward(L, nullptr, reinterpret_cast<bf16*>(da), ms);
  } catch (...) {
    L->step_follows = false;
    throw;
  }
  L->step_follows = false;
  layer_optimizer(L, ms);
}

void graph_reset(ted_layer::Graph& g) {
  if (g.exec) cudaGraphExecDestroy(g.exec);
  for (cudaEvent_t e : g.evs) cudaEventDestroy(e);
  g = ted_layer::Graph{};
}

// Capture the single-rank step once per (a, y, da).
void graph_capture(ted_layer* L, ted_layer::Graph& g, const uint16_t* a, uint16_t* y,
                   uint16_t* da) {
  graph_reset(g);
  const size_t ev0 = L->ev_used;
  const unsigned long long before = launches();
  L->capturing = true;
  CU(cudaStreamBeginCapture(L->hs, cudaStreamCaptureModeThreadLocal));
  try {
    step_body(L, a, y, da, L->hs);
  } catch (...) {
    cudaGraph_t broken = nullptr;
    cudaStreamEndCapture(L->hs, &broken);
    if (broken) cudaGraphDestroy(broken);
    L->capturing = false;
    throw;
  }
  cudaGraph_t graph = nullptr;
  CU(cudaStreamEndCapture(L->hs, &graph));
  L->capturing = false;
  cudaError_t e = cudaGraphInstantiate(&g.exec, graph, 0);
  cudaGraphDestroy(graph);
  CU(e);
  g.launches = launches() - before;
  count_launch(-int(g.launches));  // counted again on every replay
  (void)ev0;
  g.a = a;
  g.y = y;
  g.da = da;
}

}  // namespace

extern "C" {

int ted_layer_step(ted_layer* L, const uint16_t* a, uint16_t* y, uint16_t* da, void* stream) {
  return guard([&] {
    require(L && a && y && da, "null argument");
    check_fault(L);
    cudaStream_t cs = S(stream);
    cudaStream_t ms = cs;
    if (L->hs) {  // fork onto the layer's own stream (the graph is captured on it)
      CU(cudaEventRecord(L->ev_fork, cs));
      CU(cudaStreamWaitEvent(L->hs, L->ev_fork, 0));
      ms = L->hs;
    }
    // stage timing runs eagerly (event pairs around every stage; the host enqueues faster
    // than the GPU drains, so the intervals are kernel time)
    if ((L->local || (L->direct && L->devplan)) && L->hs && L->use_graph && !L->timing) {
      family_reset_if_needed(L->fam_non, ms);  // set_param resets stay outside the graph
      family_reset_if_needed(L->fam_exp, ms);
      ted_layer::Graph* hit = nullptr;
      ted_layer::Graph* lru = &L->graphs[0];
      for (auto& c : L->graphs) {
        if (c.exec && c.a == a && c.y == y && c.da == da) hit = &c;
        if (c.used < lru->used) lru = &c;
      }
      if (!hit) {
        hit = lru;
        graph_capture(L, *hit, a, y, da);
      }
      ted_layer::Graph& g = *hit;
      g.used = ++L->graph_clock;
      CU(cudaGraphLaunch(g.exec, L->hs));
      count_launch(int(g.launches));
      ledger_host_optim(L);
      L->fam_non.steps += 1;
      L->fam_exp.steps += 1;
      L->have_forward = true;
      L->last_a = reinterpret_cast<const bf16*>(a);
      L->last_y = reinterpret_cast<const bf16*>(y);
    } else {
      step_body(L, a, y, da, ms);
    }
    if (L->hs) {  // join back into the caller's stream
      CU(cudaEventRecord(L->ev_join, L->hs));
      CU(cudaStreamWaitEvent(cs, L->ev_join, 0));
    }
  });
}

int ted_layer_keep_grads(ted_layer* L, int keep) {
  return guard([&] {
    require(L != nullptr, "null layer");
    if (L->keep_grads == (keep != 0)) return;
    CU(cudaDeviceSynchronize());
    L->keep_grads = keep != 0;
    for (auto& g : L->graphs) graph_reset(g);  // the captured epilogues change
  });
}

int ted_layer_loss_async(ted_layer* L, double* loss_pinned, void* stream) {
  return guard([&] {
    require(L && loss_pinned, "null argument");
    check_fault(L);
    CU(cudaMemcpyAsync(loss_pinned, L->loss.p, sizeof(double), cudaMemcpyDeviceToHost,
                       S(stream)));
  });
}

int ted_layer_loss(ted_layer* L, double* loss, void* stream) {
  return guard([&] {
    require(L && loss, "null argument");
    // into pinned memory: a copy to the caller's pageable double would block the host behind
    // a stalled collective, out of reach of the timeout
    CU(cudaMemcpyAsync(L->h_loss.p, L->loss.p, sizeof(double), cudaMemcpyDeviceToHost,
                       S(stream)));
    wait_stream(L, S(stream));
    *loss = *L->h_loss.p;
  });
}

int ted_layer_get_stats(ted_layer* L, ted_layer_stats* o) {
  return guard([&] {
    require(L && o, "null argument");
    std::memset(o, 0, sizeof(*o));
    CU(cudaDeviceSynchronize());
    check_fault(L);
    const int E = L->E, Tc = L->Tc;
    std::vector<int> kc(size_t(Tc) * E), cp(size_t(Tc + 1) * E);
    CU(cudaMemcpy(kc.data(), L->kc.p, kc.size() * 4, cudaMemcpyDeviceToHost));
    CU(cudaMemcpy(cp.data(), L->chunk_prefix.p, cp.size() * 4, cudaMemcpyDeviceToHost));
    int64_t kept = 0;
    for (int v : kc) kept += v;
    o->tokens = L->n;
    o->dropped = L->n - kept;
    const int64_t hb = int64_t(L->hu) * 2;  // the reference's rows of hu elements
    if (L->local) {
      o->send_rows = kept;
      std::vector<int> so(E + 1);
      CU(cudaMemcpy(so.data(), L->seg_off.p, so.size() * 4, cudaMemcpyDeviceToHost));
      o->asm_rows = so[E];
      for (int e = 0; e < E && e < 64; ++e) o->kept_per_expert[e] = kc[e];
    } else {
      if (L->direct && L->devplan) {  // the step planned on the device: rebuild the host plan
        const size_t nc = size_t(Tc) * E;
        std::vector<int> all(nc * L->plane_size), cnt(nc * L->P);
        CU(cudaMemcpy(all.data(), L->kc_all.p, all.size() * sizeof(int),
                      cudaMemcpyDeviceToHost));
        for (int src = 0; src < L->P; ++src)
          std::memcpy(cnt.data() + size_t(src) * nc, all.data() + size_t(L->T * src) * nc,
                      nc * sizeof(int));
        L->plan = build_plan(L->P, L->T, E, L->dtd, L->ep, L->t, cnt.data());
      }
      o->send_rows = L->plan.send_rows;
      o->a2a_rows_offrank = L->plan.a2a_rows_offrank;
      o->a2a_bytes_fwd = 2 * L->plan.a2a_rows_total * hb;
      int64_t ag = 0;
      for (auto& x : L->plan.ag_asm_send) ag += x.rows;
      for (auto& x : L->plan.ag_home_send) ag += x.rows;
      o->ag_bytes_fwd = ag * hb;
      o->ar_bytes_fwd = L->T > 1 ? L->plan.asm_rows * hb : 0;
      o->asm_rows = L->plan.asm_rows;
      for (int le = 0; le < L->Eloc && le < 64; ++le) o->kept_per_expert[le] = L->plan.seg_rows[le];
      if (L->direct) {
        // dispatch: my chunk's rows to 1 (or T with DTD) replicas of each expert's rank;
        // return: every kept token pulls T partial rows.  Local replicas move no NVLink bytes.
        const int my_c = L->dtd ? L->t : 0;
        int64_t rows = 0;
        for (int e = 0; e < E; ++e) {
          const int ep2 = e / L->Eloc;
          const int reps = L->dtd ? L->T : 1;
          const int local_reps = (ep2 == L->ep) ? 1 : 0;  // replica (t, ep) is this GPU
          rows += int64_t(kc[size_t(my_c) * E + e]) * (reps - local_reps);
          for (int c = 0; c < Tc; ++c)
            rows += int64_t(kc[size_t(c) * E + e]) * (L->T - local_reps);
        }
        o->peer_bytes_fwd = rows * hb;
        o->peer_exchange = 1;
        o->ar_bytes_fwd = 0;  // folded into the pulls
      }
    }
    int vd[2] = {1, 1};
    CU(cudaMemcpy(vd, L->verdict.p, sizeof(vd), cudaMemcpyDeviceToHost));
    o->placement_ok = vd[0];
    o->placement_ok_all = vd[1];
  });
}

int ted_layer_ledger(ted_layer* L, ted_ledger_entry* out, int reset) {
  return guard([&] {
    require(L != nullptr, "null layer");
    CU(cudaDeviceSynchronize());
    unsigned long long d[5 * 3 * 2];
    CU(cudaMemcpy(d, L->led.p, sizeof(d), cudaMemcpyDeviceToHost));
    if (out)
      for (int ph = 0; ph < 5; ++ph)
        for (int op = 0; op < 3; ++op) {
          out[ph * 3 + op].calls = d[(ph * 3 + op) * 2] + L->led_host[ph][op][0];
          out[ph * 3 + op].payload_bytes = d[(ph * 3 + op) * 2 + 1] + L->led_host[ph][op][1];
        }
    if (reset) {
      L->led.zero();
      std::memset(L->led_host, 0, sizeof(L->led_host));
    }
  });
}

int ted_layer_timing(ted_layer* L, int enable) {
  return guard([&] {
    require(L != nullptr, "null layer");
    CU(cudaDeviceSynchronize());
    L->timing = enable != 0;
    L->ev_used = 0;
    L->stage_ms.clear();
    L->stage_cnt.clear();
  });
}

// JSON {"stage": [total_ms, launches_of_stage], ...} of everything marked since enable.
int ted_layer_timing_read(ted_layer* L, char* out, int cap) {
  return guard([&] {
    require(L && out && cap > 0, "null argument");
    CU(cudaDeviceSynchronize());
    for (size_t i = 0; i + 1 < L->ev_used; ++i) {
      const char* nm = L->ev_names[i];
      if (!nm || nm[0] == '_') continue;
      float ms = 0.f;
      CU(cudaEventElapsedTime(&ms, L->evs[i], L->evs[i + 1]));
      L->stage_ms[nm] += ms;
      L->stage_cnt[nm] += 1;
    }
    L->ev_used = 0;
    std::string js = "{";
    bool first = true;
    for (auto& kv : L->stage_ms) {
      char buf[160];
      std::snprintf(buf, sizeof(buf), "%s\"%s\": [%.6f, %lld]", first ? "" : ", ",
                    kv.first.c_str(), kv.second, (long long)L->stage_cnt[kv.first]);
      js += buf;
      first = false;
    }
    js += "}";
    std::snprintf(out, size_t(cap), "%s", js.c_str());
  });
}

unsigned long long ted_kernel_launches(void) { return ted::launches(); }

int ted_layer_get_routing(ted_layer* L, int32_t* expert, float* prob, int32_t* slot,
                          int32_t* pos_home, float* probs, float* logits) {
  return guard([&] {
    require(L != nullptr, "null layer");
    CU(cudaDeviceSynchronize());
    const size_t n = size_t(L->n), nE = n * L->E;
    if (expert) CU(cudaMemcpy(expert, L->expert.p, n * 4, cudaMemcpyDeviceToHost));
    if (prob) CU(cudaMemcpy(prob, L->prob.p, n * 4, cudaMemcpyDeviceToHost));
    if (slot) CU(cudaMemcpy(slot, L->slot.p, n * 4, cudaMemcpyDeviceToHost));
    if (pos_home) CU(cudaMemcpy(pos_home, L->pos_home.p, n * 4, cudaMemcpyDeviceToHost));
    if (probs) CU(cudaMemcpy(probs, L->probs.p, nE * 4, cudaMemcpyDeviceToHost));
    if (logits) CU(cudaMemcpy(logits, L->logits.p, nE * 4, cudaMemcpyDeviceToHost));
  });
}


}  // extern "C"
