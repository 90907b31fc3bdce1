// model.cu -- the reference's whole model on B200: Trainer / MoeRank over `layers` layers
// (run_forward / run_backward moe.cpp:334-415, forward_layer :418-433, backward_layer
// :571-580 and :688-696).  Every layer is the attention stand-in block (column-parallel
// linear -> GELU -> row-parallel linear with its TP all-reduce, parallel_linear.cpp:8-40)
// followed by the MoE branch on even layers (layer_has_experts; a ted_layer, layer.cu) or
// a dense FFN block of the same shape on odd layers.  There is no residual path (the
// reference has none).  Loss = sum(y^2) / (2 N_global) over the last layer's output, dy =
// y / N_global (moe.cpp:379-391).
//
// Dense blocks run on the same tcgen05 grouped GEMM as the experts (one group, rows padded
// to the 128-row tile with zero rows, so the wgrad reductions see zeros), bias+GELU /
// dGELU fused into the epilogues, bias on TP rank 0 before the all-reduce (the reference
// adds it after the reduce), bias gradients by deterministic column sums.  All dense
// parameters of the model form one flat family in enumerate_params order (moe.cpp:115-147,
// without the gate weights, which the MoE layers own): one gradient all-reduce over the
// non-expert data group, one AdamW launch over the ZeRO-1 owned range, one completion
// all-gather (moe.cpp:699-734).
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <chrono>
#include <cmath>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/ted.h"
#include "ted_host.h"
#include "ted_internal.h"

using namespace ted;

namespace {

__global__ void dense_init_kernel(bf16* param, float* master, int64_t begin, int64_t end,
                                  int64_t off, int64_t rows, int64_t cols, int64_t ld,
                                  int64_t full_cols, int64_t col0, uint64_t seed, float scale) {
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
    const int64_t fi = off + r * ld + c;  // padded columns stay zero
    param[fi] = __float2bfloat16(v);
    if (fi >= begin && fi < end) master[fi - begin] = v;
  }
}

// loss partials: sum of squares of y (n x h bf16) per CTA, in double
__global__ void sumsq_kernel(const bf16* __restrict__ y, int64_t count, double* part) {
  __shared__ double s[8];
  double acc = 0.0;
  for (int64_t i = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) * 8; i < count;
       i += int64_t(gridDim.x) * blockDim.x * 8) {
    const uint4 u = *reinterpret_cast<const uint4*>(y + i);
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[q]));
      acc += double(f.x) * f.x + double(f.y) * f.y;
    }
  }
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < int(blockDim.x >> 5); ++w) t += s[w];
    part[blockIdx.x] = t;
  }
}

__global__ void loss_sum_kernel(const double* part, int nparts, double scale, double* loss) {
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < nparts; ++i) t += part[i];  // fixed order: deterministic
    *loss = t * scale;
  }
}

// dy = y / N_global (moe.cpp:390-391)
__global__ void scale_kernel(const bf16* __restrict__ y, int64_t count, float s,
                             bf16* __restrict__ dy) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
       i += int64_t(gridDim.x) * blockDim.x)
    dy[i] = __float2bfloat16(__bfloat162float(y[i]) * s);
}

constexpr int kLossCtas = 296;

}  // namespace

// one TP-sharded column -> GELU -> row block (attention stand-in or dense FFN)
struct DenseBlock {
  int64_t off = 0;  // family offset of [w1 h x fT | b1 fT | w2 fT x h | b2 h]
  DevBuf<bf16> z, hb;  // pre-activation (dZ in backward) and GELU output, np x fT
};

struct ted_model {
  ted_model_cfg model{};
  ted_topo_cfg topo{};
  ted_flags flags{};
  ted_adam_cfg adam{};
  ted_tile_cfg tiles{};
  double cf = 0.0;
  int shard_opt = 0, rank = 0;
  int layers = 0, h = 0, f = 0, fT = 0, E = 0, T = 1, P = 1, D = 1, world = 1, t = 0, ep = 0,
      d = 0;
  // the reference's hidden / inner widths; h and fT are zero-padded to the 256 tile (see
  // ted_layer: pads stay exactly zero, results are the unpadded ones)
  int hu = 0, fTu = 0;
  int64_t fam_u = 0;  // the reference's dense-family length (no padding)
  int64_t n = 0, np = 0, per_block = 0;
  ncclComm_t world_c = nullptr, tp_c = nullptr, dp_c = nullptr;
  std::vector<DenseBlock> attn, ffn;  // ffn used on odd layers
  std::vector<ted_layer*> moe;        // MoE branch on even layers
  Family fam;                         // every dense block's parameters
  std::vector<DevBuf<bf16>> xin;      // layer inputs (np x h, zero pad rows); xin[L] = output
  std::vector<DevBuf<bf16>> abuf;     // attention outputs (input of the MoE / FFN part)
  DevBuf<bf16> dy0, dy1, dmid, dpart;
  bool ckpt = false, cac = false;  // activation checkpointing; communication-avoiding recompute
  DevBuf<int> seg;                    // {0, np}
  DevBuf<float> col_part;
  DevBuf<double> loss_part, loss;
  HostBuf<double> h_loss;
  bool have_forward = false;
  double timeout_s = 120.0;  // collective_timeout (moe.hpp:96)
  std::string poisoned;
  // CommLedger entries of the dense blocks and the dense family ([phase][op][calls, bytes],
  // see ted_layer_ledger); the MoE layers keep their own
  unsigned long long led[5][3][2] = {};
  int phase = 0;  // ledger phase of the dense passes running now
};

namespace {

void model_abort(ted_model* M, const std::string& why) {
  M->poisoned = why;
  for (ted_layer* L : M->moe)
    if (L) layer_abort(L, why);
  for (ncclComm_t* c : {&M->tp_c, &M->dp_c, &M->world_c})
    if (*c) {
      ncclCommAbort(*c);
      *c = nullptr;
    }
  throw RuntimeError(why);
}

// the stack's failure state: its MoE layers' (plane-barrier timeouts, NCCL async errors)
// and its own communicators' asynchronous errors
void model_check(ted_model* M) {
  if (!M->poisoned.empty()) throw RuntimeError(M->poisoned + " (model unusable after the failure)");
  for (ted_layer* L : M->moe)
    if (L) {
      try {
        layer_check_fault(L);
      } catch (const std::exception& e) {
        model_abort(M, e.what());
      }
    }
  for (ncclComm_t c : {M->tp_c, M->dp_c, M->world_c}) {
    if (!c) continue;
    ncclResult_t r = ncclSuccess;
    if (ncclCommGetAsyncError(c, &r) == ncclSuccess && r != ncclSuccess && r != ncclInProgress)
      model_abort(M, std::string("NCCL asynchronous error: ") + ncclGetErrorString(r));
  }
}

// stream wait that cannot hang (see layer.cu wait_stream)
void model_wait(ted_model* M, cudaStream_t s) {
  const auto t0 = std::chrono::steady_clock::now();
  for (;;) {
    const cudaError_t q = cudaStreamQuery(s);
    if (q == cudaSuccess) break;
    if (q != cudaErrorNotReady) CU(q);
    model_check(M);
    const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (M->timeout_s > 0 && el > M->timeout_s && M->world > 1)
      model_abort(M, "TimeoutError: rank " + std::to_string(M->rank) +
                         ": the step did not complete within " + std::to_string(M->timeout_s) +
                         " s (a peer is stalled or gone; collective_timeout)");
    std::this_thread::sleep_for(std::chrono::microseconds(50));
  }
  model_check(M);
}

void dense_params(ted_model* M, int l, bool ffn, int64_t& off) {
  DenseBlock& B = ffn ? M->ffn[size_t(l)] : M->attn[size_t(l)];
  B.off = off;
  off += M->per_block;
  // one Z / H pair per block kind (recomputed): a layer's attention block must keep its
  // own through the FFN block's recompute and backward
  const bool first = ffn ? (l == 1) : (l == 0);
  if (M->ckpt && !first) {
    const DenseBlock& owner = ffn ? M->ffn[1] : M->attn[0];
    B.z.view(owner.z);
    B.hb.view(owner.hb);
    return;
  }
  B.z.alloc(size_t(M->np) * M->fT);
  B.z.zero();
  B.hb.alloc(size_t(M->np) * M->fT);
  B.hb.zero();
}

// GEMM1 + GELU only (the part of a block's forward its backward reads): the CAC recompute
// of a block whose row-parallel all-reduce output is still in place
void dense_gemm1(ted_model* M, DenseBlock& B, const bf16* X, cudaStream_t s) {
  bf16* P = M->fam.param.p + B.off;
  GemmParams g{};
  g.mode = GEMM_ROWS;
  g.groups = 1;
  g.seg_off = M->seg.p;
  GemmOperands o{};
  o.A = X;
  o.lda = M->h;
  o.B = P;
  o.ldb = M->fT;
  o.b_mn = true;
  g.epi = EPI_BIAS_GELU;
  g.N = M->fT;
  g.K = M->h;
  g.C = B.z.p;
  g.ldc = M->fT;
  g.bias = P + int64_t(M->h) * M->fT;
  g.aux = B.hb.p;
  g.ld_aux = M->fT;
  run_gemm(o, g, M->np, s);
}

void zero_pad_rows(ted_model* M, bf16* buf, cudaStream_t s) {
  if (M->np > M->n)
    CU(cudaMemsetAsync(buf + M->n * M->h, 0, sizeof(bf16) * size_t(M->np - M->n) * M->h, s));
}

// Y = row(GELU(column(X)))  (parallel_linear.cpp:8-31; nn.cpp:92-112)
void dense_forward(ted_model* M, DenseBlock& B, const bf16* X, bf16* Y, cudaStream_t s) {
  bf16* P = M->fam.param.p + B.off;
  const int64_t ow1 = 0, ob1 = int64_t(M->h) * M->fT, ow2 = ob1 + M->fT,
                ob2 = ow2 + int64_t(M->fT) * M->h;
  GemmParams g{};
  g.mode = GEMM_ROWS;
  g.groups = 1;
  g.seg_off = M->seg.p;
  GemmOperands o{};
  o.A = X;
  o.lda = M->h;
  o.B = P + ow1;
  o.ldb = M->fT;
  o.b_mn = true;
  g.epi = EPI_BIAS_GELU;
  g.N = M->fT;
  g.K = M->h;
  g.C = B.z.p;
  g.ldc = M->fT;
  g.bias = P + ob1;
  g.aux = B.hb.p;
  g.ld_aux = M->fT;
  run_gemm(o, g, M->np, s);
  o.A = B.hb.p;
  o.lda = M->fT;
  o.B = P + ow2;
  o.ldb = M->h;
  g.epi = (M->t == 0) ? EPI_BIAS : EPI_STORE;  // bias once, before the reduce (:29)
  g.N = M->h;
  g.K = M->fT;
  g.C = Y;
  g.ldc = M->h;
  g.bias = (M->t == 0) ? P + ob2 : nullptr;
  g.aux = nullptr;
  run_gemm(o, g, M->np, s);
  if (M->T > 1) {  // row-parallel partial sums (parallel_linear.cpp:28)
    NC(ncclAllReduce(Y, Y, size_t(M->n) * M->h, ncclBfloat16, ncclSum, M->tp_c, s));
    M->led[M->phase][0][0] += 1;
    M->led[M->phase][0][1] += uint64_t(M->n) * M->hu * 2;
  }
  zero_pad_rows(M, Y, s);
}

// dX from dY; weight / bias gradients into the family (parallel_linear.cpp:13-40)
void dense_backward(ted_model* M, DenseBlock& B, const bf16* X, const bf16* dY, bf16* dX,
                    cudaStream_t s) {
  bf16* P = M->fam.param.p + B.off;
  bf16* G = M->fam.grad.p + B.off;
  const int64_t ow1 = 0, ob1 = int64_t(M->h) * M->fT, ow2 = ob1 + M->fT,
                ob2 = ow2 + int64_t(M->fT) * M->h;
  const int h = M->h, fT = M->fT;
  // dZ = (dY W2^T) * gelu'(Z), in place over Z
  GemmParams g{};
  g.mode = GEMM_ROWS;
  g.groups = 1;
  g.seg_off = M->seg.p;
  g.epi = EPI_DGELU;
  g.N = fT;
  g.K = h;
  g.C = B.z.p;
  g.ldc = fT;
  g.aux = B.z.p;
  g.ld_aux = fT;
  GemmOperands o{};
  o.A = dY;
  o.lda = h;
  o.B = P + ow2;
  o.ldb = h;
  o.b_mn = false;
  run_gemm(o, g, M->np, s);
  // dW2 = H^T dY, db2 = colsum(dY)
  g = GemmParams{};
  g.mode = GEMM_KDIM;
  g.groups = 1;
  g.seg_off = M->seg.p;
  g.epi = EPI_STORE;
  g.M = fT;
  g.N = h;
  g.C = G + ow2;
  g.ldc = h;
  g.c_group_stride = int64_t(fT) * h;
  o = GemmOperands{};
  o.A = B.hb.p;
  o.lda = fT;
  o.a_mn = true;
  o.B = dY;
  o.ldb = h;
  o.b_mn = true;
  run_gemm(o, g, M->np, s);
  check(colsum_groups(dY, h, h, M->seg.p, 1, int(M->np), M->col_part.p, G + ob2, 0, s),
        "colsum db2");
  // dX = dZ W1^T (+ TP all-reduce), dW1 = X^T dZ, db1 = colsum(dZ)
  g = GemmParams{};
  g.mode = GEMM_ROWS;
  g.groups = 1;
  g.seg_off = M->seg.p;
  g.epi = EPI_STORE;
  g.N = h;
  g.K = fT;
  g.C = dX;
  g.ldc = h;
  o = GemmOperands{};
  o.A = B.z.p;
  o.lda = fT;
  o.B = P + ow1;
  o.ldb = fT;
  o.b_mn = false;
  run_gemm(o, g, M->np, s);
  g = GemmParams{};
  g.mode = GEMM_KDIM;
  g.groups = 1;
  g.seg_off = M->seg.p;
  g.epi = EPI_STORE;
  g.M = h;
  g.N = fT;
  g.C = G + ow1;
  g.ldc = fT;
  g.c_group_stride = int64_t(h) * fT;
  o = GemmOperands{};
  o.A = X;
  o.lda = h;
  o.a_mn = true;
  o.B = B.z.p;
  o.ldb = fT;
  o.b_mn = true;
  run_gemm(o, g, M->np, s);
  check(colsum_groups(B.z.p, fT, fT, M->seg.p, 1, int(M->np), M->col_part.p, G + ob1, 0, s),
        "colsum db1");
  if (M->T > 1) {  // column-parallel input gradient (parallel_linear.cpp:19)
    NC(ncclAllReduce(dX, dX, size_t(M->n) * h, ncclBfloat16, ncclSum, M->tp_c, s));
    M->led[2][0][0] += 1;
    M->led[2][0][1] += uint64_t(M->n) * M->hu * 2;
  }
  zero_pad_rows(M, dX, s);
}

std::string moe_name(const std::string& name) {  // "layer{l}.X" -> "layer0.X"
  const size_t dot = name.find('.');
  return "layer0" + name.substr(dot);
}

struct DenseLoc {
  int64_t off, rows, cols, full_cols;
  int axis;
  double scale;
  int64_t ld;  // row stride in the family (padded columns)
};

// name -> (layer, dense block or MoE); dense parameters are sliced like slice_tensor
// (tensor.cpp:56-98): w1/b1 by columns, w2 by rows, b2 replicated
bool parse(ted_model* M, const std::string& name, int& layer, std::string& blk,
           std::string& leaf) {
  if (name.compare(0, 5, "layer") != 0) return false;
  const size_t d1 = name.find('.');
  if (d1 == std::string::npos) return false;
  try {
    layer = std::stoi(name.substr(5, d1 - 5));
  } catch (...) {
    return false;
  }
  if (layer < 0 || layer >= M->layers) return false;
  const size_t d2 = name.find('.', d1 + 1);
  blk = name.substr(d1 + 1, d2 == std::string::npos ? std::string::npos : d2 - d1 - 1);
  leaf = d2 == std::string::npos ? "" : name.substr(d2 + 1);
  return true;
}

bool dense_lookup(ted_model* M, int layer, const std::string& blk, const std::string& leaf,
                  DenseLoc& out) {
  const bool moe_layer = (layer % 2) == 0;  // layer_has_experts (moe.cpp)
  if (!(blk == "attn" || (blk == "ffn" && !moe_layer))) return false;
  const int64_t base = (blk == "attn" ? M->attn : M->ffn)[size_t(layer)].off;
  const int h = M->h, fT = M->fT, f = M->f, hu = M->hu, fTu = M->fTu;
  const double sin = 1.0 / std::sqrt(double(hu)), sout = 1.0 / std::sqrt(double(f));
  const int64_t ob1 = int64_t(h) * fT, ow2 = ob1 + fT, ob2 = ow2 + int64_t(fT) * h;
  if (leaf == "w1") out = {base, hu, fTu, f, 1, sin, fT};
  else if (leaf == "b1") out = {base + ob1, 1, fTu, f, 1, 0.1, fT};
  else if (leaf == "w2") out = {base + ow2, fTu, hu, hu, 2, sout, h};
  else if (leaf == "b2") out = {base + ob2, 1, hu, hu, 0, 0.1, h};
  else return false;
  return true;
}

void family_adam(ted_model* M, cudaStream_t s) {
  Family& F = M->fam;
  if (F.elems == 0) return;
  if (F.reset) {
    CU(cudaMemsetAsync(F.m1.p, 0, sizeof(float) * F.m1.n, s));
    CU(cudaMemsetAsync(F.m2.p, 0, sizeof(float) * F.m2.n, s));
    CU(cudaMemsetAsync(F.dstep.p, 0, sizeof(long long), s));
    F.reset = false;
  }
  check(adam_prep(F.dstep.p, F.dcoef.p, M->adam.beta1, M->adam.beta2, s), "adam_prep");
  const int64_t owned = F.end - F.begin;
  const int64_t tile = M->tiles.enabled ? std::min<int64_t>(M->tiles.tile_size, std::max<int64_t>(owned, 1))
                                        : std::max<int64_t>(owned, 1);
  F.upcast_peak = std::max<uint64_t>(F.upcast_peak, owned == 0 ? 0 : uint64_t(tile) * 4);
  check(adam_step(F.master.p, F.m1.p, F.m2.p, F.param.p, F.grad.p, F.begin, F.end, tile,
                  float(M->adam.lr), float(M->adam.beta1), float(M->adam.beta2),
                  float(1.0 - M->adam.beta1), float(1.0 - M->adam.beta2), float(M->adam.eps),
                  float(M->adam.weight_decay), 1.f, 1.f, F.dcoef.p, s),
        "adam_step");
  if (F.group > 1) {  // ZeRO-1 completion, zero-padded equal chunks (moe.cpp:718-732)
    bf16* gbuf = F.gather.p;
    CU(cudaMemsetAsync(gbuf + F.pos * F.chunk, 0, sizeof(bf16) * F.chunk, s));
    CU(cudaMemcpyAsync(gbuf + F.pos * F.chunk, F.param.p + F.begin, sizeof(bf16) * owned,
                       cudaMemcpyDeviceToDevice, s));
    NC(ncclAllGather(gbuf + F.pos * F.chunk, gbuf, size_t(F.chunk), ncclBfloat16, M->dp_c, s));
    M->led[4][1][0] += 1;
    M->led[4][1][1] += uint64_t((M->fam_u + F.group - 1) / F.group) * 2;
    for (int q = 0; q < F.group; ++q) {
      if (q == F.pos) continue;
      const int64_t b = shard_lo(F.elems, F.group, q), e = shard_lo(F.elems, F.group, q + 1);
      if (e > b)
        CU(cudaMemcpyAsync(F.param.p + b, gbuf + q * F.chunk, sizeof(bf16) * (e - b),
                           cudaMemcpyDeviceToDevice, s));
    }
  }
}

void create_model(ted_model* M, const ted_model_cfg* model, const ted_topo_cfg* topo,
                  const ted_flags* flags, const ted_adam_cfg* adam, const ted_tile_cfg* tiles,
                  double cf, int shard_opt, int rank, const void* uid) {
  require(model && topo && flags && adam && tiles, "null config pointer");
  M->model = *model;
  M->topo = *topo;
  M->flags = *flags;
  M->adam = *adam;
  M->tiles = *tiles;
  M->cf = cf;
  M->shard_opt = shard_opt;
  M->rank = rank;
  require(model->layers >= 1, "layers must be >= 1, got " + std::to_string(model->layers));
  require(model->hidden >= 1 && model->experts >= 1 && model->tokens_per_shard >= 1,
          "model: hidden, experts and tokens_per_shard must be >= 1");
  // ckpt: keep only every layer's input and recompute the layer before its backward
  // (moe.cpp:343-375, :393-415); cac (with ckpt): the recompute replays the stashed
  // collective outputs instead of communicating (channel.cpp:20-51)
  M->ckpt = flags->ckpt != 0;
  M->cac = M->ckpt && flags->cac != 0;
  M->layers = model->layers;
  M->hu = model->hidden;
  M->h = (M->hu + 255) / 256 * 256;
  M->f = 4 * M->hu;
  M->E = model->experts;
  M->n = model->tokens_per_shard;
  M->T = topo->tensor_parallel;
  M->P = topo->experts;
  M->world = topo->world_size;
  require(M->T >= 1 && M->P >= 1 && M->world % (M->T * M->P) == 0,
          "world_size must be a multiple of tensor_parallel * experts");
  M->D = M->world / (M->T * M->P);
  require(rank >= 0 && rank < M->world, "rank out of range");
  require(M->f % M->T == 0, "4*hidden must divide by tensor_parallel");
  M->fTu = M->f / M->T;
  M->fT = (M->fTu + 255) / 256 * 256;
  M->t = rank % M->T;
  M->ep = (rank / M->T) % M->P;
  M->d = rank / (M->T * M->P);
  M->np = ((M->n + 127) / 128) * 128;
  M->per_block = 2 * int64_t(M->h) * M->fT + M->fT + M->h;
  require_device();
  // communicators: world, TP (fixed e, d) and the non-expert data group (fixed t)
  // (topology.cpp:56-93); every MoE layer splits its own from the world communicator
  if (M->world > 1) {
    require(uid != nullptr, "world_size > 1 needs an NCCL unique id");
    ncclUniqueId id;
    std::memcpy(&id, uid, sizeof(id));
    NC(ncclCommInitRank(&M->world_c, M->world, id, rank));
    NC(ncclCommSplit(M->world_c, M->ep + M->P * M->d, M->t, &M->tp_c, nullptr));
    NC(ncclCommSplit(M->world_c, M->t, M->ep + M->P * M->d, &M->dp_c, nullptr));
  }
  // dense parameter family in enumerate_params order
  M->attn.resize(size_t(M->layers));
  M->ffn.resize(size_t(M->layers));
  int64_t off = 0;
  for (int l = 0; l < M->layers; ++l) {
    dense_params(M, l, false, off);
    if (l % 2 == 1) dense_params(M, l, true, off);
  }
  Family& F = M->fam;
  F.elems = off;
  M->fam_u = int64_t(M->layers + M->layers / 2) * (2 * int64_t(M->hu) * M->fTu + M->fTu + M->hu);
  F.group = shard_opt ? M->P * M->D : 1;
  F.pos = shard_opt ? M->ep + M->P * M->d : 0;
  F.begin = shard_lo(F.elems, F.group, F.pos);
  F.end = shard_lo(F.elems, F.group, F.pos + 1);
  F.chunk = (F.elems + F.group - 1) / F.group;
  F.param.alloc(size_t(F.elems + 8));
  F.param.zero();
  F.grad.alloc(size_t(F.elems + 8));
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
  // MoE layers (even layers)
  M->moe.assign(size_t(M->layers), nullptr);
  ted_model_cfg one = *model;
  one.layers = 1;
  ted_flags lf = *flags;  // checkpointing is the stack's business, not the layer's
  lf.ckpt = 0;
  lf.cac = 0;
  for (int l = 0; l < M->layers; l += 2) {
    ted_layer* L = nullptr;
    ted_layer* share = (M->ckpt && l > 0) ? M->moe[0] : nullptr;
    if (layer_create_child(&one, topo, &lf, adam, tiles, cf, shard_opt, rank, M->world_c, share,
                           &L) != TED_OK)
      throw RuntimeError(std::string("layer ") + std::to_string(l) + ": " + last_error());
    M->moe[size_t(l)] = L;
  }
  // activations
  M->xin.resize(size_t(M->layers + 1));
  M->abuf.resize(size_t(M->layers));
  for (auto& b : M->xin) {
    b.alloc(size_t(M->np) * M->h);
    b.zero();
  }
  for (size_t l = 0; l < M->abuf.size(); ++l) {
    if (M->ckpt && !M->cac && l > 0) {  // recomputed: one buffer (with CAC it is the stash
      M->abuf[l].view(M->abuf[0]);       // of the attention block's all-reduce output)
      continue;
    }
    M->abuf[l].alloc(size_t(M->np) * M->h);
    M->abuf[l].zero();
  }
  for (DevBuf<bf16>* b : {&M->dy0, &M->dy1, &M->dmid, &M->dpart}) {
    b->alloc(size_t(M->np) * M->h);
    b->zero();
  }
  std::vector<int> seg = {0, int(M->np)};
  M->seg.alloc(2);
  CU(cudaMemcpy(M->seg.p, seg.data(), sizeof(int) * 2, cudaMemcpyHostToDevice));
  M->col_part.alloc(colsum_part_floats(std::max(M->h, M->fT), 1, int(M->np)) + 64);
  M->loss_part.alloc(kLossCtas);
  M->loss.alloc(1);
  M->loss.zero();
  M->h_loss.alloc(1);
  CU(cudaDeviceSynchronize());
}

void model_forward(ted_model* M, const bf16* batch, cudaStream_t s) {
  const int h = M->h;
  M->phase = 0;
  // the caller's [n][hu] batch into the zero-padded [np][h] input
  CU(cudaMemcpy2DAsync(M->xin[0].p, size_t(h) * 2, batch, size_t(M->hu) * 2, size_t(M->hu) * 2,
                       size_t(M->n), cudaMemcpyDeviceToDevice, s));
  for (int l = 0; l < M->layers; ++l) {
    dense_forward(M, M->attn[size_t(l)], M->xin[size_t(l)].p, M->abuf[size_t(l)].p, s);
    if (l % 2 == 0) {
      layer_set_forward_mode(M->moe[size_t(l)], M->cac ? FWD_RECORD : FWD_LIVE);
      const int rc = ted_layer_forward(M->moe[size_t(l)],
                                       reinterpret_cast<const uint16_t*>(M->abuf[size_t(l)].p),
                                       reinterpret_cast<uint16_t*>(M->xin[size_t(l + 1)].p), s);
      if (rc != TED_OK) throw RuntimeError(last_error());
    } else {
      dense_forward(M, M->ffn[size_t(l)], M->abuf[size_t(l)].p, M->xin[size_t(l + 1)].p, s);
    }
  }
  const double nglob = double(M->n) * M->P * M->D;
  const int64_t cnt = M->n * h;
  sumsq_kernel<<<kLossCtas, 256, 0, s>>>(M->xin[size_t(M->layers)].p, cnt, M->loss_part.p);
  loss_sum_kernel<<<1, 32, 0, s>>>(M->loss_part.p, kLossCtas, 1.0 / (2.0 * nglob), M->loss.p);
  count_launch(2);
  CU(cudaGetLastError());
  M->have_forward = true;
}

// the layer's forward again from its checkpointed input (Phase::Recompute, moe.cpp:396-404):
// live, or with CAC replaying the recorded collective outputs (the attention / FFN
// all-reduce outputs are still in abuf / xin, the MoE exchange outputs in the layer's
// stash), in which case only the GEMM1 + GELU the backward reads are recomputed
void recompute_layer(ted_model* M, int l, cudaStream_t s) {
  const bool replay = M->cac && M->world > 1;
  M->phase = 1;  // Phase::Recompute
  DenseBlock& A = M->attn[size_t(l)];
  if (replay) dense_gemm1(M, A, M->xin[size_t(l)].p, s);
  else dense_forward(M, A, M->xin[size_t(l)].p, M->abuf[size_t(l)].p, s);
  if (l % 2 == 0) {
    ted_layer* L = M->moe[size_t(l)];
    layer_set_forward_mode(L, M->cac ? FWD_REPLAY : FWD_LIVE);
    layer_set_ledger_phase(L, 1);
    const int rc = ted_layer_forward(L, reinterpret_cast<const uint16_t*>(M->abuf[size_t(l)].p),
                                     reinterpret_cast<uint16_t*>(M->dpart.p), s);
    layer_set_ledger_phase(L, 0);
    layer_set_forward_mode(L, FWD_LIVE);
    if (rc != TED_OK) throw RuntimeError(last_error());
  } else if (replay) {
    dense_gemm1(M, M->ffn[size_t(l)], M->abuf[size_t(l)].p, s);
  } else {
    dense_forward(M, M->ffn[size_t(l)], M->abuf[size_t(l)].p, M->dpart.p, s);
  }
}

void model_backward(ted_model* M, cudaStream_t s, bool step_follows = false) {
  if (!M->have_forward) throw ConfigError("backward called before forward");
  const int h = M->h;
  const double nglob = double(M->n) * M->P * M->D;
  scale_kernel<<<sm_count() * 4, 256, 0, s>>>(M->xin[size_t(M->layers)].p, M->n * h,
                                              float(1.0 / nglob), M->dy0.p);
  count_launch(1);
  CU(cudaGetLastError());
  bf16* dy = M->dy0.p;
  bf16* dx = M->dy1.p;
  for (int l = M->layers - 1; l >= 0; --l) {
    if (M->ckpt) recompute_layer(M, l, s);
    M->phase = 2;  // Phase::Backward
    if (l % 2 == 0) {
      if (step_follows) {
        layer_backward_then_step(M->moe[size_t(l)], dy, M->dmid.p, s);
      } else {
        const int rc = ted_layer_backward(M->moe[size_t(l)],
                                          reinterpret_cast<const uint16_t*>(dy),
                                          reinterpret_cast<uint16_t*>(M->dmid.p), s);
        if (rc != TED_OK) throw RuntimeError(last_error());
      }
    } else {
      dense_backward(M, M->ffn[size_t(l)], M->abuf[size_t(l)].p, dy, M->dmid.p, s);
    }
    dense_backward(M, M->attn[size_t(l)], M->xin[size_t(l)].p, M->dmid.p, dx, s);
    std::swap(dy, dx);
  }
  M->have_forward = false;
}

void model_optimizer(ted_model* M, cudaStream_t s) {
  // run_grad_sync (moe.cpp:699-711) for the dense family, then AdamW; the MoE layers sync
  // and step their own families (gate + experts)
  if (M->P * M->D > 1) {
    NC(ncclAllReduce(M->fam.grad.p, M->fam.grad.p, size_t(M->fam.elems), ncclBfloat16, ncclSum,
                     M->dp_c, s));
    M->led[3][0][0] += 1;
    M->led[3][0][1] += uint64_t(M->fam_u) * 2;
  }
  family_adam(M, s);
  for (ted_layer* L : M->moe)
    if (L && ted_layer_optimizer_step(L, s) != TED_OK) throw RuntimeError(last_error());
}

}  // namespace

extern "C" {

int ted_model_create(const ted_model_cfg* model, const ted_topo_cfg* topo, const ted_flags* flags,
                     const ted_adam_cfg* adam, const ted_tile_cfg* tiles, double capacity_factor,
                     int shard_optimizer, int rank, const void* nccl_uid, ted_model** out) {
  return guard([&] {
    require(out != nullptr, "null output pointer");
    auto* M = new ted_model();
    try {
      create_model(M, model, topo, flags, adam, tiles, capacity_factor, shard_optimizer, rank,
                   nccl_uid);
    } catch (...) {
      ted_model_destroy(M);
      throw;
    }
    *out = M;
  });
}

void ted_model_destroy(ted_model* M) {
  if (!M) return;
  cudaDeviceSynchronize();
  for (ted_layer* L : M->moe) ted_layer_destroy(L);
  for (ncclComm_t* c : {&M->tp_c, &M->dp_c, &M->world_c})
    if (*c) {
      ncclCommDestroy(*c);
      *c = nullptr;
    }
  delete M;
}

int ted_model_set_param(ted_model* M, const char* name, const float* full) {
  return guard([&] {
    require(M && name && full, "null argument");
    int layer = 0;
    std::string blk, leaf;
    require(parse(M, name, layer, blk, leaf), std::string("no parameter named ") + name);
    if (blk == "gate" || blk.compare(0, 6, "expert") == 0) {
      require(layer % 2 == 0, std::string("no parameter named ") + name);
      if (blk != "gate") {  // experts housed on other EP ranks: nothing to set here
        int e = -1;
        try {
          e = std::stoi(blk.substr(6));
        } catch (...) {
        }
        require(e >= 0 && e < M->E, std::string("no parameter named ") + name);
        if (e / (M->E / M->P) != M->ep) return;
      }
      const int rc = ted_layer_set_param(M->moe[size_t(layer)], moe_name(name).c_str(), full);
      if (rc == TED_ERR_CONFIG) throw ConfigError(last_error());
      if (rc != TED_OK) throw RuntimeError(last_error());
      return;
    }
    DenseLoc dl;
    require(dense_lookup(M, layer, blk, leaf, dl), std::string("no parameter named ") + name);
    std::vector<float> shard(size_t(dl.rows * dl.ld), 0.f);  // family layout, pads zero
    for (int64_t r = 0; r < dl.rows; ++r)
      for (int64_t c = 0; c < dl.cols; ++c) {
        int64_t fr = r, fc = c;
        if (dl.axis == 1) fc = c + int64_t(M->t) * dl.cols;
        if (dl.axis == 2) fr = r + int64_t(M->t) * dl.rows;
        shard[size_t(r * dl.ld + c)] = full[fr * dl.full_cols + fc];
      }
    std::vector<uint16_t> b(shard.size());
    for (size_t i = 0; i < b.size(); ++i) b[i] = f2bf(shard[i]);
    Family& F = M->fam;
    CU(cudaDeviceSynchronize());  // a step in flight on a non-blocking stream may still write
    CU(cudaMemcpy(F.param.p + dl.off, b.data(), b.size() * 2, cudaMemcpyHostToDevice));
    const int64_t lo = std::max(dl.off, F.begin),
                  hi = std::min(dl.off + int64_t(b.size()), F.end);
    if (hi > lo)
      CU(cudaMemcpy(F.master.p + (lo - F.begin), shard.data() + (lo - dl.off),
                    sizeof(float) * (hi - lo), cudaMemcpyHostToDevice));
    F.reset = true;
  });
}

static int model_get(ted_model* M, const char* name, float* out, int64_t* numel, bool grad) {
  return guard([&] {
    require(M && name, "null argument");
    int layer = 0;
    std::string blk, leaf;
    require(parse(M, name, layer, blk, leaf), std::string("no parameter named ") + name);
    if (blk == "gate" || blk.compare(0, 6, "expert") == 0) {
      require(layer % 2 == 0, std::string("no parameter named ") + name);
      const std::string nm = moe_name(name);
      const int rc = grad ? ted_layer_get_grad(M->moe[size_t(layer)], nm.c_str(), out, numel)
                          : ted_layer_get_param(M->moe[size_t(layer)], nm.c_str(), out, numel);
      if (rc == TED_ERR_CONFIG) throw ConfigError(last_error());
      if (rc != TED_OK) throw RuntimeError(last_error());
      return;
    }
    DenseLoc dl;
    require(dense_lookup(M, layer, blk, leaf, dl), std::string("no parameter named ") + name);
    const int64_t cnt = dl.rows * dl.cols;
    if (numel) *numel = cnt;
    if (!out) return;
    std::vector<uint16_t> b(static_cast<size_t>(dl.rows * dl.ld));
    CU(cudaDeviceSynchronize());
    CU(cudaMemcpy(b.data(), (grad ? M->fam.grad.p : M->fam.param.p) + dl.off, b.size() * 2,
                  cudaMemcpyDeviceToHost));
    for (int64_t r = 0; r < dl.rows; ++r)
      for (int64_t c = 0; c < dl.cols; ++c) out[r * dl.cols + c] = bf2f(b[size_t(r * dl.ld + c)]);
  });
}

int ted_model_get_param(ted_model* M, const char* name, float* out, int64_t* numel) {
  return model_get(M, name, out, numel, false);
}
int ted_model_get_grad(ted_model* M, const char* name, float* out, int64_t* numel) {
  return model_get(M, name, out, numel, true);
}

int ted_model_keep_grads(ted_model* M, int keep) {
  return guard([&] {
    require(M != nullptr, "null model");
    for (ted_layer* L : M->moe)
      if (L && ted_layer_keep_grads(L, keep) != TED_OK) throw RuntimeError(last_error());
  });
}

int ted_model_init_params(ted_model* M, uint64_t seed) {
  return guard([&] {
    require(M != nullptr, "null model");
    CU(cudaDeviceSynchronize());  // after any step still in flight
    for (int l = 0; l < M->layers; ++l) {
      for (const char* blk : {"attn", "ffn"}) {
        if (std::strcmp(blk, "ffn") == 0 && l % 2 == 0) continue;
        for (const char* leaf : {"w1", "b1", "w2", "b2"}) {
          const std::string nm = "layer" + std::to_string(l) + "." + blk + "." + leaf;
          DenseLoc dl;
          dense_lookup(M, l, blk, leaf, dl);
          int64_t col0 = 0;
          if (dl.axis == 1) col0 = int64_t(M->t) * dl.cols;
          if (dl.axis == 2) col0 = int64_t(M->t) * dl.rows * dl.cols;
          uint64_t hs = 14695981039346656037ULL;
          for (unsigned char c : nm) hs = (hs ^ c) * 1099511628211ULL;
          dense_init_kernel<<<sm_count() * 4, 256>>>(M->fam.param.p, M->fam.master.p,
                                                     M->fam.begin, M->fam.end, dl.off, dl.rows,
                                                     dl.cols, dl.ld, dl.full_cols, col0,
                                                     seed * 0x9E3779B97F4A7C15ULL + hs,
                                                     float(dl.scale));
          CU(cudaGetLastError());
        }
      }
      if (l % 2 == 0) {
        const int rc = ted_layer_init_params(M->moe[size_t(l)],
                                             seed * 0x9E3779B97F4A7C15ULL + uint64_t(l) + 1);
        if (rc != TED_OK) throw RuntimeError(last_error());
      }
    }
    M->fam.reset = true;
    CU(cudaDeviceSynchronize());
  });
}

int ted_model_forward(ted_model* M, const uint16_t* batch, void* stream) {
  return guard([&] {
    require(M && batch, "null argument");
    model_check(M);
    model_forward(M, reinterpret_cast<const bf16*>(batch), S(stream));
  });
}

int ted_model_backward(ted_model* M, void* stream) {
  return guard([&] {
    require(M != nullptr, "null model");
    model_check(M);
    model_backward(M, S(stream));
  });
}

int ted_model_optimizer_step(ted_model* M, void* stream) {
  return guard([&] {
    require(M != nullptr, "null model");
    model_check(M);
    model_optimizer(M, S(stream));
  });
}

int ted_model_step(ted_model* M, const uint16_t* batch, void* stream) {
  return guard([&] {
    require(M && batch, "null argument");
    model_check(M);
    const cudaStream_t s = S(stream);
    model_forward(M, reinterpret_cast<const bf16*>(batch), s);
    model_backward(M, s, /*step_follows=*/true);
    model_optimizer(M, s);
  });
}

int ted_model_loss(ted_model* M, double* loss, void* stream) {
  return guard([&] {
    require(M && loss, "null argument");
    CU(cudaMemcpyAsync(M->h_loss.p, M->loss.p, sizeof(double), cudaMemcpyDeviceToHost,
                       S(stream)));  // pinned: see ted_layer_loss
    model_wait(M, S(stream));
    *loss = *M->h_loss.p;
  });
}

int ted_model_ledger(ted_model* M, ted_ledger_entry* out, int reset) {
  return guard([&] {
    require(M != nullptr, "null model");
    ted_ledger_entry acc[15] = {};
    for (int ph = 0; ph < 5; ++ph)
      for (int op = 0; op < 3; ++op) {
        acc[ph * 3 + op].calls = M->led[ph][op][0];
        acc[ph * 3 + op].payload_bytes = M->led[ph][op][1];
      }
    for (ted_layer* L : M->moe)
      if (L) {
        ted_ledger_entry one[15];
        if (ted_layer_ledger(L, one, reset) != TED_OK) throw RuntimeError(last_error());
        for (int i = 0; i < 15; ++i) {
          acc[i].calls += one[i].calls;
          acc[i].payload_bytes += one[i].payload_bytes;
        }
      }
    if (out) std::memcpy(out, acc, sizeof(acc));
    if (reset) std::memset(M->led, 0, sizeof(M->led));
  });
}

int ted_model_set_timeout(ted_model* M, double seconds) {
  return guard([&] {
    require(M != nullptr, "null model");
    require(seconds >= 0, "timeout must be >= 0 (0 = no limit)");
    M->timeout_s = seconds;
    for (ted_layer* L : M->moe)
      if (L) {
        const int rc = ted_layer_set_timeout(L, seconds);
        if (rc != TED_OK) throw RuntimeError(ted_last_error());
      }
  });
}

int ted_model_memory(ted_model* M, int64_t* out) {
  return guard([&] {
    require(M && out, "null argument");
    int64_t act = 0, par = 0, stash = 0;
    for (ted_layer* L : M->moe)
      if (L) {
        int64_t a = 0, p = 0, st = 0;
        layer_memory(L, &a, &p, &st);
        act += a;
        par += p;
        stash += st;
      }
    for (const auto* v : {&M->attn, &M->ffn})
      for (const DenseBlock& B : *v) act += int64_t(B.z.bytes() + B.hb.bytes());
    int64_t ckpt = 0;
    for (size_t l = 0; l < M->abuf.size(); ++l) {
      if (M->cac && M->world > 1) stash += int64_t(M->abuf[l].bytes());  // attn AR outputs
      else act += int64_t(M->abuf[l].bytes());
    }
    for (const auto& b : M->xin) ckpt += int64_t(b.bytes());  // layer inputs (+ output)
    for (const DevBuf<bf16>* b : {&M->dy0, &M->dy1, &M->dmid, &M->dpart})
      act += int64_t(b->bytes());
    const Family& F = M->fam;
    par += int64_t(F.param.bytes() + F.grad.bytes() + F.gather.bytes() + F.master.bytes() +
                   F.m1.bytes() + F.m2.bytes());
    out[0] = par;    // parameters, gradients, optimizer state
    out[1] = act;    // activations and workspaces
    out[2] = ckpt;   // layer inputs kept for the backward / recompute
    out[3] = stash;  // CAC stash of collective outputs
  });
}

int ted_model_output(ted_model* M, uint16_t* y, void* stream) {
  return guard([&] {
    require(M && y, "null argument");
    CU(cudaMemcpy2DAsync(y, size_t(M->hu) * 2, M->xin[size_t(M->layers)].p, size_t(M->h) * 2,
                         size_t(M->hu) * 2, size_t(M->n), cudaMemcpyDeviceToDevice, S(stream)));
  });
}

}  // extern "C"
