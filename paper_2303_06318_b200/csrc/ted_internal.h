// ted_internal.h -- internal (C++) declarations shared by the TED kernels and the host
// driver.  Not part of the C ABI (that is include/ted.h).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

namespace ted {

using bf16 = __nv_bfloat16;

void set_error(const std::string& m);
unsigned long long launches();
void count_launch(int k);
const char* last_error();

// ------------------------------------------------------------------ grouped GEMM
enum GemmMode { GEMM_ROWS = 0, GEMM_KDIM = 1 };
enum EpiKind { EPI_STORE = 0, EPI_BIAS = 1, EPI_BIAS_GELU = 2, EPI_DGELU = 3, EPI_ADAM = 4 };

// Optimizer-state layout of the expert weight matrices when AdamW is fused into the wgrad
// epilogue ("tile-major"): each 128x256 GEMM output tile's state is one contiguous 128 KB
// run (tiles row-major over the matrix), inside it sixteen 32x64 warp shares (sub-partition
// sp = row/32, column quarter cq) of four 32x16 fp32 half blocks (2 KB) each; inside a
// half block, 4-column chunk j of row r sits at j * 128 + r * 4.  The epilogue warp that
// owns rows r0..r0+31 of a half tile (one TMEM lane per row) thus moves each chunk with one
// fully coalesced 512 B access, and the SMs working on consecutive tiles stream through
// consecutive memory like an elementwise kernel.  Parameters and gradients stay row-major.
// Needs rows % 128 == 0 and cols % 256 == 0.  Element offset of (r, c) in a rows x cols
// matrix:
__host__ __device__ inline int64_t blk_off(int64_t r, int64_t c, int64_t cols) {
  const int64_t rr = r & 127, cc = c & 255;
  const int64_t share = ((rr >> 5) << 2) + (cc >> 6);
  return (((r >> 7) * (cols >> 8) + (c >> 8)) << 15) + ((share << 2) + ((cc >> 4) & 3)) * 512 +
         ((cc >> 2) & 3) * 128 + (rr & 31) * 4 + (cc & 3);
}

// AdamW hyper-parameters as the kernels use them (AdamConfig, optimizer.hpp:17-23; omb = 1 - beta)
struct AdamK {
  float lr, b1, b2, omb1, omb2, eps, wd;
};

struct GemmParams {
  int mode;  // GemmMode
  int epi;   // EpiKind
  int groups;
  int M, N, K;          // ROWS: N, K fixed (M per group); KDIM: M, N fixed (K per group)
  const int* seg_off;   // device [groups+1]: padded (x128) row offsets of each group
  bf16* C;
  int64_t ldc;
  int64_t c_group_stride;  // KDIM: C_g = C + g * c_group_stride
  const bf16* bias;        // EPI_BIAS*: bias_g = bias + g * bias_group_stride (nullable)
  int64_t bias_group_stride;
  bf16* aux;  // EPI_BIAS_GELU: H output; EPI_DGELU: Z input (may alias C)
  int64_t ld_aux;
  // EPI_ADAM (KDIM only): the wgrad tile is the gradient of the parameter block at the
  // same [g][row][col] of these arrays (all laid out like C); AdamW is applied in the
  // epilogue and C (the bf16 gradient) is never written.  C is the bf16 parameter output.
  float* adam_master = nullptr;
  float* adam_m1 = nullptr;
  float* adam_m2 = nullptr;
  const float* adam_coef = nullptr;  // device {1/(1-b1^t), 1/(1-b2^t)}
  bf16* adam_grad = nullptr;  // non-null: also store the bf16 gradient tile (laid out like C)
  // EPI_DGELU (ROWS mode): also write the 32-row column-sum partials of dZ (bias gradient,
  // the colsum_groups partial layout [row split][group][N]) -- skips a pass over dZ
  float* colsum_part = nullptr;
  // (EPI_ADAM: master/m1/m2 use the blk_off layout per group, group stride c_group_stride)
  AdamK adam{};
  // push return (ROWS mode, EPI_STORE / EPI_BIAS): output row r of the assembled buffer is
  // not stored in C but sent over NVLink to row row_home[r] of slot push_slot in the receive
  // buffer of every TP member td of its home shard row_src[r]:
  // push_peers[td + push_T * row_src[r]] + push_slot * push_slot_stride + row_home[r] * N
  const unsigned long long* push_peers = nullptr;
  const int* row_home = nullptr;
  const int* row_src = nullptr;
  int push_T = 1, push_slot = 0;
  int64_t push_slot_stride = 0;
  int band = 0;  // KDIM raster: row blocks (tile pairs) per band (0: the default)
  int state_policy = 0;  // AdamW state L2 hints: bit 0 plain loads, bit 1 plain stores
  int operand_hint = 0;  // AdamW wgrad: operand TMA loads with an L2 evict-last policy
};

struct GemmOperands {
  const bf16* A;
  int64_t lda;
  bool a_mn;
  const bf16* B;
  int64_t ldb;
  int64_t b_group_stride;
  bool b_mn;
};

int sm_count();
// 2-D bf16 K-major TMA map (SWIZZLE_128B), boxes of box_cols x box_rows (gemm_sm100.cu)
bool tmap_bf16_2d(CUtensorMap* m, const void* base, uint64_t cols, uint64_t rows,
                  uint64_t row_bytes, uint32_t box_cols, uint32_t box_rows);
// max_rows = number of rows the A/B row dimension spans (for the TMA bounds).
cudaError_t grouped_gemm(const GemmOperands& o, const GemmParams& p, int max_rows,
                         cudaStream_t s, const char** why);

// ------------------------------------------------------------------ routing kernels
constexpr int kRouteBlock = 64;  // tokens per routing block (gate / scan / dispatch)
constexpr int kPad = 128;         // expert segments are padded to the GEMM M tile

// top-1 gate: logits = a Wg (fp32 accumulate), argmax (lowest index on ties), softmax.
// wgT: scratch of gate_wgt_elems(h, E) bf16 (nullptr: the mma.sync variant with the gate
// weight staged in shared memory runs); with it Wg^T is transposed once per call and the
// logits run on tcgen05 with TMA-streamed token rows (gate_sm100.cu).
size_t gate_wgt_elems(int h, int E);
// the tcgen05 gate (gate_sm100.cu): wgT [gate_tc_experts(E)][h], zero rows e >= E
int gate_tc_experts(int E);
cudaError_t gate_forward_tc(const bf16* a, const bf16* wgT, int64_t n, int h, int E,
                            float* logits, float* probs, int* expert, float* prob,
                            int* blk_hist, cudaStream_t s);
cudaError_t gate_forward(const bf16* a, const bf16* wg, int64_t n, int h, int E, float* logits,
                         float* probs, int* expert, float* prob, int* blk_hist, bf16* wgT,
                         cudaStream_t s);
// Routing from caller-provided fp32 logits (same selection/softmax code path).
cudaError_t gate_route_logits(const float* logits, int64_t n, int E, float* probs, int* expert,
                              float* prob, int* blk_hist, cudaStream_t s);

struct RouteScanArgs {
  int64_t n;
  int E;
  int T;           // token chunks (DTD: tensor-parallel degree; else 1)
  int my_chunk;    // chunk this rank dispatches (DTD), -1 = all chunks (no DTD)
  int64_t cap;     // capacity C per expert per source shard (>= n: unlimited)
  int local;       // 1: single-rank layout (send == home == padded expert segments)
  const int* expert;
  const int* blk_hist;  // [nblk][E]
  int* blk_prefix;      // [nblk][E] out
  int* chunk_prefix;    // [(T+1)][E] out: S[c][e]
  int* kc;              // [T][E] out: kept tokens per (chunk, expert)
  int* send_base;       // [E] out
  int* home_base;       // [T][E] out
  int* seg_off;         // [E+1] out (local only): padded segment offsets
};
cudaError_t route_scan(const RouteScanArgs& a, cudaStream_t s);

// slot/keep -> send/home positions; copies kept rows of `a` into `xsend`.
cudaError_t dispatch_rows(const bf16* a, int64_t n, int h, int E, int T, int my_chunk,
                          int64_t cap, const int* expert, const int* blk_prefix,
                          const int* chunk_prefix, const int* send_base, const int* home_base,
                          int* slot, int* pos_send, int* pos_home, bf16* xsend, cudaStream_t s);
// zero rows [seg_off[g] + valid[g], seg_off[g+1]) of buf (valid == nullptr: use counts in
// valid_from_kc = kc row sums).
cudaError_t zero_pad_rows(bf16* buf, int64_t ld, int h, const int* seg_off, const int* valid,
                          int G, int max_pad_rows, cudaStream_t s);

// y[k] = prob[k] * fhome[pos_home[k]] (0 when dropped); per-block sum(y^2) partials.
cudaError_t combine_forward(const bf16* fhome, const int* pos_home, const float* prob,
                            int64_t n, int h, bf16* y, float* loss_part, cudaStream_t s);
cudaError_t loss_finalize(const float* loss_part, int nblk, double inv_2n, double* loss,
                          cudaStream_t s);
// dfe[pos_send[k]] = prob[k] * dy[k];  dchosen[k] = <fhome[pos_home[k]], dy[k]>;
// dlogits[k][j] = dchosen * p_e * (delta_je - p_j).  dy == nullptr: dy = y * dy_scale.
cudaError_t combine_backward(const bf16* fhome, const int* pos_home, const int* pos_send,
                             const float* prob, const float* probs, const int* expert,
                             int64_t n, int h, int E, const bf16* dy, const bf16* y,
                             float dy_scale, bf16* dfe, float* dlogits, cudaStream_t s);
// Where token k's expert-side row lives: locally (home layout, pos_home) or, for the
// peer-memory exchange, in the assembled buffer of replica my_t of expert e's EP rank:
// peers[my_t + Tp * (e / Eloc)] + (pull_base[c][e] + pos_home[k] - home_base[c][e]) rows.
struct RowSrc {
  const bf16* local = nullptr;  // home-layout rows (local mode)
  const int* pos_home = nullptr;
  const unsigned long long* peers = nullptr;  // device table of peer buffer bases
  const long long* pull_base = nullptr;       // [Tc][E]
  const int* home_base = nullptr;             // [Tc][E]
  const int* expert = nullptr;
  int64_t chunk_len = 0;
  int Tc = 1, E = 1, Eloc = 1, Tp = 1, my_t = 0;
  // 1: read replica my_t (already TP-reduced);  Tp: sum the row over every TP replica
  // (the row-parallel all-reduce of parallel_linear.cpp:28 folded into the consumer)
  int nsum = 1;
  // local mode with nsum > 1: the T partial rows were pushed into this rank's receive
  // buffer by the experts' GEMM epilogues, slot t at local + t * slot_stride
  int64_t slot_stride = 0;
};
// da[k] = row(k) + sum_j dlogits[k][j] Wg[:, j]
cudaError_t gate_backward_input(const RowSrc& src, const float* dlogits, const bf16* wg,
                                int64_t n, int h, int E, bf16* da, cudaStream_t s);

// ---- peer-memory exchange (CUDA IPC pointers over NVLink) -------------------------
// Scatter every kept row of this rank's chunk straight into the assembled buffer of its
// expert's EP rank: replica my_t, or every TP replica (DTD: one source per row).
// Destination row = disp_base[e] + pos_send[k] - send_base[e].  Ends with a system fence.
struct PeerDst {
  const unsigned long long* peers = nullptr;  // plane rank -> buffer base
  const long long* disp_base = nullptr;       // [E]
  const int* send_base = nullptr;             // [E]
  int Eloc = 1, Tp = 1, my_t = 0, all_replicas = 0;
  // fault injection (corrupt_drop) on the peer exchange: this rank dispatches another
  // chunk than its slot; rows past the slot's reserved block (clamp_rows[e]) are not
  // written, so the wrong chunk lands misplaced like the reference's instead of overrunning
  const int* clamp_rows = nullptr;
  // all_replicas: 0 = every replica; 1 = replica my_t only (the reference's EP all-to-all);
  // 2 = the other replicas only (its DTD all-gather) -- the timed pass splits the fused
  // scatter into these two launches to report all-to-all and all-gather time separately
  int part = 0;
};
cudaError_t scatter_rows_peer(const bf16* a, const int* pos_send, const int* expert, int64_t n,
                              int h, const PeerDst& dst, const float* scale, bool scale_by_prob,
                              cudaStream_t s);
// y[k] = prob[k] * row(k), fhome[k] = row(k) (token order, for the backward), loss partials
// barrier of the EP x TP plane through IPC-mapped flag arrays (flags[r] = member r's array);
// a member missing for timeout_ns (0: no limit) sets *fault = 1 + its plane rank and the
// barrier returns (no trap); with *fault set every barrier returns at once
cudaError_t plane_barrier_peer(const unsigned long long* flags, int PS, int me,
                               unsigned* epoch_dev, int* fault, unsigned long long timeout_ns,
                               cudaStream_t s);
// home row (-1: pad) and source EP member of every assembled row, for the push return
cudaError_t push_map(const int* kc_all, int T, int P, int E, int Tc, int my_ep, const int* seg,
                     int* row_home, int* row_src, cudaStream_t s);
// CommLedger entries of one MoE pass (forward / recompute / backward) of this rank, from
// the device-resident routed counts: led[phase][op][calls, bytes] += ...
cudaError_t ledger_moe_pass(unsigned long long* led, int phase, int P, int T, int dtd, int Tc,
                            int E, int Eloc, int my_t, int my_ep, const int* kc, const int* kc_all,
                            int src_stride, const int* seg_valid, int h, cudaStream_t s);
// the peer-exchange plan on the device: seg = [seg_off Eloc+1][valid rows Eloc],
// disp_base [E], pull_base [Tc][E] from the plane-gathered counts
cudaError_t plan_peer(const int* kc_all, int T, int P, int E, int Tc, int my_ep, int my_c,
                      int* seg, long long* disp_base, long long* pull_base, cudaStream_t s);
cudaError_t combine_pull(const RowSrc& src, const float* prob, int64_t n, int h, bf16* y,
                         bf16* fhome, float* loss_part, cudaStream_t s);
// dchosen = <fhome[k], dy[k]> (token-order fhome), dlogits, and p*dy rows scattered to the
// experts' dFe buffers like scatter_rows_peer.
cudaError_t combine_backward_peer(const bf16* fhome, const int* pos_home, const int* pos_send,
                                  const float* prob, const float* probs, const int* expert,
                                  int64_t n, int h, int E, const bf16* dy, const bf16* y,
                                  float dy_scale, const PeerDst& dst, float* dlogits,
                                  cudaStream_t s);
// dWg = a^T dlogits (deterministic two-stage reduction), written as bf16 (+ fp32 copy).
cudaError_t gate_backward_weight(const bf16* a, const float* dlogits, int64_t n, int h, int E,
                                 float* part, bf16* dwg, cudaStream_t s);
size_t gate_dw_part_floats(int64_t n, int h, int E);
// db_g[j] = sum over rows of group g of D[row][j]  (D [rows][w] bf16)
// the second half of colsum_groups: sum the 32-row partials (written by a DGELU epilogue)
cudaError_t colsum_finish(const float* part, int w, const int* seg_off, int G, bf16* out,
                          int64_t out_stride, cudaStream_t s);
cudaError_t colsum_groups(const bf16* D, int64_t ld, int w, const int* seg_off, int G,
                          int max_rows_per_group, float* part, bf16* out, int64_t out_stride,
                          cudaStream_t s);
size_t colsum_part_floats(int w, int G, int max_rows_per_group);

// out[k] = src[pos[k]], zero when pos[k] < 0 (dispatch backward un-permute)
cudaError_t gather_rows(const bf16* src, const int* pos, int64_t n, int h, bf16* out,
                        cudaStream_t s);
// per-block expert histogram from an expert-id array (ted_route without the gate)
cudaError_t expert_hist(const int* expert, int64_t n, int E, int* blk_hist, cudaStream_t s);
cudaError_t keep_from_slot(const int* slot, int64_t n, int64_t cap, uint8_t* keep,
                           cudaStream_t s);
// DTD placement verdict (moe.cpp:537-556) from the dispatch's pos_send / pos_home:
// verdict[0] = this forward, verdict[1] &= (sticky).  slot_chunk < 0: no DTD.
cudaError_t placement_verdict(const int* pos_send, const int* pos_home, int64_t n, int T,
                              int slot_chunk, int* verdict, cudaStream_t s);
cudaError_t dlogits_from_dchosen(const float* probs, const int* expert, const float* dchosen,
                                 int64_t n, int E, float* dlogits, cudaStream_t s);

// AdamW (optimizer.cpp:58-104) over [begin, end) of a flat family.
cudaError_t adam_step(float* master, float* m1, float* m2, bf16* param, const bf16* grad,
                      int64_t begin, int64_t end, int64_t tile, float lr, float b1, float b2,
                      float omb1, float omb2, float eps, float wd, float inv_c1, float inv_c2,
                      const float* coef, cudaStream_t s);
// device-side step counter += 1 and coef = {1/(1-b1^step), 1/(1-b2^step)} (graph-safe);
// a non-null coef passed to the Adam launchers overrides inv_c1 / inv_c2.
cudaError_t adam_prep(long long* step, float* coef, double b1, double b2, cudaStream_t s);

// AdamW over nseg equal, equally strided segments of an unsharded family.  blk_cols > 0:
// each segment is a (seg_len / blk_cols) x blk_cols matrix whose optimizer state uses the
// blk_off layout (parameters and gradients row-major).
cudaError_t adam_segments(float* master, float* m1, float* m2, bf16* param, const bf16* grad,
                          int nseg, int64_t seg_stride, int64_t seg_off, int64_t seg_len, float lr,
                          float b1, float b2, float omb1, float omb2, float eps, float wd,
                          float inv_c1, float inv_c2, const float* coef, int grid,
                          cudaStream_t s, int blk_cols = 0);

}  // namespace ted
