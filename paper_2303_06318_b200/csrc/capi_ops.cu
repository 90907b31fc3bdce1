// capi_ops.cu -- extern "C" operator entry points of include/ted.h (everything except
// the ted_layer_* object, which lives in layer.cu).  Plain pointers, status codes, no
// exceptions across the boundary, no CPU fallback.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../../include/ted.h"
#include "ted_internal.h"

using namespace ted;

namespace {

struct CfgErr : std::runtime_error {
  using std::runtime_error::runtime_error;
};

template <class F>
int guard(F&& f) {
  try {
    f();
    return TED_OK;
  } catch (const CfgErr& e) {
    set_error(e.what());
    return TED_ERR_CONFIG;
  } catch (const std::exception& e) {
    set_error(e.what());
    return TED_ERR_RUNTIME;
  }
}

void need(bool ok, const std::string& m) {
  if (!ok) throw CfgErr(m);
}
void cuda_ok(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}
void device_ok() {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
    throw std::runtime_error("no CUDA device: the TED kernels are sm_100a-only (no CPU fallback)");
}
cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Operator workspace: one grow-only device arena per (device, stream), carved per call.
// Calls on one stream are ordered, so they can share it; a call that needs more than the
// arena holds re-allocates it once (stream-ordered), after which the hot call allocates
// nothing.  ted_ops_reserve() sizes it up front (e.g. before capturing a CUDA graph).
struct Arena {
  char* p = nullptr;
  size_t bytes = 0;
};
std::mutex g_arena_mu;
std::map<std::pair<int, cudaStream_t>, Arena> g_arenas;

char* arena(cudaStream_t s, size_t bytes) {
  int dev = 0;
  cuda_ok(cudaGetDevice(&dev), "cudaGetDevice");
  std::lock_guard<std::mutex> lk(g_arena_mu);
  Arena& a = g_arenas[{dev, s}];
  if (a.bytes < bytes) {
    if (a.p) cuda_ok(cudaFreeAsync(a.p, s), "workspace free");
    a.p = nullptr;
    a.bytes = 0;
    const size_t grow = std::max(bytes, size_t(1) << 20);
    cuda_ok(cudaMallocAsync(reinterpret_cast<void**>(&a.p), grow, s), "workspace alloc");
    a.bytes = grow;
  }
  return a.p;
}

// carves typed, 256 B aligned sub-buffers out of one arena request
struct Carve {
  std::vector<std::pair<void**, size_t>> parts;
  template <class T>
  Carve& add(T** dst, size_t count) {
    parts.emplace_back(reinterpret_cast<void**>(dst), (count * sizeof(T) + 255) & ~size_t(255));
    return *this;
  }
  void take(cudaStream_t s) {
    size_t total = 0;
    for (auto& p : parts) total += p.second;
    char* base = arena(s, total);
    for (auto& p : parts) {
      *p.first = base;
      base += p.second;
    }
  }
};

int64_t pad128(int64_t x) { return (x + 127) / 128 * 128; }

}  // namespace

extern "C" {

void ted_default_configs(ted_model_cfg* m, ted_topo_cfg* t, ted_flags* f, ted_adam_cfg* a,
                         ted_tile_cfg* tiles) {
  if (m) *m = ted_model_cfg{1, 8, 2, 8, 1};                 // moe.hpp:24-30
  if (t) *t = ted_topo_cfg{1, 1, 1, 1, 1};                  // topology.hpp:22-28
  if (f) *f = ted_flags{0, 0, 0, 0, 0};                     // moe.hpp:40-46 (ckpt off here)
  if (a) *a = ted_adam_cfg{1e-4, 0.9, 0.999, 1e-8, 0.01};   // optimizer.hpp:17-23
  if (tiles) *tiles = ted_tile_cfg{1, 1800000};             // optimizer.hpp:36-39
}

const char* ted_last_error(void) { return last_error(); }
const char* ted_version(void) { return "ted-b200 0.1 (sm_100a)"; }

int ted_set_device(int dev) {
  return guard([&] { cuda_ok(cudaSetDevice(dev), "cudaSetDevice"); });
}

int ted_derive_config(int world, int tp, int ep, ted_topo_cfg* out) {
  return guard([&] {
    need(world >= 1, "world_size must be >= 1, got " + std::to_string(world));
    need(tp >= 1, "tensor_parallel must be >= 1, got " + std::to_string(tp));
    need(ep >= 1, "experts must be >= 1, got " + std::to_string(ep));
    need(world % tp == 0, "tensor_parallel (" + std::to_string(tp) +
                              ") does not divide world_size (" + std::to_string(world) + ")");
    const int nonexp = world / tp;
    need(nonexp % ep == 0, "experts (" + std::to_string(ep) +
                               ") does not divide world_size / tensor_parallel (" +
                               std::to_string(nonexp) + ")");
    *out = ted_topo_cfg{world, tp, ep, nonexp / ep, nonexp};
  });
}

int ted_shard_range(int64_t total, int parts, int index, int64_t* begin, int64_t* end) {
  return guard([&] {
    need(parts >= 1, "shard_range: parts must be >= 1, got " + std::to_string(parts));
    need(index >= 0 && index < parts, "shard_range: index " + std::to_string(index) +
                                          " outside [0, " + std::to_string(parts) + ")");
    need(total >= 0, "shard_range: negative element count");
    const int64_t base = total / parts, extra = total % parts;
    *begin = index * base + (index < extra ? index : extra);
    *end = *begin + base + (index < extra ? 1 : 0);
  });
}

int ted_gate_forward(const uint16_t* a, const uint16_t* wg, int64_t n, int h, int E,
                     float* logits, float* probs, int32_t* expert, float* prob, void* stream) {
  return guard([&] {
    need(E >= 1 && E <= 64, "gate: experts must be in [1, 64]");
    need(h % 256 == 0, "gate: hidden must be a multiple of 256");
    need(n >= 0, "gate: negative token count");
    device_ok();
    const int nblk = int((n + kRouteBlock - 1) / kRouteBlock);
    int* hist = nullptr;
    bf16* wgT = nullptr;
    Carve()
        .add(&hist, size_t(nblk) * E)
        .add(&wgT, std::max<size_t>(gate_wgt_elems(h, E), 1))
        .take(S(stream));
    cuda_ok(gate_forward(reinterpret_cast<const bf16*>(a), reinterpret_cast<const bf16*>(wg), n,
                         h, E, logits, probs, expert, prob, hist, wgT, S(stream)),
            "gate_forward");
  });
}

int ted_gate_route_logits(const float* logits, int64_t n, int E, float* probs, int32_t* expert,
                          float* prob, void* stream) {
  return guard([&] {
    need(E >= 1 && E <= 64, "gate: experts must be in [1, 64]");
    device_ok();
    const int nblk = int((n + kRouteBlock - 1) / kRouteBlock);
    int* hist = nullptr;
    Carve().add(&hist, size_t(nblk) * E).take(S(stream));
    cuda_ok(gate_route_logits(logits, n, E, probs, expert, prob, hist, S(stream)),
            "gate_route_logits");
  });
}

int ted_route(const int32_t* expert, int64_t n, int E, int64_t capacity, int T, int32_t* slot,
              uint8_t* keep, int32_t* kept_counts, void* stream) {
  return guard([&] {
    need(E >= 1 && E <= 64, "route: experts must be in [1, 64]");
    need(T >= 1 && T <= 8, "route: chunks must be in [1, 8]");
    need(T == 1 || n % T == 0, "route: chunks must divide the token count");
    device_ok();
    const int64_t cap = capacity <= 0 ? n : capacity;
    cudaStream_t s = S(stream);
    const int nblk = int((n + kRouteBlock - 1) / kRouteBlock);
    int *hist, *pre, *cp, *kc, *sb, *hb, *so, *ps, *ph;
    Carve()
        .add(&hist, size_t(nblk) * E)
        .add(&pre, size_t(nblk) * E)
        .add(&cp, size_t(T + 1) * E)
        .add(&kc, size_t(T) * E)
        .add(&sb, size_t(E))
        .add(&hb, size_t(T) * E)
        .add(&so, size_t(E + 1))
        .add(&ps, size_t(n))
        .add(&ph, size_t(n))
        .take(s);
    cuda_ok(expert_hist(expert, n, E, hist, s), "expert_hist");
    RouteScanArgs ra{};
    ra.n = n;
    ra.E = E;
    ra.T = T;
    ra.my_chunk = -1;
    ra.cap = cap;
    ra.local = 0;
    ra.expert = expert;
    ra.blk_hist = hist;
    ra.blk_prefix = pre;
    ra.chunk_prefix = cp;
    ra.kc = kc;
    ra.send_base = sb;
    ra.home_base = hb;
    ra.seg_off = so;
    cuda_ok(route_scan(ra, s), "route_scan");
    cuda_ok(dispatch_rows(nullptr, n, 0, E, T, -1, cap, expert, pre, cp, sb, hb, slot, ps, ph,
                          nullptr, s),
            "dispatch_rows");
    if (keep) cuda_ok(keep_from_slot(slot, n, cap, keep, s), "keep");
    if (kept_counts)
      cuda_ok(cudaMemcpyAsync(kept_counts, kc, sizeof(int) * T * E, cudaMemcpyDeviceToDevice, s),
              "memcpy");
  });
}

int ted_gate_backward(const uint16_t* a, const uint16_t* wg, const float* probs,
                      const int32_t* expert, const float* dchosen, int64_t n, int h, int E,
                      uint16_t* dwg, uint16_t* dinput, void* stream) {
  return guard([&] {
    need(E >= 1 && E <= 64, "gate: experts must be in [1, 64]");
    need(h % 256 == 0, "gate: hidden must be a multiple of 256");
    device_ok();
    cudaStream_t s = S(stream);
    float *dl, *part;
    Carve().add(&dl, size_t(n) * E).add(&part, gate_dw_part_floats(n, h, E)).take(s);
    cuda_ok(dlogits_from_dchosen(probs, expert, dchosen, n, E, dl, s), "dlogits");
    if (dwg)
      cuda_ok(gate_backward_weight(reinterpret_cast<const bf16*>(a), dl, n, h, E, part,
                                   reinterpret_cast<bf16*>(dwg), s),
              "gate_backward_weight");
    if (dinput)
      cuda_ok(gate_backward_input(RowSrc{}, dl, reinterpret_cast<const bf16*>(wg), n, h, E,
                                  reinterpret_cast<bf16*>(dinput), s),
              "gate_backward_input");
  });
}

int ted_grouped_gemm(int mode, int epilogue, int groups, int M, int N, int K,
                     const int32_t* seg_off, int max_rows, const uint16_t* A, int64_t lda,
                     int a_mn, const uint16_t* B, int64_t ldb, int64_t b_group_stride, int b_mn,
                     uint16_t* C, int64_t ldc, int64_t c_group_stride, const uint16_t* bias,
                     int64_t bias_group_stride, uint16_t* aux, int64_t ld_aux, void* stream) {
  return guard([&] {
    device_ok();
    GemmOperands o{};
    o.A = reinterpret_cast<const bf16*>(A);
    o.lda = lda;
    o.a_mn = a_mn != 0;
    o.B = reinterpret_cast<const bf16*>(B);
    o.ldb = ldb;
    o.b_group_stride = b_group_stride;
    o.b_mn = b_mn != 0;
    GemmParams p{};
    p.mode = mode;
    p.epi = epilogue;
    p.groups = groups;
    p.M = M;
    p.N = N;
    p.K = K;
    p.seg_off = seg_off;
    p.C = reinterpret_cast<bf16*>(C);
    p.ldc = ldc;
    p.c_group_stride = c_group_stride;
    p.bias = reinterpret_cast<const bf16*>(bias);
    p.bias_group_stride = bias_group_stride;
    p.aux = reinterpret_cast<bf16*>(aux);
    p.ld_aux = ld_aux;
    const char* why = nullptr;
    cudaError_t e = grouped_gemm(o, p, max_rows, S(stream), &why);
    if (e != cudaSuccess) {
      if (why) throw CfgErr(why);
      cuda_ok(e, "grouped_gemm");
    }
  });
}

int ted_adam_step(float* master, float* m1, float* m2, uint16_t* param, const uint16_t* grad,
                  int64_t begin, int64_t end, int64_t step, const ted_adam_cfg* adam,
                  const ted_tile_cfg* tiles, uint64_t* upcast_peak, void* stream) {
  return guard([&] {
    need(adam != nullptr && tiles != nullptr, "adam: null config");
    need(end >= begin && begin >= 0, "adam: bad owned range");
    need(step >= 1, "adam: step counts from 1");
    need(!tiles->enabled || tiles->tile_size >= 1,
         "step_owned: tile_size must be >= 1, got " + std::to_string(tiles->tile_size));
    device_ok();
    const int64_t owned = end - begin;
    const int64_t one = owned > 1 ? owned : 1;
    const int64_t tile = tiles->enabled ? (tiles->tile_size < one ? tiles->tile_size : one) : one;
    if (upcast_peak) *upcast_peak = owned == 0 ? 0 : uint64_t(tile) * 4u;
    const double c1 = 1.0 - std::pow(adam->beta1, double(step));
    const double c2 = 1.0 - std::pow(adam->beta2, double(step));
    cuda_ok(adam_step(master, m1, m2, reinterpret_cast<bf16*>(param),
                      reinterpret_cast<const bf16*>(grad), begin, end, tile, float(adam->lr),
                      float(adam->beta1), float(adam->beta2), float(1.0 - adam->beta1),
                      float(1.0 - adam->beta2), float(adam->eps),
                      float(adam->weight_decay), float(1.0 / c1), float(1.0 / c2), nullptr,
                      S(stream)),
            "adam_step");
  });
}

int ted_placement_verdict(const int32_t* pos_send, const int32_t* pos_home, int64_t n, int T,
                          int slot_chunk, int32_t* verdict, void* stream) {
  return guard([&] {
    need(n >= 0 && T >= 1, "placement_verdict: bad sizes");
    need(slot_chunk < T, "placement_verdict: slot chunk outside [0, T)");
    device_ok();
    cuda_ok(placement_verdict(pos_send, pos_home, n, T, slot_chunk, verdict, S(stream)),
            "placement_verdict");
  });
}


// ------------------------------------------------------------ operator workspace
int ted_ops_reserve(size_t bytes, void* stream) {
  return guard([&] {
    device_ok();
    arena(S(stream), bytes);
  });
}

int ted_ops_release(void) {
  return guard([&] {
    std::lock_guard<std::mutex> lk(g_arena_mu);
    for (auto& kv : g_arenas)
      if (kv.second.p) cudaFreeAsync(kv.second.p, kv.first.second);
    g_arenas.clear();
  });
}

// ------------------------------------------------------------ single-rank MoE operators
int64_t ted_dispatch_rows_bound(int64_t n, int E, int64_t capacity) {
  if (n < 0 || E < 1) return 0;
  const int64_t kept = capacity > 0 ? std::min<int64_t>(n, int64_t(E) * capacity) : n;
  return pad128(kept + int64_t(E) * (kPad - 1));
}

int ted_dispatch_forward(const uint16_t* a, const int32_t* expert, int64_t n, int h, int E,
                         int64_t capacity, int32_t* slot, int32_t* pos, uint16_t* x_asm,
                         int32_t* seg_off, int32_t* kept_counts, void* stream) {
  return guard([&] {
    need(E >= 1 && E <= 64, "dispatch: experts must be in [1, 64]");
    need(h >= 8 && h % 8 == 0, "dispatch: hidden must be a positive multiple of 8");
    need(n >= 0, "dispatch: negative token count");
    need(x_asm && seg_off && kept_counts && (n == 0 || (expert && pos)), "dispatch: null argument");
    device_ok();
    cudaStream_t s = S(stream);
    const int64_t cap = capacity <= 0 ? std::max<int64_t>(n, 1) : capacity;
    const int nblk = int((n + kRouteBlock - 1) / kRouteBlock);
    int *hist, *pre, *cp, *sb, *hb, *ps, *sl;
    Carve()
        .add(&hist, size_t(std::max(nblk, 1)) * E)
        .add(&pre, size_t(std::max(nblk, 1)) * E)
        .add(&cp, size_t(2) * E)
        .add(&sb, size_t(E))
        .add(&hb, size_t(E))
        .add(&ps, size_t(std::max<int64_t>(n, 1)))
        .add(&sl, size_t(std::max<int64_t>(n, 1)))
        .take(s);
    cuda_ok(expert_hist(expert, n, E, hist, s), "expert_hist");
    RouteScanArgs ra{};
    ra.n = n;
    ra.E = E;
    ra.T = 1;
    ra.my_chunk = -1;
    ra.cap = cap;
    ra.local = 1;  // single rank: send == home == the padded expert segments
    ra.expert = expert;
    ra.blk_hist = hist;
    ra.blk_prefix = pre;
    ra.chunk_prefix = cp;
    ra.kc = kept_counts;
    ra.send_base = sb;
    ra.home_base = hb;
    ra.seg_off = seg_off;
    cuda_ok(route_scan(ra, s), "route_scan");
    cuda_ok(dispatch_rows(reinterpret_cast<const bf16*>(a), n, h, E, 1, -1, cap, expert, pre, cp,
                          sb, hb, slot ? slot : sl, ps, pos, reinterpret_cast<bf16*>(x_asm), s),
            "dispatch_rows");
    // pad rows of every segment zeroed (the wgrad reductions run over them)
    cuda_ok(zero_pad_rows(reinterpret_cast<bf16*>(x_asm), h, h, seg_off, kept_counts, E, kPad, s),
            "zero_pad_rows");
  });
}

int ted_dispatch_backward(const uint16_t* dx_asm, const int32_t* pos, int64_t n, int h,
                          uint16_t* da, void* stream) {
  return guard([&] {
    need(h >= 8 && h % 8 == 0, "dispatch backward: hidden must be a positive multiple of 8");
    need(n >= 0, "dispatch backward: negative token count");
    device_ok();
    cuda_ok(gather_rows(reinterpret_cast<const bf16*>(dx_asm), pos, n, h,
                        reinterpret_cast<bf16*>(da), S(stream)),
            "gather_rows");
  });
}

int ted_combine_forward(const uint16_t* f_asm, const int32_t* pos, const float* prob, int64_t n,
                        int h, uint16_t* y, void* stream) {
  return guard([&] {
    need(h >= 8 && h % 8 == 0, "combine: hidden must be a positive multiple of 8");
    need(n >= 0, "combine: negative token count");
    device_ok();
    const int nblk = int((n + kRouteBlock - 1) / kRouteBlock);
    float* part = nullptr;
    Carve().add(&part, size_t(std::max(nblk, 1)) + 1).take(S(stream));
    cuda_ok(combine_forward(reinterpret_cast<const bf16*>(f_asm), pos, prob, n, h,
                            reinterpret_cast<bf16*>(y), part, S(stream)),
            "combine_forward");
  });
}

int ted_combine_backward(const uint16_t* f_asm, const int32_t* pos, const float* prob,
                         const float* probs, const int32_t* expert, const uint16_t* dy, int64_t n,
                         int h, int E, const int32_t* seg_off, const int32_t* kept_counts,
                         uint16_t* df_asm, float* dlogits, void* stream) {
  return guard([&] {
    need(E >= 1 && E <= 64, "combine backward: experts must be in [1, 64]");
    need(h >= 8 && h % 8 == 0, "combine backward: hidden must be a positive multiple of 8");
    need(dy && dlogits && df_asm, "combine backward: null argument");
    device_ok();
    cudaStream_t s = S(stream);
    cuda_ok(combine_backward(reinterpret_cast<const bf16*>(f_asm), pos, pos, prob, probs, expert, n,
                             h, E, reinterpret_cast<const bf16*>(dy), nullptr, 1.f,
                             reinterpret_cast<bf16*>(df_asm), dlogits, s),
            "combine_backward");
    if (seg_off && kept_counts)
      cuda_ok(zero_pad_rows(reinterpret_cast<bf16*>(df_asm), h, h, seg_off, kept_counts, E, kPad, s),
              "zero_pad_rows");
  });
}

int ted_gate_backward_dlogits(const uint16_t* a, const uint16_t* wg, const float* dlogits,
                              int64_t n, int h, int E, uint16_t* dwg, uint16_t* dinput,
                              const uint16_t* dispatch_grad, const int32_t* pos, void* stream) {
  return guard([&] {
    need(E >= 1 && E <= 64, "gate: experts must be in [1, 64]");
    need(h % 256 == 0, "gate: hidden must be a multiple of 256");
    device_ok();
    cudaStream_t s = S(stream);
    if (dwg) {
      float* part = nullptr;
      Carve().add(&part, gate_dw_part_floats(n, h, E)).take(s);
      cuda_ok(gate_backward_weight(reinterpret_cast<const bf16*>(a), dlogits, n, h, E, part,
                                   reinterpret_cast<bf16*>(dwg), s),
              "gate_backward_weight");
    }
    if (dinput) {
      RowSrc src{};
      if (dispatch_grad && pos) {  // da = dX[pos] + dlogits Wg^T  (moe.cpp:685)
        src.local = reinterpret_cast<const bf16*>(dispatch_grad);
        src.pos_home = pos;
      }
      cuda_ok(gate_backward_input(src, dlogits, reinterpret_cast<const bf16*>(wg), n, h, E,
                                  reinterpret_cast<bf16*>(dinput), s),
              "gate_backward_input");
    }
  });
}

namespace {
void ffn_shapes_ok(int E, int h, int f, int64_t rows) {
  need(E >= 1 && E <= 128, "expert ffn: experts (groups) must be in [1, 128]");
  need(h % 256 == 0, "expert ffn: hidden must be a multiple of 256 (tensor-core N tile)");
  need(f % 256 == 0, "expert ffn: inner width must be a multiple of 256");
  need(rows >= 128 && rows % 128 == 0 && rows <= INT32_MAX,
       "expert ffn: rows (the assembled-buffer bound) must be a positive multiple of 128");
}
}  // namespace

int ted_expert_ffn_forward(const uint16_t* x_asm, const int32_t* seg_off, int64_t rows, int E,
                           int h, int f, const uint16_t* w1, int64_t w1_stride,
                           const uint16_t* b1, int64_t b1_stride, const uint16_t* w2,
                           int64_t w2_stride, const uint16_t* b2, int64_t b2_stride, uint16_t* z,
                           uint16_t* hact, uint16_t* f_asm, void* stream) {
  return guard([&] {
    ffn_shapes_ok(E, h, f, rows);
    need(x_asm && seg_off && w1 && w2 && z && hact && f_asm, "expert ffn: null argument");
    device_ok();
    cudaStream_t s = S(stream);
    auto bf = [](const uint16_t* p) { return reinterpret_cast<const bf16*>(p); };
    // Z = X W1 + b1, H = gelu(Z)  (column_parallel_forward + gelu_forward)
    GemmOperands o{bf(x_asm), h, false, bf(w1), f, w1_stride, true};
    GemmParams g{};
    g.mode = GEMM_ROWS;
    g.epi = EPI_BIAS_GELU;
    g.groups = E;
    g.N = f;
    g.K = h;
    g.seg_off = seg_off;
    g.C = reinterpret_cast<bf16*>(z);
    g.ldc = f;
    g.bias = bf(b1);
    g.bias_group_stride = b1_stride;
    g.aux = reinterpret_cast<bf16*>(hact);
    g.ld_aux = f;
    const char* why = nullptr;
    if (grouped_gemm(o, g, int(rows), s, &why) != cudaSuccess)
      throw std::runtime_error(std::string("expert ffn gemm1: ") + (why ? why : "launch failed"));
    // F = H W2 + b2  (row_parallel_forward on one rank)
    o = GemmOperands{bf(hact), f, false, bf(w2), h, w2_stride, true};
    g.epi = EPI_BIAS;
    g.N = h;
    g.K = f;
    g.C = reinterpret_cast<bf16*>(f_asm);
    g.ldc = h;
    g.bias = bf(b2);
    g.bias_group_stride = b2_stride;
    g.aux = nullptr;
    if (grouped_gemm(o, g, int(rows), s, &why) != cudaSuccess)
      throw std::runtime_error(std::string("expert ffn gemm2: ") + (why ? why : "launch failed"));
  });
}

int ted_expert_ffn_backward(const uint16_t* x_asm, uint16_t* z, const uint16_t* hact,
                            const uint16_t* df_asm, const int32_t* seg_off, int64_t rows, int E,
                            int h, int f, const uint16_t* w1, int64_t w1_stride,
                            const uint16_t* w2, int64_t w2_stride, uint16_t* dx_asm,
                            uint16_t* dw1, int64_t dw1_stride, uint16_t* db1, int64_t db1_stride,
                            uint16_t* dw2, int64_t dw2_stride, uint16_t* db2, int64_t db2_stride,
                            void* stream) {
  return guard([&] {
    ffn_shapes_ok(E, h, f, rows);
    need(x_asm && z && hact && df_asm && seg_off && w1 && w2 && dx_asm && dw1 && db1 && dw2 && db2,
         "expert ffn backward: null argument");
    device_ok();
    cudaStream_t s = S(stream);
    auto bf = [](const uint16_t* p) { return reinterpret_cast<const bf16*>(p); };
    auto mb = [](uint16_t* p) { return reinterpret_cast<bf16*>(p); };
    float* part = nullptr;
    Carve()
        .add(&part, std::max(colsum_part_floats(f, E, int(rows)), colsum_part_floats(h, E, int(rows))))
        .take(s);
    const char* why = nullptr;
    auto run = [&](const GemmOperands& o, const GemmParams& g, const char* what) {
      if (grouped_gemm(o, g, int(rows), s, &why) != cudaSuccess)
        throw std::runtime_error(std::string(what) + ": " + (why ? why : "launch failed"));
    };
    // dZ = (dF W2^T) * gelu'(Z), in place over Z, with the db1 column-sum partials
    GemmParams g{};
    g.mode = GEMM_ROWS;
    g.epi = EPI_DGELU;
    g.groups = E;
    g.seg_off = seg_off;
    g.N = f;
    g.K = h;
    g.C = mb(z);
    g.ldc = f;
    g.aux = mb(z);
    g.ld_aux = f;
    g.colsum_part = part;
    run(GemmOperands{bf(df_asm), h, false, bf(w2), h, w2_stride, false}, g, "dgrad2");
    cuda_ok(colsum_finish(part, f, seg_off, E, mb(db1), db1_stride, s), "db1");
    // dW2 = H^T dF, db2 = colsum(dF)
    g = GemmParams{};
    g.mode = GEMM_KDIM;
    g.epi = EPI_STORE;
    g.groups = E;
    g.seg_off = seg_off;
    g.M = f;
    g.N = h;
    g.C = mb(dw2);
    g.ldc = h;
    g.c_group_stride = dw2_stride;
    run(GemmOperands{bf(hact), f, true, bf(df_asm), h, 0, true}, g, "wgrad2");
    cuda_ok(colsum_groups(bf(df_asm), h, h, seg_off, E, int(rows), part, mb(db2), db2_stride, s),
            "db2");
    // dX = dZ W1^T
    g = GemmParams{};
    g.mode = GEMM_ROWS;
    g.epi = EPI_STORE;
    g.groups = E;
    g.seg_off = seg_off;
    g.N = h;
    g.K = f;
    g.C = mb(dx_asm);
    g.ldc = h;
    run(GemmOperands{bf(z), f, false, bf(w1), f, w1_stride, false}, g, "dgrad1");
    // dW1 = X^T dZ
    g = GemmParams{};
    g.mode = GEMM_KDIM;
    g.epi = EPI_STORE;
    g.groups = E;
    g.seg_off = seg_off;
    g.M = h;
    g.N = f;
    g.C = mb(dw1);
    g.ldc = f;
    g.c_group_stride = dw1_stride;
    run(GemmOperands{bf(x_asm), h, true, bf(z), f, 0, true}, g, "wgrad1");
  });
}

}  // extern "C"
