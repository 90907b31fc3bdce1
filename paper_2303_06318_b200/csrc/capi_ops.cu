// capi_ops.cu -- extern "C" operator entry points of include/ted.h (everything except
// the ted_layer_* object, which lives in layer.cu).  Plain pointers, status codes, no
// exceptions across the boundary, no CPU fallback.
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <stdexcept>
#include <string>

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

template <class T>
struct Scratch {  // stream-ordered temporary
  T* p = nullptr;
  cudaStream_t s;
  Scratch(size_t n, cudaStream_t st) : s(st) {
    if (n) cuda_ok(cudaMallocAsync(reinterpret_cast<void**>(&p), n * sizeof(T), s), "malloc");
  }
  ~Scratch() {
    if (p) cudaFreeAsync(p, s);
  }
};

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
    Scratch<int> hist(size_t(nblk) * E, S(stream));
    cuda_ok(gate_forward(reinterpret_cast<const bf16*>(a), reinterpret_cast<const bf16*>(wg), n,
                         h, E, logits, probs, expert, prob, hist.p, S(stream)),
            "gate_forward");
  });
}

int ted_gate_route_logits(const float* logits, int64_t n, int E, float* probs, int32_t* expert,
                          float* prob, void* stream) {
  return guard([&] {
    need(E >= 1 && E <= 64, "gate: experts must be in [1, 64]");
    device_ok();
    const int nblk = int((n + kRouteBlock - 1) / kRouteBlock);
    Scratch<int> hist(size_t(nblk) * E, S(stream));
    cuda_ok(gate_route_logits(logits, n, E, probs, expert, prob, hist.p, S(stream)),
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
    Scratch<int> hist(size_t(nblk) * E, s), pre(size_t(nblk) * E, s), cp(size_t(T + 1) * E, s),
        kc(size_t(T) * E, s), sb(size_t(E), s), hb(size_t(T) * E, s), so(size_t(E + 1), s),
        ps(size_t(n), s), ph(size_t(n), s);
    cuda_ok(expert_hist(expert, n, E, hist.p, s), "expert_hist");
    RouteScanArgs ra{};
    ra.n = n;
    ra.E = E;
    ra.T = T;
    ra.my_chunk = -1;
    ra.cap = cap;
    ra.local = 0;
    ra.expert = expert;
    ra.blk_hist = hist.p;
    ra.blk_prefix = pre.p;
    ra.chunk_prefix = cp.p;
    ra.kc = kc.p;
    ra.send_base = sb.p;
    ra.home_base = hb.p;
    ra.seg_off = so.p;
    cuda_ok(route_scan(ra, s), "route_scan");
    cuda_ok(dispatch_rows(nullptr, n, 0, E, T, -1, cap, expert, pre.p, cp.p, sb.p, hb.p, slot,
                          ps.p, ph.p, nullptr, s),
            "dispatch_rows");
    if (keep) cuda_ok(keep_from_slot(slot, n, cap, keep, s), "keep");
    if (kept_counts)
      cuda_ok(cudaMemcpyAsync(kept_counts, kc.p, sizeof(int) * T * E, cudaMemcpyDeviceToDevice, s),
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
    Scratch<float> dl(size_t(n) * E, s), part(gate_dw_part_floats(n, h, E), s);
    cuda_ok(dlogits_from_dchosen(probs, expert, dchosen, n, E, dl.p, s), "dlogits");
    if (dwg)
      cuda_ok(gate_backward_weight(reinterpret_cast<const bf16*>(a), dl.p, n, h, E, part.p,
                                   reinterpret_cast<bf16*>(dwg), s),
              "gate_backward_weight");
    if (dinput)
      cuda_ok(gate_backward_input(RowSrc{}, dl.p, reinterpret_cast<const bf16*>(wg), n, h, E,
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

}  // extern "C"
