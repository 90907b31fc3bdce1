// ted_host.h -- host-side infrastructure shared by the layer (layer.cu) and the model
// stack (model.cu): error types and the C-ABI status mapping (types.hpp:48-70), CUDA/NCCL
// checks, device buffers, ZeRO-1 shard bounds (optimizer.cpp:12-28).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>

#include "../../include/ted.h"
#include "ted_internal.h"

namespace ted {

struct ConfigError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct RuntimeError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

#define CU(x)                                                                              \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess)                                                                 \
      throw ::ted::RuntimeError(std::string("CUDA: ") + cudaGetErrorString(e_) + " at " + \
                                __FILE__ + ":" + std::to_string(__LINE__) + " (" #x ")");  \
  } while (0)
#define NC(x)                                                                                 \
  do {                                                                                        \
    ncclResult_t r_ = (x);                                                                    \
    if (r_ != ncclSuccess)                                                                    \
      throw ::ted::RuntimeError(std::string("NCCL: ") + ncclGetErrorString(r_) + " at " +    \
                                __FILE__ + ":" + std::to_string(__LINE__));                   \
  } while (0)

template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  bool owned = true;  // false: a view of another buffer (activation sharing under ckpt)
  void alloc(size_t count) {
    free();
    n = count;
    if (count) CU(cudaMalloc(&p, sizeof(T) * count));
  }
  void view(const DevBuf& other) {
    free();
    p = other.p;
    n = other.n;
    owned = false;
  }
  size_t bytes() const { return owned ? sizeof(T) * n : 0; }
  void zero() {
    if (n) CU(cudaMemset(p, 0, sizeof(T) * n));
  }
  void free() {
    if (p && owned) cudaFree(p);
    p = nullptr;
    n = 0;
    owned = true;
  }
  ~DevBuf() { free(); }
};

template <class T>
struct HostBuf {
  T* p = nullptr;
  void alloc(size_t count) {
    if (p) cudaFreeHost(p);
    p = nullptr;
    if (count) CU(cudaMallocHost(&p, sizeof(T) * count));
  }
  ~HostBuf() {
    if (p) cudaFreeHost(p);
  }
};

// a flat parameter family (flatten_family, moe.cpp:303-312): bf16 params and grads, fp32
// AdamW state over the ZeRO-1 owned range [begin, end)
struct Family {
  int64_t elems = 0;      // family length
  int group = 1, pos = 0;  // ZeRO-1 data group size / position
  int64_t begin = 0, end = 0;
  int64_t chunk = 0;  // completion all-gather chunk
  DevBuf<bf16> param, grad, gather;
  DevBuf<float> master, m1, m2;
  bool blocked = false;  // weight-matrix state in the blk_off layout (fused AdamW epilogue)
  DevBuf<long long> dstep;  // steps_done on the device (graph-safe)
  DevBuf<float> dcoef;      // {1/(1-b1^steps), 1/(1-b2^steps)}
  int64_t steps = 0;
  bool reset = false;
  uint64_t upcast_peak = 0;
  ncclComm_t dp = nullptr;
};

inline int64_t shard_lo(int64_t total, int parts, int i) {
  const int64_t base = total / parts, extra = total % parts;
  return i * base + (i < extra ? i : extra);
}

// exceptions -> status codes (0 ok, 2 config, 1 runtime); the message goes to ted_last_error
template <class F>
int guard(F&& f) {
  try {
    f();
    return TED_OK;
  } catch (const ConfigError& e) {
    set_error(e.what());
    return TED_ERR_CONFIG;
  } catch (const std::invalid_argument& e) {
    set_error(e.what());
    return TED_ERR_CONFIG;
  } catch (const std::exception& e) {
    set_error(e.what());
    return TED_ERR_RUNTIME;
  }
}

inline void require(bool ok, const std::string& msg) {
  if (!ok) throw ConfigError(msg);
}

inline void require_device() {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
    throw RuntimeError("no CUDA device: the TED kernels are sm_100a-only (no CPU fallback)");
  int dev = 0, major = 0;
  CU(cudaGetDevice(&dev));
  CU(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev));
  if (major != 10) throw RuntimeError("TED kernels need an sm_100 (B200) device");
}

inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

inline void check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw RuntimeError(std::string(what) + ": " + cudaGetErrorString(e));
}

inline uint16_t f2bf(float x) {
  uint32_t u;
  std::memcpy(&u, &x, 4);
  if ((u & 0x7fffffffu) > 0x7f800000u) return uint16_t((u >> 16) | 0x40);  // NaN
  u += 0x7fffu + ((u >> 16) & 1u);
  return uint16_t(u >> 16);
}
inline float bf2f(uint16_t b) {
  uint32_t u = uint32_t(b) << 16;
  float x;
  std::memcpy(&x, &u, 4);
  return x;
}

inline void run_gemm(const GemmOperands& o, const GemmParams& p, int64_t rows, cudaStream_t s) {
  const char* why = nullptr;
  cudaError_t e = grouped_gemm(o, p, int(rows), s, &why);
  if (e != cudaSuccess)
    throw RuntimeError(std::string("grouped_gemm: ") + (why ? why : cudaGetErrorString(e)));
}

// a MoE layer of a model stack whose communicators are split from the model's world
// communicator `parent` (layer.cu); the C-ABI twin is ted_layer_create
// `share` (optional): an earlier MoE layer of the same stack whose activation buffers this
// layer reuses (activation checkpointing: every layer recomputes its forward right
// before its backward, so one set of activations serves the whole stack)
int layer_create_child(const ted_model_cfg* model, const ted_topo_cfg* topo,
                       const ted_flags* flags, const ted_adam_cfg* adam,
                       const ted_tile_cfg* tiles, double capacity_factor, int shard_optimizer,
                       int rank, ncclComm_t parent, ted_layer* share, ted_layer** out);
// forward modes for activation checkpointing with communication-avoiding recompute (CAC,
// channel.cpp:20-51): LIVE runs everything; RECORD also stashes the exchange outputs
// (assembled expert rows and the combined home rows); REPLAY is the recompute that takes
// them from the stash instead of communicating and reruns only what the backward reads
enum { FWD_LIVE = 0, FWD_RECORD = 1, FWD_REPLAY = 2 };
void layer_set_forward_mode(ted_layer* L, int mode);
// backward when the optimizer step follows (Trainer::step): with an unsharded expert
// family the AdamW update runs inside the wgrad epilogues and the layer's next
// optimizer step skips that family
void layer_backward_then_step(ted_layer* L, const bf16* dy, bf16* da, cudaStream_t s);
// device bytes this layer owns (activations and workspaces, parameters and optimizer
// state, CAC stash)
void layer_memory(const ted_layer* L, int64_t* activations, int64_t* params, int64_t* stash);
// failure detection of a layer (plane-barrier timeout word, NCCL async errors, an earlier
// fault): throws RuntimeError("TimeoutError: ...") and aborts the layer's communicators
void layer_check_fault(ted_layer* L);
// ledger phase of the layer's next forwards (0 Forward, 1 Recompute)
void layer_set_ledger_phase(ted_layer* L, int phase);
void layer_abort(ted_layer* L, const std::string& why);

}  // namespace ted
