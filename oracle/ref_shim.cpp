// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY (oracle side; never linked into the product).
//
// A thin extern "C" face over the *unmodified* reference library (tedsim,
// /root/reference/proj/core/src/*.cpp, compiled by oracle/Makefile into
// oracle/_ref/libtedsim_ref.so).  It lets the Python test-suite and the
// bench.py reference arm call the reference's own public functions:
//
//   gate_forward / gate_backward            moe.cpp:158-208
//   linear_forward / linear_backward / gelu nn.cpp:78-121
//   OptimizerShard::create / step_owned      optimizer.cpp:30-104
//   SerialModel / Trainer                    moe.cpp:759-1121
//   predict_comm_volume                      cost_model.cpp:346-416
//   mix_seed / seeded_init                   tensor.cpp:100-129
//
// `ref_moe_sublayer` composes those public free functions into the MoE branch
// of SerialModel::forward_layer / backward_layer (moe.cpp:989-1015 and
// :1034-1064) on *injected* inputs, because SerialModel has no batch setter.
// Experts run on one std::thread each (the reference's own concurrency model:
// one rank-thread per expert, runner.hpp:18-39).
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "tedsim/cost_model.hpp"
#include "tedsim/moe.hpp"
#include "tedsim/nn.hpp"
#include "tedsim/optimizer.hpp"
#include "tedsim/tensor.hpp"
#include "tedsim/topology.hpp"

using namespace tedsim;

namespace {
thread_local std::string g_err;

Tensor mk(const double* p, std::int64_t r, std::int64_t c) {
  Tensor t = Tensor::zeros({r, c});
  if (p) std::memcpy(t.data.data(), p, sizeof(double) * r * c);
  return t;
}
Tensor mk1(const double* p, std::int64_t n) {
  Tensor t = Tensor::zeros({n});
  if (p) std::memcpy(t.data.data(), p, sizeof(double) * n);
  return t;
}
void put(const Tensor& t, double* out) {
  if (out) std::memcpy(out, t.data.data(), sizeof(double) * t.data.size());
}
template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const InvalidConfigError& e) {
    g_err = e.what();
    return 2;
  } catch (const InvalidGroupError& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

std::uint64_t ref_mix_seed(std::uint64_t seed, const char* tag) { return mix_seed(seed, tag); }

void ref_seeded_init(double* out, std::int64_t n, std::uint64_t seed, double scale) {
  Tensor t = seeded_init({n}, seed, scale);
  std::memcpy(out, t.data.data(), sizeof(double) * n);
}

int ref_gate_forward(const double* a, const double* w, int n, int h, int E, int* expert,
                     double* chosen, double* probs) {
  return guard([&] {
    GateResult g = gate_forward(mk(a, n, h), mk(w, h, E));
    for (int k = 0; k < n; ++k) {
      expert[k] = g.expert_of[k];
      chosen[k] = g.chosen_prob[k];
    }
    put(g.probs, probs);
  });
}

int ref_gate_backward(const double* a, const double* w, int n, int h, int E,
                      const double* dchosen, double* dweight, double* dinput) {
  return guard([&] {
    Tensor A = mk(a, n, h), W = mk(w, h, E);
    GateResult g = gate_forward(A, W);
    std::vector<double> dc(dchosen, dchosen + n);
    GateGrads gg = gate_backward(A, W, g, dc);
    put(gg.dweight, dweight);
    put(gg.dinput, dinput);
  });
}

double ref_gelu(double x) { return gelu_scalar(x); }
double ref_gelu_grad(double x) { return gelu_grad_scalar(x); }

// MoE branch on injected inputs (no capacity: the reference routes exactly).
// a [n,h]; wg [h,E]; w1 [E][h,f]; b1 [E][f]; w2 [E][f,h]; b2 [E][h]; dy [n,h] (may be null).
// Outputs: y [n,h]; da [n,h]; dwg [h,E]; dw1/db1/dw2/db2 like the weights.
int ref_moe_sublayer(int n, int h, int f, int E, const double* a, const double* wg,
                     const double* w1, const double* b1, const double* w2, const double* b2,
                     const double* dy, double* y, double* da, double* dwg, double* dw1,
                     double* db1, double* dw2, double* db2, int threads) {
  return guard([&] {
    const Tensor A = mk(a, n, h), Wg = mk(wg, h, E);
    GateResult gate = gate_forward(A, Wg);
    std::vector<std::vector<int>> rows(E);
    for (int k = 0; k < n; ++k) rows[gate.expert_of[k]].push_back(k);
    std::vector<Tensor> fe(E), dxe(E);
    auto run_expert = [&](int e) {
      const Tensor W1 = mk(w1 + (std::int64_t)e * h * f, h, f);
      const Tensor B1 = mk1(b1 + (std::int64_t)e * f, f);
      const Tensor W2 = mk(w2 + (std::int64_t)e * f * h, f, h);
      const Tensor B2 = mk1(b2 + (std::int64_t)e * h, h);
      Tensor xe = Tensor::zeros({(std::int64_t)rows[e].size(), h});
      for (std::size_t i = 0; i < rows[e].size(); ++i)
        std::memcpy(&xe.data[i * h], &A.data[(std::int64_t)rows[e][i] * h], sizeof(double) * h);
      const Tensor z1 = linear_forward(xe, W1, B1);
      const Tensor h1 = gelu_forward(z1);
      fe[e] = linear_forward(h1, W2, B2);
      if (!dy) return;
      Tensor dfe = Tensor::zeros({(std::int64_t)rows[e].size(), h});
      for (std::size_t i = 0; i < rows[e].size(); ++i) {
        const int k = rows[e][i];
        const double p = gate.chosen_prob[k];
        for (int j = 0; j < h; ++j) dfe.data[i * h + j] = p * dy[(std::int64_t)k * h + j];
      }
      LinearGrads rb = linear_backward(h1, W2, dfe);
      const Tensor dz1 = gelu_backward(z1, rb.dx);
      LinearGrads cb = linear_backward(xe, W1, dz1);
      if (dw1) std::memcpy(dw1 + (std::int64_t)e * h * f, cb.dw.data.data(), sizeof(double) * h * f);
      if (db1) std::memcpy(db1 + (std::int64_t)e * f, cb.db.data.data(), sizeof(double) * f);
      if (dw2) std::memcpy(dw2 + (std::int64_t)e * f * h, rb.dw.data.data(), sizeof(double) * f * h);
      if (db2) std::memcpy(db2 + (std::int64_t)e * h, rb.db.data.data(), sizeof(double) * h);
      dxe[e] = std::move(cb.dx);
    };
    if (threads > 1) {
      std::vector<std::thread> pool;
      for (int e = 0; e < E; ++e) pool.emplace_back(run_expert, e);
      for (auto& t : pool) t.join();
    } else {
      for (int e = 0; e < E; ++e) run_expert(e);
    }
    std::vector<double> dchosen(n, 0.0);
    std::vector<double> fhome((std::size_t)n * h, 0.0);
    for (int e = 0; e < E; ++e)
      for (std::size_t i = 0; i < rows[e].size(); ++i)
        std::memcpy(&fhome[(std::size_t)rows[e][i] * h], &fe[e].data[i * h], sizeof(double) * h);
    for (int k = 0; k < n; ++k) {
      const double p = gate.chosen_prob[k];
      double d = 0.0;
      for (int j = 0; j < h; ++j) {
        if (y) y[(std::int64_t)k * h + j] = p * fhome[(std::size_t)k * h + j];
        if (dy) d += fhome[(std::size_t)k * h + j] * dy[(std::int64_t)k * h + j];
      }
      dchosen[k] = d;
    }
    if (!dy) return;
    GateGrads gg = gate_backward(A, Wg, gate, dchosen);
    put(gg.dweight, dwg);
    if (da) {
      for (std::int64_t i = 0; i < (std::int64_t)n * h; ++i) da[i] = gg.dinput.data[i];
      for (int e = 0; e < E; ++e)
        for (std::size_t i = 0; i < rows[e].size(); ++i)
          for (int j = 0; j < h; ++j)
            da[(std::int64_t)rows[e][i] * h + j] += dxe[e].data[i * h + j];
    }
  });
}

// OptimizerShard over a family: `steps` steps with the given gradients
// (grads [steps][family]); writes the final out_full, master, m1, m2 (owned range).
int ref_adam(std::int64_t family, const double* values, int group_size, int position,
             double lr, double b1, double b2, double eps, double wd, int tiles_enabled,
             std::int64_t tile_size, int steps, const double* grads, double* out_full,
             double* master, double* m1, double* m2, std::uint64_t* upcast_peak) {
  return guard([&] {
    AdamConfig adam{lr, b1, b2, eps, wd};
    TileConfig tc;
    tc.enabled = tiles_enabled != 0;
    tc.tile_size = tile_size;
    std::vector<double> vals(values, values + family);
    OptimizerShard opt = OptimizerShard::create(vals, group_size, position, adam, tc);
    std::vector<double> out(family, 0.0);
    for (int s = 0; s < steps; ++s) {
      std::vector<double> g(grads + (std::int64_t)s * family, grads + (std::int64_t)(s + 1) * family);
      opt.step_owned(g, out);
    }
    std::memcpy(out_full, out.data(), sizeof(double) * family);
    if (master) std::memcpy(master, opt.master.data(), sizeof(double) * opt.master.size());
    if (m1) std::memcpy(m1, opt.m1.data(), sizeof(double) * opt.m1.size());
    if (m2) std::memcpy(m2, opt.m2.data(), sizeof(double) * opt.m2.size());
    if (upcast_peak) *upcast_peak = opt.upcast_peak_bytes;
  });
}

int ref_shard_range(std::int64_t total, int parts, int index, std::int64_t* begin,
                    std::int64_t* end) {
  return guard([&] {
    ShardRange r = shard_range(total, parts, index);
    *begin = r.begin;
    *end = r.end;
  });
}

int ref_derive_config(int world, int tp, int experts, int* out5) {
  return guard([&] {
    TedConfig c = derive_config(world, tp, experts);
    out5[0] = c.world_size;
    out5[1] = c.tensor_parallel;
    out5[2] = c.experts;
    out5[3] = c.expert_data_parallel;
    out5[4] = c.nonexpert_data_parallel;
  });
}

// Whole SerialModel step (attention stand-in + MoE + Adam) -> loss.
int ref_serial_step(int layers, int hidden, int experts, int tokens_per_shard,
                    std::uint64_t seed, int data_shards, int steps, double* losses) {
  return guard([&] {
    MoeModelConfig m{layers, hidden, experts, tokens_per_shard, seed};
    SerialModel s(m, data_shards);
    for (int i = 0; i < steps; ++i) losses[i] = s.step().loss;
  });
}

// Trainer step with rank-threads -> loss per step; also the forward ledger
// payload bytes of the expert all-to-all and tensor all-gather.
int ref_trainer_step(int layers, int hidden, int experts, int tokens_per_shard,
                     std::uint64_t seed, int world, int tp, int dtd, int ckpt, int cac,
                     int steps, double* losses, std::uint64_t* a2a_bytes,
                     std::uint64_t* ag_bytes) {
  return guard([&] {
    MoeModelConfig m{layers, hidden, experts, tokens_per_shard, seed};
    TrainerOptions o;
    o.flags.dtd = dtd != 0;
    o.flags.ckpt = ckpt != 0;
    o.flags.cac = cac != 0;
    Trainer t(m, derive_config(world, tp, experts), o);
    for (int i = 0; i < steps; ++i) losses[i] = t.step().loss;
    const CommLedger L = t.fabric().ledger_snapshot();
    if (a2a_bytes)
      *a2a_bytes = L.at(Phase::Forward, GroupKind::Expert, CollectiveOp::AllToAll).payload_bytes;
    if (ag_bytes)
      *ag_bytes = L.at(Phase::Forward, GroupKind::Tensor, CollectiveOp::AllGather).payload_bytes;
  });
}

// predict_comm_volume forward-phase payloads (summed over ranks).
int ref_predict_comm(int layers, int hidden, int experts, int tokens_per_shard, int world,
                     int tp, int dtd, int ckpt, int cac, std::uint64_t* out3) {
  return guard([&] {
    MoeModelConfig m{layers, hidden, experts, tokens_per_shard, 1};
    RunFlags fl;
    fl.dtd = dtd != 0;
    fl.ckpt = ckpt != 0;
    fl.cac = cac != 0;
    CommLedger L = predict_comm_volume(m, derive_config(world, tp, experts), fl, 1, true);
    out3[0] = L.at(Phase::Forward, GroupKind::Expert, CollectiveOp::AllToAll).payload_bytes;
    out3[1] = L.at(Phase::Forward, GroupKind::Tensor, CollectiveOp::AllGather).payload_bytes;
    out3[2] = L.at(Phase::Forward, GroupKind::Tensor, CollectiveOp::AllReduce).payload_bytes;
  });
}

}  // extern "C"
