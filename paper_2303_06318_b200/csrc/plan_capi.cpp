// plan_capi.cpp -- CPU-only C face of the exchange planner (ted_plan.h), so the
// multi-rank host logic can be tested with gloo on machines without a GPU.  The same
// header is compiled into libted_b200.so, where the NCCL calls consume the plan.
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>

#include "ted_plan.h"

namespace {
thread_local std::string g_err;
}

extern "C" {

const char* ted_plan_last_error() { return g_err.c_str(); }

// Flattened plan.  Arrays sized by the caller: seg_off [Eloc+1], seg_rows [Eloc],
// chunk_row [Tc+1], send_off [E]; transfer lists as (peer,row,rows) triples with
// capacity `cap` each; counts returned in counts[6] =
// {a2a_send, a2a_recv, ag_asm_send, ag_asm_recv, ag_home_send, ag_home_recv}.
int ted_plan_build(int P, int T, int E, int dtd, int my_ep, int my_t, const int* cnt,
                   int* seg_off, int* seg_rows, int64_t* chunk_row, int64_t* send_off,
                   int64_t* lists /* [6][cap][3] */, int cap, int* counts,
                   int64_t* totals /* asm_rows, send_rows, a2a_offrank, a2a_total */) {
  try {
    ted::LayerPlan L = ted::build_plan(P, T, E, dtd != 0, my_ep, my_t, cnt);
    std::memcpy(seg_off, L.seg_off.data(), sizeof(int) * L.seg_off.size());
    std::memcpy(seg_rows, L.seg_rows.data(), sizeof(int) * L.seg_rows.size());
    std::memcpy(chunk_row, L.chunk_row.data(), sizeof(int64_t) * L.chunk_row.size());
    std::memcpy(send_off, L.send_off.data(), sizeof(int64_t) * L.send_off.size());
    const std::vector<ted::PeerXfer>* v[6] = {&L.a2a_send,    &L.a2a_recv,     &L.ag_asm_send,
                                              &L.ag_asm_recv, &L.ag_home_send, &L.ag_home_recv};
    for (int i = 0; i < 6; ++i) {
      if (int(v[i]->size()) > cap) throw std::runtime_error("plan list capacity exceeded");
      counts[i] = int(v[i]->size());
      for (size_t j = 0; j < v[i]->size(); ++j) {
        int64_t* q = lists + (int64_t(i) * cap + int64_t(j)) * 3;
        q[0] = (*v[i])[j].peer;
        q[1] = (*v[i])[j].row;
        q[2] = (*v[i])[j].rows;
      }
    }
    totals[0] = L.asm_rows;
    totals[1] = L.send_rows;
    totals[2] = L.a2a_rows_offrank;
    totals[3] = L.a2a_rows_total;
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// blk_row / blk_cnt [Eloc][Tc][P] of this rank's assembled layout
int ted_plan_blocks(int P, int T, int E, int dtd, int my_ep, int my_t, const int* cnt,
                    int64_t* blk_row, int* blk_cnt) {
  try {
    ted::LayerPlan L = ted::build_plan(P, T, E, dtd != 0, my_ep, my_t, cnt);
    std::memcpy(blk_row, L.blk_row.data(), sizeof(int64_t) * L.blk_row.size());
    std::memcpy(blk_cnt, L.blk_cnt.data(), sizeof(int) * L.blk_cnt.size());
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// the device plan's per-expert function run on the CPU (kc_all: [plane][Tc][E] in plane
// order t + T*ep): seg [2*Eloc+1], disp_base [E], pull_base [Tc][E]
int ted_plan_peer_tables(int T, int P, int E, int Tc, int my_ep, int my_c, const int* kc_all,
                         int* seg, long long* disp_base, long long* pull_base) {
  if (E < 1 || P < 1 || E % P != 0) {
    g_err = "experts must be a multiple of the expert-parallel degree";
    return 2;
  }
  for (int e = 0; e < E; ++e)
    ted::peer_plan_expert(kc_all, T, P, E, Tc, my_ep, my_c, e, disp_base, pull_base, seg);
  return 0;
}

}  // extern "C"
