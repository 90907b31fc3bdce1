// ted_plan.h -- host-side exchange plan for one MoE layer on one rank (pure C++, no CUDA).
//
// Restates the reference's dispatch bookkeeping (moe.cpp:454-530, DTD :440-452,
// :478-493, :532-552) for the B200 layout, generalised to E experts over an EP group
// of P members (E_loc = E / P local experts; the reference forces E_loc = 1,
// topology.cpp:23-28):
//
//   send layout (per source rank, chunk c it dispatches): experts ascending, each
//       expert's kept rows in ascending token order (moe.cpp:456-462).
//   assembled layout (expert rank): local expert major; inside an expert, TP member
//       (= DTD chunk) major, then source member (moe.cpp:465-489); every expert
//       segment padded to 128 rows for the tensor-core tiles.
//   home layout (source rank, all chunks): chunk major, then experts ascending --
//       chunk c is exactly what TP member c dispatched (moe.cpp:532-536).
//
// Input: cnt[s][c][e] = kept rows of source s (EP position), chunk c, expert e --
// gathered over the EP group.  TP peers route identical replicated tokens, so the
// per-chunk counts of every chunk are known to every TP peer.
#pragma once
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace ted {

struct PeerXfer {
  int peer;        // member position in the communicator
  int64_t row;     // first row in the local buffer
  int64_t rows;    // row count (> 0)
};

struct LayerPlan {
  int P = 1, T = 1, E = 1, Eloc = 1, Tc = 1;
  int my_ep = 0, my_t = 0;
  bool dtd = false;
  // assembled layout
  std::vector<int> seg_off;    // [Eloc+1] padded
  std::vector<int> seg_rows;   // [Eloc]   real rows
  std::vector<int64_t> blk_row;  // [Eloc][Tc][P] first row of block (le, c, s)
  std::vector<int> blk_cnt;      // [Eloc][Tc][P]
  int64_t asm_rows = 0;        // seg_off[Eloc]
  // home layout
  std::vector<int64_t> chunk_row;  // [Tc+1] first home row of chunk c
  std::vector<int64_t> send_off;   // [E] row of expert e inside my chunk's send block
  int64_t send_rows = 0;           // rows I dispatch
  // EP all-to-all (dispatch direction; the return trip swaps send/recv)
  std::vector<PeerXfer> a2a_send;  // rows of my send buffer -> EP member (one per (m, le))
  std::vector<PeerXfer> a2a_recv;  // rows of assembled buffer <- EP member
  // TP all-gather-v (DTD), assembled side and home side
  std::vector<PeerXfer> ag_asm_send, ag_asm_recv;
  std::vector<PeerXfer> ag_home_send, ag_home_recv;
  // byte accounting (payload rows; x h x 2 B for the ledger)
  int64_t a2a_rows_offrank = 0;  // rows that leave this rank in the dispatch A2A
  int64_t a2a_rows_total = 0;    // all dispatch rows incl. self (reference ledger rule)
};

inline int64_t pad_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

// cnt: [P][Tc][E] row-major.  Tc = dtd ? T : 1.  my_chunk = dtd ? my_t : 0.
inline LayerPlan build_plan(int P, int T, int E, bool dtd, int my_ep, int my_t,
                            const int* cnt) {
  if (P < 1 || T < 1 || E < 1 || E % P != 0)
    throw std::invalid_argument("plan: experts (" + std::to_string(E) +
                                ") must be a multiple of the expert-parallel degree (" +
                                std::to_string(P) + ")");
  LayerPlan L;
  L.P = P;
  L.T = T;
  L.E = E;
  L.Eloc = E / P;
  L.dtd = dtd && T > 1;
  L.Tc = L.dtd ? T : 1;
  L.my_ep = my_ep;
  L.my_t = my_t;
  const int Tc = L.Tc, Eloc = L.Eloc;
  const int my_c = L.dtd ? my_t : 0;
  auto C = [&](int s, int c, int e) { return cnt[(int64_t(s) * Tc + c) * E + e]; };

  // assembled layout
  L.seg_off.assign(Eloc + 1, 0);
  L.seg_rows.assign(Eloc, 0);
  L.blk_row.assign(size_t(Eloc) * Tc * P, 0);
  L.blk_cnt.assign(size_t(Eloc) * Tc * P, 0);
  int64_t off = 0;
  for (int le = 0; le < Eloc; ++le) {
    const int e = my_ep * Eloc + le;
    L.seg_off[le] = int(off);
    int64_t r = off;
    for (int c = 0; c < Tc; ++c)
      for (int s = 0; s < P; ++s) {
        const size_t i = (size_t(le) * Tc + c) * P + s;
        L.blk_row[i] = r;
        L.blk_cnt[i] = C(s, c, e);
        r += C(s, c, e);
      }
    L.seg_rows[le] = int(r - off);
    off = pad_up(r, 128);
  }
  L.seg_off[Eloc] = int(off);
  L.asm_rows = off;

  // home layout (my own shard; identical on TP peers)
  L.chunk_row.assign(Tc + 1, 0);
  for (int c = 0; c < Tc; ++c) {
    int64_t s = 0;
    for (int e = 0; e < E; ++e) s += C(my_ep, c, e);
    L.chunk_row[c + 1] = L.chunk_row[c] + s;
  }
  L.send_off.assign(E, 0);
  {
    int64_t o = 0;
    for (int e = 0; e < E; ++e) {
      L.send_off[e] = o;
      o += C(my_ep, my_c, e);
    }
    L.send_rows = o;
  }

  // dispatch A2A: to member m, expert e = m*Eloc + le, rows C(my_ep, my_c, e)
  for (int m = 0; m < P; ++m)
    for (int le = 0; le < Eloc; ++le) {
      const int e = m * Eloc + le;
      const int64_t rows = C(my_ep, my_c, e);
      L.a2a_rows_total += rows;
      if (m != my_ep) L.a2a_rows_offrank += rows;
      if (rows > 0) L.a2a_send.push_back({m, L.send_off[e], rows});
    }
  // receive from source s, my local expert le, chunk my_c
  for (int s = 0; s < P; ++s)
    for (int le = 0; le < Eloc; ++le) {
      const size_t i = (size_t(le) * Tc + my_c) * P + s;
      if (L.blk_cnt[i] > 0) L.a2a_recv.push_back({s, L.blk_row[i], L.blk_cnt[i]});
    }

  if (L.dtd) {
    // assembled-side AG-v over TP: my blocks (le, my_c, *) to every peer; theirs back.
    for (int t = 0; t < T; ++t) {
      if (t == my_t) continue;
      for (int le = 0; le < Eloc; ++le) {
        const size_t mine = (size_t(le) * Tc + my_c) * P;
        int64_t rows = 0;
        for (int s = 0; s < P; ++s) rows += L.blk_cnt[mine + s];
        if (rows > 0) L.ag_asm_send.push_back({t, L.blk_row[mine], rows});
        const size_t theirs = (size_t(le) * Tc + t) * P;
        int64_t rr = 0;
        for (int s = 0; s < P; ++s) rr += L.blk_cnt[theirs + s];
        if (rr > 0) L.ag_asm_recv.push_back({t, L.blk_row[theirs], rr});
      }
    }
    // home-side AG-v over TP: chunk my_c to peers; chunk t from peer t.
    for (int t = 0; t < T; ++t) {
      if (t == my_t) continue;
      const int64_t mine = L.chunk_row[my_c + 1] - L.chunk_row[my_c];
      if (mine > 0) L.ag_home_send.push_back({t, L.chunk_row[my_c], mine});
      const int64_t theirs = L.chunk_row[t + 1] - L.chunk_row[t];
      if (theirs > 0) L.ag_home_recv.push_back({t, L.chunk_row[t], theirs});
    }
  }
  return L;
}

#ifdef __CUDACC__
#define TED_HD __host__ __device__
#else
#define TED_HD
#endif

// The peer-exchange plan as the device computes it (plan_peer_kernel, one call per
// expert e): from the plane-gathered chunk counts (member t + T*ep contributes [Tc][E];
// the t = 0 members' rows are the sources' counts) the row where this rank's block
// (expert e, chunk c, source my_ep) starts in e's assembled buffer -- pull_base[c*E + e],
// and disp_base[e] for this rank's own chunk my_c -- plus, for a local expert, its
// segment (seg[le] = start, seg[Eloc+1+le] = valid rows, seg[Eloc] = padded end).  Same
// offsets as build_plan's blk_row / seg_off (tested on the CPU through plan_capi.cpp).
TED_HD inline void peer_plan_expert(const int* kc_all, int T, int P, int E, int Tc, int my_ep,
                                    int my_c, int e, long long* disp_base,
                                    long long* pull_base, int* seg) {
  const int Eloc = E / P;
  const int ep2 = e / Eloc, le = e % Eloc;
  auto C = [&](int s_, int c, int ee) { return kc_all[(int64_t(T) * s_ * Tc + c) * E + ee]; };
  long long base = 0;  // segment start of local expert le on rank ep2 (128-padded)
  for (int l2 = 0; l2 < le; ++l2) {
    long long rows = 0;
    for (int c = 0; c < Tc; ++c)
      for (int s_ = 0; s_ < P; ++s_) rows += C(s_, c, ep2 * Eloc + l2);
    base += (rows + 127) / 128 * 128;
  }
  long long r = base;
  for (int c = 0; c < Tc; ++c) {
    long long before = 0;
    for (int s_ = 0; s_ < my_ep; ++s_) before += C(s_, c, e);
    pull_base[c * E + e] = r + before;
    if (c == my_c) disp_base[e] = r + before;
    for (int s_ = 0; s_ < P; ++s_) r += C(s_, c, e);
  }
  if (ep2 == my_ep) {
    seg[le] = int(base);
    seg[Eloc + 1 + le] = int(r - base);
    if (le == Eloc - 1) seg[Eloc] = int((r + 127) / 128 * 128);
  }
}

}  // namespace ted
