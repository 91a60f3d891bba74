// Chain-per-SM engine: Simulation::step() x n (engine.hpp:293-308, 350-426)
// run by ONE persistent CTA, so that K chains of a mu/T sweep each own an SM
// ("multiple large-scale simulations on a single GPU
// simultaneously"; the paper's microcell kernel already runs on one SM,
// PAPER.md:608).
//
// The multi-SM engine (engine2.cu) spreads one chain over the whole GPU and
// pays cross-SM flag latency (~1 us per hop, ~20 us per round) for it; at the
// dilute sweep state points a round ends after ~47 moves whatever its size,
// so that latency is the whole cost. Here every hand-off of a round is a CTA
// barrier and the state is private to the SM. A round of 64 move slots:
//
//   evaluate  each half-warp takes one slot: S(n) over the pruned 3x3x3 brick
//             window of the new point (occupancies from a shared-memory
//             replica of the mirror's, records from L2), and per lane one
//             candidate N offset d = -8..7: pid = index_from(pick, N + d),
//             e[pid], ΔU, the acceptance test and the overflow test (the
//             maintained-energy form of engine2.cu: displace ΔU = S(n) -
//             pair(n, x_pid) - e[pid], insert ΔU = S(n), delete ΔU = -e[pid]);
//   walk      one warp walks the slots in move order tracking d (ballots);
//   verify    each warp checks its slots against the earlier accepted moves:
//             a consumed move that read anything an earlier accepted move of
//             the round changes (its particle index, its target brick / cell,
//             a changed position within r_c of its new point or of its
//             particle), or an accepted move within 2 r_c of an earlier one,
//             ends the round there (it is re-evaluated in the next round);
//   commit    one warp per accepted move applies the neighbours' e updates
//             (old window first, then new; the round's accepted moves are
//             > 2 r_c apart so the sets are disjoint) with fire-and-forget
//             atomics, while one warp loads the structural commits
//             (commit.cuh; the movers' records were fetched during the
//             verify) and orders them, and one refills the proposal ring and
//             accumulates the statistics / trace; after a barrier the
//             structural stores (a deletion relabelling a particle inserted
//             earlier in the round takes its data from that insertion;
//             commits that touch an earlier one are re-loaded and applied
//             after it, in move order) and the movers' e (in move order).
//
// Windows use the brick's known periodic image (dims >= 5) instead of
// box.hpp's rint, with the same operations and roundings.
//
// The chain is the reference's: the same proposals (gen.cu), the same
// acceptance arithmetic and order, the same grid and mirror commits
// (byte-identical reference layout) — tests/test_gpu_engine_sm.py.
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "commit.cuh"
#include "internal.h"
#include "slot.cuh"
#include "sync.cuh"

namespace gcmcb {

namespace {

#ifndef GCMC_SM_THREADS
#define GCMC_SM_THREADS 512
#endif
constexpr int kST = GCMC_SM_THREADS;  // threads (256: no register cap below 255, no spills)
constexpr int kSW = kST / 32;       // warps
constexpr int kSM = 64;             // move slots per round
constexpr int kSAhead = 2 * kSM;    // proposals loaded ahead of the round
constexpr int kSRing = 4 * kSM;     // proposal ring (a refill never reaches the current round)
#ifndef GCMC_SM_ACC
#define GCMC_SM_ACC 24
#endif
constexpr int kSAcc = GCMC_SM_ACC;  // accepted moves per round (at most)
constexpr int kSOff = 16;           // N offsets per slot: d = -8..7 <-> half-warp lane d + 8
constexpr int kSHalf = kSOff / 2;
constexpr int kEW = kSW - 2;        // warps applying neighbour energy updates
constexpr int kCW = kSW - 2;        // warp loading / storing the structural commits
constexpr int kXW = kSW - 1;        // warp: proposal ring, statistics, trace
constexpr int kStash = 48;          // new-window updates buffered per e-update warp
constexpr int kSCand = 384;         // window candidates expanded per workspace (beyond: searched)
constexpr double kSHuge = 1e4;
#ifndef GCMC_SM_UNROLL
#define GCMC_SM_UNROLL 4  // window candidates per lane in flight (evaluation)
#endif      // |pair(n, x_pid)| above this: re-sum without pid

struct SmArgs {
  Grid g;
  Mirror m;
  Box b;
  Store s;
  double2* ep;
  ChainState* st;
  const Proposal* props;
  gcmc_trace_rec* trace;
  uint64_t nmoves, capn;
  double beta, mu, lambda3, vol, temp;
  uint64_t equil, interval;
  int tail;
  double tail_cu, tail_cp, tail_s3, tail_bu, tail_bp;
  int smem_occ;  // mirror occupancy replica in shared memory
  int max_acc;
  unsigned long long* diag;  // GCMC_SM_PHASES: per-role cycles per round (max over warps)
};

// A window workspace: bricks, exclusive occupancy prefix and the expanded
// (brick entry << 7 | slot) candidate list (slot.cuh's layout, sized small:
// shared memory left to L1 keeps the call frames cached).
struct SWs {
  uint32_t brick[kMaxEnt];
  uint8_t sc[kMaxEnt];  // periodic image of each brick: 2 bits per axis (0: none, 1: +L, 2: -L)
  int pre[kMaxEnt + 1];
  uint16_t cand[kSCand];
  int nent0, nent, total;
};

struct WalkRes {  // one warp's walk of the round
  int len, nacc, err, why;
  int acc_i[kSAcc];
  int acc_d[kSAcc];
  int8_t d[kSM];  // N offset before each slot
};

struct SmShared {
  Proposal ring[kSRing];
  // evaluation results per slot and N offset
  double off_du[kSM][kSOff], off_dw[kSM][kSOff], off_mu[kSM][kSOff], off_mw[kSM][kSOff];
  float off_x[kSM][kSOff][3];   // position of the offset's particle (conflict tests; exact: the store)
  int32_t off_ia[kSM][kSOff];   // the offset's particle (insert: the new index), -1: none
  uint32_t off_po[kSM][kSOff];  // brick point of its position (kNoPoint: none)
  int32_t off_co[kSM][kSOff];   // reference cell of its position
  uint32_t macc[kSM], movf[kSM];
  uint32_t ptn[kSM];            // brick point of the new position (kNoPoint: deletion)
  int32_t cn[kSM];              // reference cell of the new position
  uint8_t mkind[kSM];
  WalkRes wr[1];
  int cmin;
  // structural commits
  MoveData md[kSAcc];
  CommitIn cin[kSAcc];
  int8_t cfwd[kSAcc];   // forwarded deletion: the insertion lane it takes q from (-1: none)
  Touch ctouch[kSAcc];  // commit ordering scratch
  unsigned cexm[kSAcc], cdepm;
  int8_t ckind[kSAcc];
  double4 xacc[kSAcc];  // the accepted movers' store records (exact position, record), loaded in the verify
  int32_t rsacc[kSAcc]; // ... and reference slots
  uint8_t cskip[kSAcc]; // insertion relabelled away by a forwarded deletion: index n not written
  uint32_t cdep;
  // window workspaces: [warp][half] (evaluation), [warp][0] (energy updates)
  SWs ws[kSW][2];
  struct Stash {
    int32_t id[kStash];
    double u[kStash], w[kStash];
  } stash[kEW];
  // statistics
  double st_e[kSAcc + 1], st_w[kSAcc + 1];
  uint64_t st_n[kSAcc + 1];
  double st_v[kSAcc + 1][4];
  unsigned smp[kSM / 32];
  ChainState ks;
  unsigned long long pairs;
  unsigned long long stops[6];
  uint64_t base, n;  // the round's first move and N
  uint64_t nprev;    // N at the start of the previous round (error report)
  unsigned long long rmax[16], racc[16];  // diagnostics: role cycles (round max, sum)
};

enum SStop { kSEnd, kSRange, kSVerify, kSFull, kSOverflow };

__device__ __forceinline__ bool grid_on(const SmArgs& a) { return a.g.kind != GCMC_ALL_PAIRS; }

// The round after the verify: the walk's prefix cut at the first conflict.
struct RoundOut {
  int len, nacc, err;
};
__device__ __forceinline__ RoundOut round_out(const SmShared& sh) {
  const WalkRes& w = sh.wr[0];
  RoundOut r{w.len, w.nacc, w.err};
  if (sh.cmin < w.len) {
    r.len = sh.cmin;
    r.err = 0;
    int k = 0;
    while (k < w.nacc && w.acc_i[k] < r.len) ++k;
    r.nacc = k;
  }
  return r;
}

// Occupancies (replica or global), exclusive prefix over nent <= 54 bricks and
// the candidate expansion (slot.cuh's win_finish for one warp and SWs).
__device__ __forceinline__ void win_finish_s(const Mirror& m, SWs& ws, const uint8_t* occ_s, int nent,
                                             int nent0, int lane) {
  __syncwarp();
  int o0 = 0, o1 = 0;
  if (lane < nent) {
    const uint32_t id = ws.brick[lane];
    o0 = occ_s ? (int)occ_s[id] : __ldcg(m.occ + id);
  }
  if (lane + 32 < nent) {
    const uint32_t id = ws.brick[lane + 32];
    o1 = occ_s ? (int)occ_s[id] : __ldcg(m.occ + id);
  }
  int sc = o0 | (o1 << 16);
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, sc, o);
    if (lane >= o) sc += t;
  }
  const int last = __shfl_sync(0xffffffffu, sc, 31);
  const int tot0 = last & 0xffff;
  const int e0 = (sc & 0xffff) - o0, e1 = tot0 + (sc >> 16) - o1;
  if (lane < nent) ws.pre[lane] = e0;
  if (lane + 32 < nent) ws.pre[lane + 32] = e1;
  const int total = tot0 + (last >> 16);
  if (lane == 0) {
    ws.nent0 = nent0;
    ws.nent = nent;
    ws.pre[nent] = total;
    ws.total = total;
  }
#pragma unroll 1
  for (int k = 0; k < o0; ++k)
    if (e0 + k < kSCand) ws.cand[e0 + k] = (uint16_t)((lane << 7) | k);
#pragma unroll 1
  for (int k = 0; k < o1; ++k)
    if (e1 + k < kSCand) ws.cand[e1 + k] = (uint16_t)(((lane + 32) << 7) | k);
}

// Record index of window candidate f.
__device__ __forceinline__ int cand_record(const Mirror& m, const SWs& ws, int f, int* ent = nullptr) {
  int e, k;
  if (f < kSCand) {
    const int c = ws.cand[f];
    e = c >> 7;
    k = c & 127;
  } else {
    int lo = 0, hi = ws.nent - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (ws.pre[mid] <= f) lo = mid; else hi = mid - 1;
    }
    e = lo;
    k = f - ws.pre[lo];
  }
  if (ent) *ent = e;
  return (int)ws.brick[e] * m.cap + k;
}

// Image code of the brick at window offset o (0..26) around brick point
// (cx, cy, cz): per axis whether the neighbour wraps (+L: beyond the upper
// face, -L: below 0). With dims >= 5 the minimum-image shift of every record
// in that brick relative to any point of the centre brick is exactly that
// (|dx| <= 2 L / dims < L / 2 inside, >= L - 2 L / dims > L / 2 wrapped), so
// rint(dx / L) of box.hpp:45-55 is known without computing it.
__device__ __forceinline__ uint8_t image_code(int cx, int cy, int cz, int o, int d) {
  const int x = cx + o % 3 - 1, y = cy + (o / 3) % 3 - 1, z = cz + o / 9 - 1;
  return (uint8_t)((x < 0 ? 2 : (x >= d ? 1 : 0)) | ((y < 0 ? 2 : (y >= d ? 1 : 0)) << 2) |
                   ((z < 0 ? 2 : (z >= d ? 1 : 0)) << 4));
}
__device__ __forceinline__ double image_shift(unsigned c, double l) {
  return c == 0u ? 0.0 : (c == 1u ? l : -l);
}
// min_image_dist2 (common.cuh) with the image known: the same operations and
// roundings (dx - L * rint(dx / L) with rint = 0 / +1 / -1 is dx - 0 / L / -L).
__device__ __forceinline__ double image_dist2(double ax, double ay, double az, double bx, double by,
                                              double bz, unsigned code, double l) {
  const double dx = __dsub_rn(__dsub_rn(ax, bx), image_shift(code & 3u, l));
  const double dy = __dsub_rn(__dsub_rn(ay, by), image_shift((code >> 2) & 3u, l));
  const double dz = __dsub_rn(__dsub_rn(az, bz), image_shift((code >> 4) & 3u, l));
  return __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
}
// The pair distance of a window candidate: known image when dims >= 5.
__device__ __forceinline__ double cand_dist2(const Mirror& m, const Box& b, const SWs& ws, int e, double px,
                                             double py, double pz, double rx, double ry, double rz) {
  return m.dims >= 5 ? image_dist2(px, py, pz, rx, ry, rz, ws.sc[e], b.l)
                     : min_image_dist2(px, py, pz, rx, ry, rz, b);
}

// engine.hpp:28-59 with one exponential (same operation order): the exchange
// ratio's prefactor for N = nd, then the acceptance probability of ΔU.
__device__ __forceinline__ double exchange_prefactor(const SmArgs& a, int kind, int64_t nd) {
  const double nn = (double)nd;
  return kind == 1 ? __ddiv_rn(a.vol, __dmul_rn(a.lambda3, __dadd_rn(nn, 1.0)))
                   : (kind == 2 ? __ddiv_rn(__dmul_rn(a.lambda3, nn), a.vol) : 1.0);
}
__device__ __forceinline__ double accept_prob(const SmArgs& a, int kind, double du, double fpre) {
  const double x = kind == 0 ? __dmul_rn(-a.beta, du)
                 : (kind == 1 ? __dmul_rn(a.beta, __dsub_rn(a.mu, du)) : __dmul_rn(-a.beta, __dadd_rn(a.mu, du)));
  const double ex = exp(x);
  return metropolis(kind == 0 ? ex : __dmul_rn(fpre, ex));
}

// ------------------------------------------------------------- evaluation
// Half-warp window of point (x, y, z): the pruned 3x3x3 brick window (from
// the proposal's precomputed offset mask when present), occupancies and the
// expansion. hl = lane in the half (0..15); each lane takes offsets hl and
// hl + 16 of the window and entries hl and hl + 16 of the compacted list.
__device__ __forceinline__ void half_window(const SmArgs& a, SWs& ws, const uint8_t* occ_s, const Proposal& pr,
                                            bool on, int hl, int hw) {
  const Mirror& m = a.m;
  uint32_t wm = 0u, bpt = 0u;
  if (on) {
    if (pr.wmask != kNoMask) {
      wm = pr.wmask;
      bpt = pr.bpt;
    } else {
      bpt = (uint32_t)mpoint(m, pr.x, pr.y, pr.z);
    }
  }
  const bool pruned = on && m.dims >= 3 && pr.wmask == kNoMask;  // window not precomputed
  uint32_t wl = 0u;
  if (pruned) {
    uint32_t id;
    const bool k0 = window_keep(m, a.b, pr.x, pr.y, pr.z, pt_x(bpt), pt_y(bpt), pt_z(bpt), hl, id);
    const bool k1 = hl + 16 < 27 && window_keep(m, a.b, pr.x, pr.y, pr.z, pt_x(bpt), pt_y(bpt), pt_z(bpt), hl + 16, id);
    wl = (k0 ? 1u << hl : 0u) | (k1 ? 1u << (hl + 16) : 0u);
  }
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) wl |= __shfl_xor_sync(0xffffffffu, wl, o, 16);
  if (pruned) wm = wl;
  if (m.dims < 3) wm = on ? (1u << m.nb) - 1u : 0u;  // tiny boxes: every brick
  if (!on) wm = 0u;
  if (m.dims < 3) {
    if (hl < (int)m.nb) ws.brick[hl] = (uint32_t)hl;
    if (hl + 16 < (int)m.nb) ws.brick[hl + 16] = (uint32_t)(hl + 16);
  } else {
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const int o = hl + 16 * t;
      if (o < 27 && ((wm >> o) & 1u)) {
        const int d = m.dims;
        int cx = pt_x(bpt) + o % 3 - 1, cy = pt_y(bpt) + (o / 3) % 3 - 1, cz = pt_z(bpt) + o / 9 - 1;
        cx += cx < 0 ? d : 0;
        cx -= cx >= d ? d : 0;
        cy += cy < 0 ? d : 0;
        cy -= cy >= d ? d : 0;
        cz += cz < 0 ? d : 0;
        cz -= cz >= d ? d : 0;
        const int at = __popc(wm & ((1u << o) - 1u));
        ws.brick[at] = (uint32_t)cx + (uint32_t)d * ((uint32_t)cy + (uint32_t)d * (uint32_t)cz);
        ws.sc[at] = image_code(pt_x(bpt), pt_y(bpt), pt_z(bpt), o, d);
      }
    }
  }
  const int nent = __popc(wm);
  __syncwarp();
  int o0 = 0, o1 = 0;
  if (hl < nent) {
    const uint32_t id = ws.brick[hl];
    o0 = occ_s ? (int)occ_s[id] : __ldcg(m.occ + id);
  }
  if (hl + 16 < nent) {
    const uint32_t id = ws.brick[hl + 16];
    o1 = occ_s ? (int)occ_s[id] : __ldcg(m.occ + id);
  }
  int sc = o0 | (o1 << 16);
#pragma unroll
  for (int o = 1; o < 16; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, sc, o, 16);
    if (hl >= o) sc += t;
  }
  const int last = __shfl_sync(0xffffffffu, sc, 15, 16);
  const int tot0 = last & 0xffff;
  const int e0 = (sc & 0xffff) - o0, e1 = tot0 + (sc >> 16) - o1;
  if (hl < nent) ws.pre[hl] = e0;
  if (hl + 16 < nent) ws.pre[hl + 16] = e1;
  const int total = tot0 + (last >> 16);
  if (hl == 0) {
    ws.nent0 = nent;
    ws.nent = nent;
    ws.pre[nent] = total;
    ws.total = total;
  }
#pragma unroll 1
  for (int k = 0; k < o0; ++k)
    if (e0 + k < kSCand) ws.cand[e0 + k] = (uint16_t)((hl << 7) | k);
#pragma unroll 1
  for (int k = 0; k < o1; ++k)
    if (e1 + k < kSCand) ws.cand[e1 + k] = (uint16_t)(((hl + 16) << 7) | k);
  __syncwarp();
}

template <bool kImg, int U>
__device__ __forceinline__ void half_sum_t(const Mirror& m, const Box& b, const SWs& ws, double px, double py,
                                           double pz, int excl, bool on, int hl, double& su, double& sw) {
  su = 0.0;
  sw = 0.0;
  const int total = on ? ws.total : 0;
  const int tmax = max(total, __shfl_xor_sync(0xffffffffu, total, 16));
#pragma unroll 1
  for (int base = 0; base < tmax; base += 16 * U) {
    double rx[U], ry[U], rz[U];
    bool ok[U];
    int ent[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int f = base + 16 * u + hl;
      ok[u] = f < total;
      rx[u] = ry[u] = rz[u] = 0.0;
      ent[u] = 0;
      if (ok[u]) {
        const int idx = cand_record(m, ws, f, &ent[u]);
        if (idx == excl) {
          ok[u] = false;
        } else {
          rx[u] = __ldcg(m.rx + idx);
          ry[u] = __ldcg(m.ry + idx);
          rz[u] = __ldcg(m.rz + idx);
        }
      }
    }
    // branch-free: the four pair chains interleave (a term outside r_c adds
    // +0.0, which leaves the sum's bits unchanged)
    double pu[U], pw[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const double r2 = kImg ? image_dist2(px, py, pz, rx[u], ry[u], rz[u], ws.sc[ent[u]], b.l)
                             : min_image_dist2(px, py, pz, rx[u], ry[u], rz[u], b);
      const bool in = ok[u] && r2 <= b.rc2;
      double tu, tw;
      lj_pair_clamped(in ? r2 : b.rc2, b, tu, tw);
      pu[u] = in ? tu : 0.0;
      pw[u] = in ? tw : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      su = __dadd_rn(su, pu[u]);
      sw = __dadd_rn(sw, pw[u]);
    }
  }
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) {
    su = __dadd_rn(su, __shfl_xor_sync(0xffffffffu, su, o, 16));
    sw = __dadd_rn(sw, __shfl_xor_sync(0xffffffffu, sw, o, 16));
  }
}

// Half-warp Σ pair(p, record) over the workspace's candidates except record
// `excl`: four candidates per lane in flight, lane sums then an xor tree
// inside the half (fixed order: every lane of the half gets the same bits).
__device__ __forceinline__ void half_sum(const Mirror& m, const Box& b, const SWs& ws, double px, double py,
                                         double pz, int excl, bool on, int hl, double& su, double& sw) {
  if (m.dims >= 5)
    half_sum_t<true, GCMC_SM_UNROLL>(m, b, ws, px, py, pz, excl, on, hl, su, sw);
  else
    half_sum_t<false, GCMC_SM_UNROLL>(m, b, ws, px, py, pz, excl, on, hl, su, sw);
}

// Two slots per warp call: half hw evaluates slot s0 + kSW * hw.
__device__ __forceinline__ void eval_pair(const SmArgs& a, SmShared& sh, const uint8_t* occ_s, int s0,
                                          int fit, uint64_t base, uint64_t n, int warp, int lane) {
  // diagnostics build (-DGCMC_SM_STEPS): cycles of the steps, max over warps
  unsigned long long tq = clock64();
  auto step = [&](int k) {
#ifdef GCMC_SM_EVAL_STEPS
    const unsigned long long t = clock64();
    if (lane == 0) atomicMax(&sh.rmax[k], t - tq);
    tq = t;
#else
    (void)k;
#endif
  };
  const int hw = lane >> 4, hl = lane & 15;
  const int s = s0 + kSW * hw;
  const bool on = s < fit;
  const Proposal& pr = sh.ring[(base + (uint64_t)(on ? s : s0)) % kSRing];
  const int kind = on ? pr.kind : 2;
  const bool grid = grid_on(a);
  const int dd = hl - kSHalf;
  const int64_t nd = (int64_t)n + dd;
  const bool valid = on && (kind == 1 ? nd >= 0 : nd >= 1);  // kinds 0/2 at N <= 0: counted rejection
  uint64_t pid = 0;
  double xox = 0.0, xoy = 0.0, xoz = 0.0, eu = 0.0, ew = 0.0;
  int xrec = -1;
  // candidate particles (one L2 hop, issued first)
  if (kind != 1 && valid) {
    pid = index_from(pr.pick, (uint64_t)nd);
    if (pid < a.capn) {  // beyond the store: an index this round inserts (the verify stops there)
      const double4 o = ld_cg(a.s.pos + pid);
      xox = o.x;
      xoy = o.y;
      xoz = o.z;
      xrec = bslot_in(o);
      const double2 e2 = __ldcg(a.ep + pid);
      eu = e2.x;
      ew = e2.y;
    }
  }
  const double fpre = exchange_prefactor(a, kind, nd);
  step(9);
  SWs& ws = sh.ws[warp][hw];
  const bool win = on && kind != 2;
  uint32_t pn = (uint32_t)kNoPoint;
  int cb = -1, ob = 0, ocb = 0;
  if (win) {
    pn = (uint32_t)(pr.wmask != kNoMask ? (uint64_t)pr.bpt : mpoint(a.m, pr.x, pr.y, pr.z));
    cb = grid ? (pr.wmask != kNoMask ? pr.cell : cell_of(a.g, pr.x, pr.y, pr.z)) : -1;
    ob = occ_s ? (int)occ_s[mbrick(a.m, pn)] : __ldcg(a.m.occ + mbrick(a.m, pn));
    if (grid) ocb = __ldcg(a.g.occ + cb);
  }
  half_window(a, ws, occ_s, pr, win, hl, hw);
  step(10);
  double su = 0.0, sw = 0.0;
  half_sum(a.m, a.b, ws, pr.x, pr.y, pr.z, -1, win, hl, su, sw);
  step(11);
  if (win && hl == 0) atomicAdd(&sh.pairs, (unsigned long long)ws.total);
  double du = 0.0, dw = 0.0, mu_ = 0.0, mw = 0.0, p = 0.0;
  bool slow = false;
  if (valid) {
    if (kind == 1) {
      du = su;
      dw = sw;
      mu_ = su;
      mw = sw;
    } else if (kind == 0) {
      const double r2 = min_image_dist2(pr.x, pr.y, pr.z, xox, xoy, xoz, a.b);
      double tu = 0.0, tw = 0.0;
      if (r2 <= a.b.rc2) lj_pair_clamped(r2, a.b, tu, tw);
      slow = fabs(tu) > kSHuge || fabs(tw) > kSHuge;
      mu_ = __dsub_rn(su, tu);
      mw = __dsub_rn(sw, tw);
    } else {
      du = -eu;
      dw = -ew;
    }
  }
  // rare: the mover's own pair is large -> S(n) without its record, re-summed
  unsigned sl = __ballot_sync(0xffffffffu, slow);
  while (sl) {
    const int src = __ffs(sl) - 1;
    sl &= sl - 1;
    const int xr = __shfl_sync(0xffffffffu, xrec, src);
    const bool mine = (src >> 4) == hw;
    double au, aw;
    half_sum(a.m, a.b, ws, pr.x, pr.y, pr.z, xr, win && mine, hl, au, aw);
    if (lane == src) {
      mu_ = au;
      mw = aw;
    }
  }
  if (kind == 0) {
    du = __dsub_rn(mu_, eu);
    dw = __dsub_rn(mw, ew);
  }
  {
    const double pp = accept_prob(a, kind, du, fpre);
    if (valid) p = pp;
  }
  const bool acc = valid && pr.acc < p;
  step(12);
  // overflow of the commit (exact: occupancies before the round)
  bool ovf = false;
  if (valid && kind != 2) {
    const bool same_b = kind == 0 && mbrick(a.m, mpoint(a.m, xox, xoy, xoz)) == mbrick(a.m, pn);
    if (!same_b && ob >= a.m.cap) ovf = true;
    if (grid) {
      const bool same_c = kind == 0 && cell_of(a.g, xox, xoy, xoz) == cb;
      if (!same_c && ocb >= a.g.cap) ovf = true;
    }
  }
  const uint32_t accm = (__ballot_sync(0xffffffffu, acc) >> (16 * hw)) & 0xffffu;
  const uint32_t ovm = (__ballot_sync(0xffffffffu, ovf) >> (16 * hw)) & 0xffffu;
  if (on) {
    sh.off_du[s][hl] = du;
    sh.off_dw[s][hl] = dw;
    sh.off_mu[s][hl] = mu_;
    sh.off_mw[s][hl] = mw;
    sh.off_x[s][hl][0] = (float)xox;
    sh.off_x[s][hl][1] = (float)xoy;
    sh.off_x[s][hl][2] = (float)xoz;
    const bool has_x = kind != 1 && nd >= 1 && pid < a.capn;
    sh.off_ia[s][hl] = kind == 1 ? (int32_t)nd : (nd >= 1 ? (int32_t)pid : -1);
    sh.off_po[s][hl] = has_x ? (uint32_t)mpoint(a.m, xox, xoy, xoz) : (uint32_t)kNoPoint;
    sh.off_co[s][hl] = has_x && grid ? cell_of(a.g, xox, xoy, xoz) : -1;
    if (hl == 0) {
      sh.macc[s] = accm;
      sh.movf[s] = ovm;
      sh.mkind[s] = (uint8_t)kind;
      sh.ptn[s] = pn;
      sh.cn[s] = cb;
    }
  }
  step(13);
  __syncwarp();
}

// ------------------------------------------------------------- walk
// Moves in order tracking the N offset d; stops at a move whose d is outside
// the evaluated range, at an accepted move whose commit would overflow, or
// after max_acc accepts. Two ballots per 64 moves plus two per event (one
// warp; the others wait at the barrier after it).
__device__ __forceinline__ void walk(const SmArgs& a, const SmShared& sh, WalkRes& W, int fit, int lane) {
  int d = 0, start = 0, nacc = 0, len = fit, err = 0, why = kSEnd;
  const int i0 = lane, i1 = lane + 32;
  const bool in0 = i0 < fit, in1 = i1 < fit;
  const uint32_t am0 = in0 ? sh.macc[i0] : 0u, om0 = in0 ? sh.movf[i0] : 0u;
  const uint32_t am1 = in1 ? sh.macc[i1] : 0u, om1 = in1 ? sh.movf[i1] : 0u;
  const unsigned kd0 = in0 ? sh.mkind[i0] : 0u, kd1 = in1 ? sh.mkind[i1] : 0u;
  int d0 = 0, d1 = 0;  // the N offset before slots i0 / i1
#pragma unroll 1
  for (;;) {
    const int j = d + kSHalf;
    const bool inr = j >= 0 && j < kSOff;
    const int jj = j & (kSOff - 1);
    const bool act0 = in0 && i0 >= start, act1 = in1 && i1 >= start;
    if (act0) d0 = d;
    if (act1) d1 = d;
    const bool st0 = act0 && !inr, ac0 = act0 && inr && ((am0 >> jj) & 1u);
    const bool st1 = act1 && !inr, ac1 = act1 && inr && ((am1 >> jj) & 1u);
    const unsigned ev0 = __ballot_sync(0xffffffffu, st0 || ac0);
    const unsigned ev1 = __ballot_sync(0xffffffffu, st1 || ac1);
    if (!(ev0 | ev1)) break;
    const bool first = ev0 != 0u;
    const int el = __ffs(first ? ev0 : ev1) - 1;
    const int e = (first ? 0 : 32) + el;
    const unsigned mine = first ? ((st0 ? 1u : 0u) | (((om0 >> jj) & 1u) << 1) | (kd0 << 2))
                                : ((st1 ? 1u : 0u) | (((om1 >> jj) & 1u) << 1) | (kd1 << 2));
    const unsigned info = __shfl_sync(0xffffffffu, mine, el);
    if (info & 1u) {
      len = e;
      why = kSRange;
      break;
    }
    if (info & 2u) {
      len = e;
      err = 1;
      why = kSOverflow;
      break;
    }
    if (lane == 0) {
      W.acc_i[nacc] = e;
      W.acc_d[nacc] = d;
    }
    ++nacc;
    const int k = (int)(info >> 2);
    d += k == 1 ? 1 : (k == 2 ? -1 : 0);
    start = e + 1;
    if (nacc == a.max_acc) {
      len = e + 1;
      why = kSFull;
      break;
    }
  }
  // slots after the last event carry the final d
  if (in0 && i0 >= start) d0 = d;
  if (in1 && i1 >= start) d1 = d;
  if (in0) W.d[i0] = (int8_t)d0;
  if (in1) W.d[i1] = (int8_t)d1;
  if (lane == 0) {
    W.len = len;
    W.nacc = nacc;
    W.err = err;
    W.why = why;
  }
  __syncwarp();
}

// ------------------------------------------------------------- verify
// A consumed slot's read / write set at its decided N offset.
struct RW {
  int kind;
  int32_t ia, ib;   // particle read/written (insert: the new index), last index (delete)
  uint32_t pn, po;  // brick points: new position, the particle's position
  int32_t cn, co;   // reference cells of the same
  double nx, ny, nz, ox, oy, oz;
};
__device__ __forceinline__ RW rw_of(const SmArgs& a, const SmShared& sh, uint64_t base, uint64_t n, int i,
                                    int d) {
  const Proposal& pr = sh.ring[(base + (uint64_t)i) % kSRing];
  RW r;
  r.kind = sh.mkind[i];
  r.pn = sh.ptn[i];
  r.cn = sh.cn[i];
  r.nx = pr.x;
  r.ny = pr.y;
  r.nz = pr.z;
  const int o = d + kSHalf;
  const int64_t nd = (int64_t)n + d;
  r.ia = sh.off_ia[i][o];
  r.ib = r.kind == 2 && nd >= 1 ? (int32_t)(nd - 1) : -1;
  r.po = sh.off_po[i][o];
  r.co = sh.off_co[i][o];
  r.ox = sh.off_x[i][o][0];
  r.oy = sh.off_x[i][o][1];
  r.oz = sh.off_x[i][o][2];
  return r;
}

__device__ __forceinline__ bool near_rc(const Box& b, double ax, double ay, double az, double bx,
                                        double by, double bz, double lim) {
  return min_image_dist2(ax, ay, az, bx, by, bz, b) <= lim;
}

// Does consumed slot i read anything accepted slot j (< i) changed, or (i
// accepted) lie within 2 r_c of it? Brick filters first, then distances with
// a margin (conservative: a false conflict only ends the round early).
__device__ __forceinline__ bool conflicts(const SmArgs& a, const RW& I, const RW& J, bool i_acc) {
  const bool grid = grid_on(a);
  if (I.kind != 1 && I.ia >= 0 && (I.ia == J.ia || I.ia == J.ib)) return true;
  const uint32_t ln = I.pn, lo = I.po, an = J.pn, ao = J.po;
  const uint32_t kNP = (uint32_t)kNoPoint;
  if (ln != kNP) {  // i's target brick / cell (its overflow test read their occupancies)
    const uint32_t lb = mbrick(a.m, ln);
    if (ao != kNP && (lb == mbrick(a.m, ao) || (grid && I.cn == J.co))) return true;
    if (an != kNP && (lb == mbrick(a.m, an) || (grid && I.cn == J.cn))) return true;
  }
  // the particles' positions are single-precision copies here: every
  // distance gets a margin of 4e-7 L (two roundings of <= 6e-8 L per axis)
  const double eps = 4e-7 * a.b.l;
  const double lim1 = (a.b.rc + eps) * (a.b.rc + eps);
  if (ln != kNP) {
    if (ao != kNP && mnear(a.m, ln, ao) && near_rc(a.b, I.nx, I.ny, I.nz, J.ox, J.oy, J.oz, lim1)) return true;
    if (an != kNP && mnear(a.m, ln, an) && near_rc(a.b, I.nx, I.ny, I.nz, J.nx, J.ny, J.nz, lim1)) return true;
  }
  if (lo != kNP) {
    if (ao != kNP && mnear(a.m, lo, ao) && near_rc(a.b, I.ox, I.oy, I.oz, J.ox, J.oy, J.oz, lim1)) return true;
    if (an != kNP && mnear(a.m, lo, an) && near_rc(a.b, I.ox, I.oy, I.oz, J.nx, J.ny, J.nz, lim1)) return true;
  }
  if (i_acc) {  // two accepted moves: every changed point more than 2 r_c apart
    const double lim2 = (2.0 * a.b.rc + eps) * (2.0 * a.b.rc + eps);
    const int dm = a.m.dims;
    auto far = [&](uint32_t p, double px, double py, double pz, uint32_t q, double qx, double qy, double qz) {
      if (p == kNP || q == kNP) return true;
      const int dx = abs(pt_x(p) - pt_x(q)), dy = abs(pt_y(p) - pt_y(q)), dz = abs(pt_z(p) - pt_z(q));
      const bool bnear = min(dx, dm - dx) <= 2 && min(dy, dm - dy) <= 2 && min(dz, dm - dz) <= 2;
      return !(bnear && near_rc(a.b, px, py, pz, qx, qy, qz, lim2));
    };
    if (!far(ln, I.nx, I.ny, I.nz, an, J.nx, J.ny, J.nz) || !far(ln, I.nx, I.ny, I.nz, ao, J.ox, J.oy, J.oz) ||
        !far(lo, I.ox, I.oy, I.oz, an, J.nx, J.ny, J.nz) || !far(lo, I.ox, I.oy, I.oz, ao, J.ox, J.oy, J.oz))
      return true;
  }
  return false;
}

// This warp's slots (warp + kSW q) against every earlier accepted move:
// lane = (slot q, accepted k) pairs.
__device__ __forceinline__ void verify(const SmArgs& a, SmShared& sh, const WalkRes& W, uint64_t base,
                                       uint64_t n, int warp, int lane) {
  const int len = W.len, nacc = W.nacc;
  for (int p = lane; p < (kSM / kSW) * kSAcc; p += 32) {
    const int q = p / kSAcc, k = p % kSAcc;
    const int i = warp + kSW * q;
    if (i >= len || k >= nacc) continue;
    const int j = W.acc_i[k];
    if (j >= i) continue;
    const int di = W.d[i];
    const RW I = rw_of(a, sh, base, n, i, di);
    const RW J = rw_of(a, sh, base, n, j, W.acc_d[k]);
    const bool i_acc = (sh.macc[i] >> (di + kSHalf)) & 1u;
    if (conflicts(a, I, J, i_acc)) atomicMin(&sh.cmin, i);
  }
}

// ------------------------------------------------------------- commits
// One warp: the pruned 3x3x3 brick window of (x, y, z) appended at entry `at`
// of ws (bricks and image codes; wmask / bpt: the proposal's precomputed
// window, kNoMask: compute it). Returns the number of entries added.
__device__ __forceinline__ int warp_window(const SmArgs& a, SWs& ws, int at, double x, double y, double z,
                                          uint32_t wmask, uint32_t bpt, int lane) {
  const Mirror& m = a.m;
  if (m.dims < 3) {
    if (lane < (int)m.nb) {
      ws.brick[at + lane] = (uint32_t)lane;
      ws.sc[at + lane] = 0;
    }
    return (int)m.nb;
  }
  if (wmask == kNoMask) {
    bpt = (uint32_t)mpoint(m, x, y, z);
    uint32_t id;
    const bool keep = lane < 27 && window_keep(m, a.b, x, y, z, pt_x(bpt), pt_y(bpt), pt_z(bpt), lane, id);
    wmask = __ballot_sync(0xffffffffu, keep);
  }
  if (lane < 27 && ((wmask >> lane) & 1u)) {
    const int d = m.dims;
    int cx = pt_x(bpt) + lane % 3 - 1, cy = pt_y(bpt) + (lane / 3) % 3 - 1, cz = pt_z(bpt) + lane / 9 - 1;
    cx += cx < 0 ? d : 0;
    cx -= cx >= d ? d : 0;
    cy += cy < 0 ? d : 0;
    cy -= cy >= d ? d : 0;
    cz += cz < 0 ? d : 0;
    cz -= cz >= d ? d : 0;
    const int e = at + __popc(wmask & ((1u << lane) - 1u));
    ws.brick[e] = (uint32_t)cx + (uint32_t)d * ((uint32_t)cy + (uint32_t)d * (uint32_t)cz);
    ws.sc[e] = image_code(pt_x(bpt), pt_y(bpt), pt_z(bpt), lane, d);
  }
  return __popc(wmask);
}

// Neighbour energy updates of accepted move k (one warp): e_j -= pair(old,
// x_j) for the neighbours of the old position, then e_j += pair(new, x_j) for
// those of the new one, found on the state before the round's commits (the
// mover's own record excluded: the one at its old position).
template <bool kImg>
__device__ __noinline__ void energy_updates(const SmArgs& a, SmShared& sh, const uint8_t* occ_s,
                                            uint64_t base, int k, int warp, int lane) {
  unsigned long long tq = clock64();
  auto step = [&](int q) {
#ifdef GCMC_SM_STEPS
    const unsigned long long t = clock64();
    if (lane == 0) atomicMax(&sh.rmax[q], t - tq);
    tq = t;
#else
    (void)q;
#endif
  };
  SWs& ws = sh.ws[warp][0];
  auto& S = sh.stash[warp];
  const WalkRes& W = sh.wr[0];
  const int i = W.acc_i[k];
  const int kind = sh.mkind[i];
  const Proposal& pr = sh.ring[(base + (uint64_t)i) % kSRing];
  double ox = 0.0, oy = 0.0, oz = 0.0;
  if (kind != 1) {  // the mover's exact position (loaded during the verify)
    ox = sh.xacc[k].x;
    oy = sh.xacc[k].y;
    oz = sh.xacc[k].z;
  }
  // window 0: old position (-), window 1: new position (+)
  int nent = 0;
  if (kind != 1) nent = warp_window(a, ws, 0, ox, oy, oz, kNoMask, 0u, lane);
  const int nent0 = nent;
  if (kind != 2) nent += warp_window(a, ws, nent, pr.x, pr.y, pr.z, pr.wmask, pr.bpt, lane);
  step(9);
  win_finish_s(a.m, ws, occ_s, nent, nent0, lane);
  __syncwarp();
  step(10);
  const int total = ws.total;
  if (lane == 0) atomicAdd(&sh.pairs, (unsigned long long)total);
  int nst = 0;  // stash entries (warp-uniform)
#pragma unroll 1
  for (int b0 = 0; b0 < total; b0 += 128) {
    double rx[4], ry[4], rz[4];
    int32_t rid[4];
    bool ok[4], w1[4];
    int ent[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int f = b0 + 32 * u + lane;
      ok[u] = f < total;
      w1[u] = false;
      rx[u] = ry[u] = rz[u] = 0.0;
      rid[u] = -1;
      ent[u] = 0;
      if (ok[u]) {
        int e;
        const int idx = cand_record(a.m, ws, f, &e);
        ent[u] = e;
        w1[u] = e >= nent0;
        rx[u] = __ldcg(a.m.rx + idx);
        ry[u] = __ldcg(a.m.ry + idx);
        rz[u] = __ldcg(a.m.rz + idx);
        rid[u] = __ldcg(a.m.rid + idx);
      }
    }
    // branch-free pair chains (interleaved), then the updates
    bool hits[4];
    double pus[4], pws[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const double cx = w1[u] ? pr.x : ox, cy = w1[u] ? pr.y : oy, cz = w1[u] ? pr.z : oz;
      const double r2 = kImg ? image_dist2(cx, cy, cz, rx[u], ry[u], rz[u], ws.sc[ent[u]], a.b.l)
                             : min_image_dist2(cx, cy, cz, rx[u], ry[u], rz[u], a.b);
      const bool mover = kind != 1 && rx[u] == ox && ry[u] == oy && rz[u] == oz;  // its own record
      hits[u] = ok[u] && !mover && r2 <= a.b.rc2;
      lj_pair_clamped(hits[u] ? r2 : a.b.rc2, a.b, pus[u], pws[u]);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const bool hit = hits[u];
      const double pu = pus[u], pw = pws[u];
      if (hit && !w1[u]) {  // old window: now
        atomicAdd(&a.ep[rid[u]].x, -pu);
        atomicAdd(&a.ep[rid[u]].y, -pw);
      }
      const bool later = hit && w1[u];
      const unsigned lm = __ballot_sync(0xffffffffu, later);
      if (later) {
        const int q = nst + __popc(lm & ((1u << lane) - 1u));
        if (q < kStash) {  // (beyond: the new window is re-scanned below)
          S.id[q] = rid[u];
          S.u[q] = pu;
          S.w[q] = pw;
        }
      }
      nst += __popc(lm);
    }
  }
  step(11);
  __syncwarp();  // the old-window updates happen-before the new-window ones
  if (nst <= kStash) {
    for (int q = lane; q < nst; q += 32) {
      atomicAdd(&a.ep[S.id[q]].x, S.u[q]);
      atomicAdd(&a.ep[S.id[q]].y, S.w[q]);
    }
    step(12);
  } else {  // rare (a very dense window): the new window again, applied directly
#pragma unroll 1
    for (int f = lane; f < total; f += 32) {
      int e;
      const int idx = cand_record(a.m, ws, f, &e);
      if (e < nent0) continue;
      const double rx = __ldcg(a.m.rx + idx), ry = __ldcg(a.m.ry + idx), rz = __ldcg(a.m.rz + idx);
      if (kind != 1 && rx == ox && ry == oy && rz == oz) continue;
      const double r2 = cand_dist2(a.m, a.b, ws, e, pr.x, pr.y, pr.z, rx, ry, rz);
      if (r2 <= a.b.rc2) {
        double pu, pw;
        lj_pair_clamped(r2, a.b, pu, pw);
        const int32_t id = __ldcg(a.m.rid + idx);
        atomicAdd(&a.ep[id].x, pu);
        atomicAdd(&a.ep[id].y, pw);
      }
    }
  }
}

// The mover of accepted move k: kind, pid (displace / delete), store size
// before the move.
__device__ __forceinline__ void mover_of(const SmShared& sh, uint64_t base, uint64_t n, int k, int& i,
                                         int& kind, uint64_t& pid, uint64_t& nn) {
  const WalkRes& W = sh.wr[0];
  i = W.acc_i[k];
  kind = sh.mkind[i];
  nn = (uint64_t)((int64_t)n + W.acc_d[k]);
  pid = kind == 1 ? 0 : index_from(sh.ring[(base + (uint64_t)i) % kSRing].pick, nn);
}

// Structural commit loads (lane k = accepted move k) and their order
// (engine2.cu:commit_round's rules): a commit that touches an earlier one of
// the round (cell, brick or particle) is re-loaded and applied after it; an
// insertion that reuses the index an earlier deletion vacated is exempt
// unless that deletion is itself ordered (its loads then follow the
// insertion's stores). A deletion whose relabel source q = n - 1 is the
// particle an earlier insertion of the round created takes q's data
// (position, reference slot, record) from the insertion's lane instead of
// waiting for its stores, and is stored after it; that insertion then need
// not write index n at all (the deletion moves it to pid).
__device__ __noinline__ void commit_loads(const SmArgs& a, SmShared& sh, uint64_t base, uint64_t n,
                                          int nacc, int lane) {
  unsigned long long tq = clock64();
  auto step = [&](int k) {
#ifdef GCMC_SM_CL_STEPS
    const unsigned long long t = clock64();
    if (lane == 0) atomicMax(&sh.rmax[k], t - tq);
    tq = t;
#else
    (void)k;
#endif
  };
  const bool mine = lane < nacc;
  int kind = 0, i = 0;
  uint64_t pid = 0, nn = 0;
  Touch tc{};
  MoveData md{};
  CommitIn c{};
  if (mine) {
    mover_of(sh, base, n, lane, i, kind, pid, nn);
    const Proposal& pr = sh.ring[(base + (uint64_t)i) % kSRing];
    md.nx = pr.x;
    md.ny = pr.y;
    md.nz = pr.z;
    md.rslot_pid = md.bslot_pid = -1;
    if (kind != 1) {  // load_move's fields, loaded during the verify
      const double4 o = sh.xacc[lane];
      md.ox = o.x;
      md.oy = o.y;
      md.oz = o.z;
      md.rslot_pid = sh.rsacc[lane];
      md.bslot_pid = bslot_in(o);
    }
    commit_load(a.g, a.m, a.s, kind, pid, nn, md, c);
    tc = touch_of(a.m, kind, pid, nn, c);
  }
  __syncwarp();
  step(9);
  // forwarding
  int fsrc = -1;
  {
    const int64_t myq = (mine && kind == 2 && pid != nn - 1) ? (int64_t)(nn - 1) : -2;
#pragma unroll 1
    for (int j = 0; j < nacc - 1; ++j) {
      const int kj = __shfl_sync(0xffffffffu, kind, j);
      const uint64_t nnj = __shfl_sync(0xffffffffu, nn, j);
      if (j < lane && kj == 1 && (int64_t)nnj == myq) fsrc = j;
    }
    const int f = fsrc >= 0 ? fsrc : lane;
    const double fx = __shfl_sync(0xffffffffu, md.nx, f), fy = __shfl_sync(0xffffffffu, md.ny, f),
                 fz = __shfl_sync(0xffffffffu, md.nz, f);
    const int focb = __shfl_sync(0xffffffffu, c.occ_cb, f), fcb = __shfl_sync(0xffffffffu, c.cb, f);
    const int fbb = __shfl_sync(0xffffffffu, c.bb, f), fobb = __shfl_sync(0xffffffffu, c.occ_bb, f);
    if (fsrc >= 0) {
      c.qx = fx;
      c.qy = fy;
      c.qz = fz;
      c.rslot_q = focb;
      c.bslot_q = fbb * a.m.cap + fobb;
      c.cl = fcb;
      tc = touch_of(a.m, kind, pid, nn, c);
    }
  }
  step(10);
  if (mine) sh.cfwd[lane] = (int8_t)fsrc;
  const unsigned fwd_src = __reduce_or_sync(0xffffffffu, (mine && fsrc >= 0) ? (1u << fsrc) : 0u);
  const bool away = mine && kind == 1 && ((fwd_src >> lane) & 1u);
  const int chain = (fsrc >= 0 ? 1 : 0) | (away ? 2 : 0);
  // every (later k, earlier j) pair of the round's commits in parallel over
  // the lanes, Touches from shared memory
  auto order = [&](bool chain_form, bool& dep) {
    Touch tme = tc;
    if (chain_form && (chain & 1)) tme.part[1] = -1;
    if (chain_form && (chain & 2)) tme.part[0] = -1;
    if (mine) {
      sh.ctouch[lane] = tme;
      sh.cexm[lane] = 0u;
      sh.ckind[lane] = (int8_t)kind;
    }
    if (lane == 0) sh.cdepm = 0u;
    __syncwarp();
    const int npairs = nacc * (nacc - 1) / 2;
    for (int p = lane; p < npairs; p += 32) {
      int kk = (int)((1.0f + sqrtf(1.0f + 8.0f * (float)p)) * 0.5f);  // p = kk (kk - 1) / 2 + j
      while (kk * (kk - 1) / 2 > p) --kk;
      while ((kk + 1) * kk / 2 <= p) ++kk;
      const int j = p - kk * (kk - 1) / 2;
      Touch tm = sh.ctouch[kk];
      const Touch tj = sh.ctouch[j];
      if (sh.ckind[kk] == 1 && sh.ckind[j] == 2 && tm.part[0] >= 0 && tm.part[0] == tj.part[1]) {
        tm.part[0] = -1;
        atomicOr(&sh.cexm[kk], 1u << j);
      }
      if (j == sh.cfwd[kk]) {  // the forwarded particle's index, cell and record are expected
        tm.part[1] = -1;
        tm.cell[2] = -1;
        tm.brick[2] = -1;
      }
      if (touches(tm, tj)) atomicOr(&sh.cdepm, 1u << kk);
    }
    __syncwarp();
    dep = mine && ((sh.cdepm >> lane) & 1u);
    const unsigned exm = mine ? sh.cexm[lane] : 0u;
    // an exempted / forwarded commit is ordered after its partner when the
    // partner itself is (it then loads or stores late)
#pragma unroll 1
    for (int it = 0; it < 32; ++it) {
      const unsigned b = __ballot_sync(0xffffffffu, dep);
      const bool nd = dep || (b & exm) || (fsrc >= 0 && ((b >> fsrc) & 1u));
      if (__ballot_sync(0xffffffffu, nd) == b) break;
      dep = nd;
    }
    __syncwarp();
  };
  bool dep = false;
  order(true, dep);
  step(11);
  const bool chains_free = !__any_sync(0xffffffffu, chain != 0 && dep);
  if (!chains_free) order(false, dep);  // full ordering (rare)
  step(12);
  const unsigned deps = __ballot_sync(0xffffffffu, dep);
  if (mine) {
    sh.md[lane] = md;
    sh.cin[lane] = c;
    sh.cskip[lane] = (uint8_t)(chains_free && away);
  }
  if (lane == 0) sh.cdep = deps;
  if (a.diag && lane == 0) {  // diagnostics: ordered commits and commits per round
    sh.racc[14] += __popc(deps);
    sh.racc[15] += nacc;
  }
  __syncwarp();
  step(13);
}

__device__ __noinline__ void commit_stores(const SmArgs& a, SmShared& sh, uint64_t base, uint64_t n,
                                           int nacc, int lane) {
  const bool mine = lane < nacc;
  const unsigned deps = sh.cdep;
  int kind = 0, i = 0;
  uint64_t pid = 0, nn = 0;
  if (mine) mover_of(sh, base, n, lane, i, kind, pid, nn);
  long long e1, e2, e3;
  const bool free_ = mine && !((deps >> lane) & 1u);
  const bool fwd = mine && sh.cfwd[lane] >= 0;
  if (free_ && !fwd)
    commit_store(a.g, a.m, a.s, &a.st->peak, kind, pid, nn, sh.md[lane], sh.cin[lane], e1, e2, e3,
                 sh.cskip[lane] != 0);
  __syncwarp();  // forwarded deletions after their insertions
  if (free_ && fwd)
    commit_store(a.g, a.m, a.s, &a.st->peak, kind, pid, nn, sh.md[lane], sh.cin[lane], e1, e2, e3);
  if (deps) {
    __syncwarp();
#pragma unroll 1
    for (int j = 0; j < nacc; ++j) {
      if (((deps >> j) & 1u) && lane == j) {
        MoveData md = sh.md[lane];
        load_move(a.s, kind, pid, md);
        commit_move(a.g, a.m, a.s, &a.st->peak, kind, pid, nn, md, e1, e2, e3);
      }
      __syncwarp();
    }
  }
  // the movers' e, in move order (displace: pid, insert: its new index,
  // delete: pid <- e[q], q = n - 1, the latest earlier write to q or memory,
  // which already carries the round's neighbour updates)
  const bool copies = mine && kind == 2 && pid != nn - 1;
  const int64_t ex = !mine ? -1 : (kind == 1 ? (int64_t)nn : (kind == 0 || copies ? (int64_t)pid : -1));
  const int64_t eq = copies ? (int64_t)(nn - 1) : -2;
  double esu = 0.0, esw = 0.0;
  if (mine && kind != 2) {
    const int dk = sh.wr[0].acc_d[lane] + kSHalf;
    esu = sh.off_mu[i][dk];
    esw = sh.off_mw[i][dk];
  }
  if (copies) {
    const double2 el = __ldcg(a.ep + (nn - 1));
    esu = el.x;
    esw = el.y;
  }
#pragma unroll 1
  for (int j = 0; j < nacc - 1; ++j) {
    const int64_t xj = __shfl_sync(0xffffffffu, ex, j);
    const double vu = __shfl_sync(0xffffffffu, esu, j), vw = __shfl_sync(0xffffffffu, esw, j);
    if (lane > j && xj == eq) {
      esu = vu;
      esw = vw;
    }
  }
#pragma unroll 1
  for (int j = 0; j < nacc; ++j) {
    if (lane == j && ex >= 0) __stcg(a.ep + ex, make_double2(esu, esw));
    __syncwarp();
  }
}

// ------------------------------------------------------------- statistics
// reported_energy() and pressure() (engine.hpp:277-291) with the tail terms
// of tail_corrections() (potential.hpp:63-72), same operation order.
__device__ __forceinline__ void observe(const SmArgs& a, uint64_t n, double u, double w, double& ru,
                                        double& p) {
  const double rho = __ddiv_rn((double)n, a.vol);
  p = __dadd_rn(__dmul_rn(rho, a.temp), __ddiv_rn(w, __dmul_rn(3.0, a.vol)));
  ru = u;
  if (a.tail) {
    const double tu = __dmul_rn(
        __dmul_rn(__dmul_rn(__dmul_rn(a.tail_cu, rho), a.b.eps), a.tail_s3), a.tail_bu);
    const double tp = __dmul_rn(
        __dmul_rn(__dmul_rn(__dmul_rn(__dmul_rn(a.tail_cp, rho), rho), a.b.eps), a.tail_s3),
        a.tail_bp);
    p = __dadd_rn(p, tp);
    ru = __dadd_rn(ru, __dmul_rn((double)n, tu));
  }
}

// Counters, U / W in move order, samples (engine.hpp:293-308, 413-426) and
// the trace records (MoveOutcome, engine.hpp:104-110) of the decided round.
__device__ __noinline__ void statistics(const SmArgs& a, SmShared& sh, uint64_t base, uint64_t n, int len,
                                        int nacc, int lane) {
  const WalkRes& W = sh.wr[0];
  ChainState& ks = sh.ks;
  if (lane == 0) {
    double energy = ks.energy, virial = ks.virial;
    uint64_t cur = n;
    sh.st_e[0] = energy;
    sh.st_w[0] = virial;
    sh.st_n[0] = cur;
    for (int k = 0; k < nacc; ++k) {
      const int i = W.acc_i[k], dk = W.acc_d[k] + kSHalf;
      energy = __dadd_rn(energy, sh.off_du[i][dk]);
      virial = __dadd_rn(virial, sh.off_dw[i][dk]);
      const int kind = sh.mkind[i];
      ++ks.accepted[kind];
      cur = kind == 1 ? cur + 1 : (kind == 2 ? cur - 1 : cur);
      sh.st_e[k + 1] = energy;
      sh.st_w[k + 1] = virial;
      sh.st_n[k + 1] = cur;
    }
    ks.energy = energy;
    ks.virial = virial;
  }
  __syncwarp();
  for (int k = lane; k <= nacc; k += 32) {
    const uint64_t cur = sh.st_n[k];
    double ru, p;
    observe(a, cur, sh.st_e[k], sh.st_w[k], ru, p);
    const double nd = (double)cur;
    sh.st_v[k][0] = nd;
    sh.st_v[k][1] = __dmul_rn(nd, nd);
    sh.st_v[k][2] = ru;
    sh.st_v[k][3] = p;
  }
  const uint64_t step0 = ks.step;
  unsigned att0 = 0, att1 = 0, att2 = 0;
#pragma unroll
  for (int h = 0; h < kSM / 32; ++h) {
    const int i = lane + 32 * h;
    const bool in = i < len;
    const int kind = in ? sh.mkind[i] : 3;
    att0 += __popc(__ballot_sync(0xffffffffu, kind == 0));
    att1 += __popc(__ballot_sync(0xffffffffu, kind == 1));
    att2 += __popc(__ballot_sync(0xffffffffu, kind == 2));
    const uint64_t st = step0 + (uint64_t)i + 1;
    const bool smp = in && st > a.equil && (a.interval == 1 || (st - a.equil) % a.interval == 0);
    const unsigned b = __ballot_sync(0xffffffffu, smp);
    if (lane == 0) sh.smp[h] = b;
  }
  __syncwarp();
  if (lane == 0) {
    double sn = ks.sum_n, sn2 = ks.sum_n2, su = ks.sum_u, sp = ks.sum_p;
    uint64_t samples = 0;
    int lo = 0;
    for (int k = 0; k <= nacc; ++k) {
      const int hi = k < nacc ? W.acc_i[k] : len;
      int c = 0;
#pragma unroll
      for (int h = 0; h < kSM / 32; ++h) {
        const int a0 = lo - 32 * h, a1 = hi - 32 * h;
        const unsigned m_hi = a1 >= 32 ? 0xffffffffu : (a1 <= 0 ? 0u : (1u << a1) - 1u);
        const unsigned m_lo = a0 >= 32 ? 0xffffffffu : (a0 <= 0 ? 0u : (1u << a0) - 1u);
        c += __popc(sh.smp[h] & m_hi & ~m_lo);
      }
      const double v0 = sh.st_v[k][0], v1 = sh.st_v[k][1], v2 = sh.st_v[k][2], v3 = sh.st_v[k][3];
      for (int j = 0; j < c; ++j) {
        sn = __dadd_rn(sn, v0);
        sn2 = __dadd_rn(sn2, v1);
        su = __dadd_rn(su, v2);
        sp = __dadd_rn(sp, v3);
      }
      samples += (uint64_t)c;
      lo = hi;
    }
    ks.attempted[0] += att0;
    ks.attempted[1] += att1;
    ks.attempted[2] += att2;
    ks.step = step0 + (uint64_t)len;
    ks.samples += samples;
    ks.sum_n = sn;
    ks.sum_n2 = sn2;
    ks.sum_u = su;
    ks.sum_p = sp;
  }
  if (a.trace) {
    for (int i = lane; i < len; i += 32) {
      const int dk = W.d[i] + kSHalf;
      int dn = 0, acc = 0;
      for (int k = 0; k < nacc; ++k) {
        const int ak = sh.mkind[W.acc_i[k]];
        if (W.acc_i[k] <= i) dn += ak == 1 ? 1 : (ak == 2 ? -1 : 0);
        if (W.acc_i[k] == i) acc = 1;
      }
      gcmc_trace_rec t;
      t.kind = sh.mkind[i];
      t.accepted = acc;
      t.delta_u = sh.off_du[i][dk];
      t.delta_w = sh.off_dw[i][dk];
      {  // recomputed: the same operations as the evaluation's
        const int kind = sh.mkind[i];
        const int64_t nd = (int64_t)n + W.d[i];
        const bool valid = kind == 1 ? nd >= 0 : nd >= 1;
        t.acceptance_prob = valid ? accept_prob(a, kind, sh.off_du[i][dk], exchange_prefactor(a, kind, nd)) : 0.0;
      }
      t.n_after = (uint64_t)((int64_t)n + dn);
      a.trace[base + (uint64_t)i] = t;
    }
  }
  __syncwarp();
}

// Proposals [lo, hi) into the ring (plain loads: the array is read-only for
// the kernel's lifetime; one warp).
__device__ __forceinline__ void ring_load(const SmArgs& a, Proposal* ring, uint64_t lo, uint64_t hi, int lane) {
  constexpr unsigned W = sizeof(Proposal) / 8;
  const unsigned cnt = (unsigned)(hi - lo) * W;
  for (unsigned k0 = 0; k0 < cnt; k0 += 32 * 8) {
    uint64_t v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const unsigned k = k0 + 32 * u + lane;
      v[u] = k < cnt ? __ldg(reinterpret_cast<const unsigned long long*>(a.props + lo + k / W) + k % W) : 0ull;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const unsigned k = k0 + 32 * u + lane;
      if (k < cnt) reinterpret_cast<uint64_t*>(&ring[(lo + k / W) % kSRing])[k % W] = v[u];
    }
  }
}

// ------------------------------------------------------------- the kernel
// One CTA per chain: the chain's arguments by value (one chain) or from a
// device list indexed by blockIdx.x (K chains in one launch).
template <bool kMulti>
__global__ void __launch_bounds__(kST, kST <= 256 ? 2 : 1) k_engine_sm(SmArgs args, const SmArgs* __restrict__ list) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ SmArgs a;
  auto& sh = *reinterpret_cast<SmShared*>(smem);
  uint8_t* occ_s = nullptr;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) a = kMulti ? list[blockIdx.x] : args;
  __syncthreads();
  if (a.smem_occ) {
    occ_s = smem + ((sizeof(SmShared) + 15) & ~size_t(15));
    for (uint32_t b = tid; b < a.m.nb; b += kST) occ_s[b] = (uint8_t)__ldcg(a.m.occ + b);
  }
  if (tid == 0) {
    sh.ks = *a.st;
    sh.pairs = 0;
    for (int k = 0; k < 6; ++k) sh.stops[k] = 0;
    for (int k = 0; k < 16; ++k) sh.rmax[k] = sh.racc[k] = 0;
    sh.base = 0;
    sh.n = a.st->n;
    sh.cmin = kSM;
  }
  uint64_t ring_hi = a.nmoves < (uint64_t)kSAhead ? a.nmoves : (uint64_t)kSAhead;  // (warp kXW)
  if (warp == kXW) ring_load(a, sh.ring, 0, ring_hi, lane);
  uint64_t rounds = 0;
  // per-phase cycles of thread 0 (between the round's barriers), reported in
  // ChainState::pad[0..4] for the diagnostics of engine_sm_run
  unsigned long long ph[5] = {0, 0, 0, 0, 0}, t0 = clock64();
  auto mark = [&](int k) {
    if (tid == 0) {
      const unsigned long long t = clock64();
      ph[k] += t - t0;
      t0 = t;
    }
  };
  bool stop = false;
  // role timers (diagnostics): lane 0 of each warp, max over warps per round
  const bool dg = a.diag != nullptr;
  unsigned long long rt0 = 0;
  auto role_start = [&]() {
    if (dg) rt0 = clock64();
  };
  auto role_end = [&](int k) {
    if (dg && lane == 0) atomicMax(&sh.rmax[k], clock64() - rt0);
    if (dg) rt0 = clock64();
  };
  for (;;) {
    __syncthreads();
    if (dg && tid == 0)
      for (int k = 0; k < 16; ++k) {
        sh.racc[k] += sh.rmax[k];
        sh.rmax[k] = 0;
      }
    const uint64_t base = sh.base, n = sh.n;
    const int fit = base >= a.nmoves ? 0 : (a.nmoves - base < (uint64_t)kSM ? (int)(a.nmoves - base) : kSM);
    if (fit == 0 || stop) break;
    mark(0);
    // ---- evaluate (two slots per call: half-warps)
    role_start();
#pragma unroll 1
    for (int s0 = warp; s0 < kSM; s0 += 2 * kSW) eval_pair(a, sh, occ_s, s0, fit, base, n, warp, lane);
    role_end(0);
    __syncthreads();
    mark(1);
    // ---- walk (every warp) and verify (this warp's slots)
    WalkRes& W = sh.wr[0];
    role_start();
    if (warp == 0) walk(a, sh, W, fit, lane);
    role_end(1);
    __syncthreads();
    if (warp == kXW && lane < W.nacc) {  // the accepted movers' records, ahead of the commits
      const int i = W.acc_i[lane];
      if (sh.mkind[i] != 1) {
        const int32_t pid = sh.off_ia[i][W.acc_d[lane] + kSHalf];
        sh.xacc[lane] = ld_cg(a.s.pos + pid);
        sh.rsacc[lane] = __ldcg(a.s.rslot + pid);
      }
    }
    verify(a, sh, W, base, n, warp, lane);
    role_end(2);
    __syncthreads();
    mark(2);
    const RoundOut ro = round_out(sh);
    const int len = ro.len, nacc = ro.nacc;
    // ---- commits, part 1: neighbour energy updates, structural loads; the
    // ring's next proposals and the statistics
    role_start();
    if (warp < kEW) {
      for (int k = warp; k < nacc; k += kEW) {
        if (a.m.dims >= 5)
          energy_updates<true>(a, sh, occ_s, base, k, warp, lane);
        else
          energy_updates<false>(a, sh, occ_s, base, k, warp, lane);
      }
      role_end(3);
    } else if (warp == kCW) {
      commit_loads(a, sh, base, n, nacc, lane);
      role_end(4);
    } else {
      const uint64_t nbase = base + (uint64_t)len;
      const uint64_t want = nbase + kSAhead < a.nmoves ? nbase + kSAhead : a.nmoves;
      if (want > ring_hi) {  // (entries of moves < base - kSM: none of this round's)
        ring_load(a, sh.ring, ring_hi, want, lane);
        ring_hi = want;
      }
      role_end(5);
      statistics(a, sh, base, n, len, nacc, lane);
      role_end(6);
      if (lane == 0) {
        ++sh.stops[sh.cmin < sh.wr[0].len ? (int)kSVerify : sh.wr[0].why];
      }
    }
    __syncthreads();  // the round's e updates and every mirror read happen-before the stores
    mark(3);
    // ---- commits, part 2: structural stores, the movers' e, the replica
    role_start();
    if (warp == kCW) {
      commit_stores(a, sh, base, n, nacc, lane);
      role_end(7);
    } else if (warp == kXW) {
      if (occ_s && lane < nacc) {  // replica = the mirror's occupancies after the round
        uint32_t* occ_w = reinterpret_cast<uint32_t*>(occ_s);
        const CommitIn& c = sh.cin[lane];
        const int kind = sh.mkind[sh.wr[0].acc_i[lane]];
        if (c.mir_move) atomicSub(occ_w + (c.ba >> 2), 1u << (8 * (c.ba & 3)));
        if (kind != 2 && (c.mir_move || kind == 1)) atomicAdd(occ_w + (c.bb >> 2), 1u << (8 * (c.bb & 3)));
      }
      int dn = 0;
      for (int k = 0; k < nacc; ++k) {
        const int ak = sh.mkind[sh.wr[0].acc_i[k]];
        dn += ak == 1 ? 1 : (ak == 2 ? -1 : 0);
      }
      if (lane == 0) {
        sh.base = base + (uint64_t)len;
        sh.n = (uint64_t)((int64_t)n + dn);
        sh.nprev = n;
        sh.cmin = kSM;
      }
      role_end(8);
    }
    stop = ro.err != 0;
    ++rounds;
    mark(4);
  }
  __syncthreads();
  if (tid == 0) {
    ChainState& ks = sh.ks;
    const uint64_t base = sh.base, n = sh.n;
    a.st->n = n;
    a.st->step = ks.step;
    a.st->energy = ks.energy;
    a.st->virial = ks.virial;
    for (int k = 0; k < 3; ++k) {
      a.st->attempted[k] = ks.attempted[k];
      a.st->accepted[k] = ks.accepted[k];
    }
    a.st->samples = ks.samples;
    a.st->sum_u = ks.sum_u;
    a.st->sum_p = ks.sum_p;
    a.st->sum_n = ks.sum_n;
    a.st->sum_n2 = ks.sum_n2;
    a.st->moves_done = base;
    a.st->rounds = rounds;
    a.st->pair_evals += sh.pairs;
    for (int k = 0; k < 5; ++k) a.st->pad[k] = ph[k];
    a.st->pad[8] = rounds;
    if (a.diag)
      for (int k = 0; k < 16; ++k) a.diag[k] = sh.racc[k];
    if (stop) {  // overflow at move `base` (slot len of the last round)
      const WalkRes& W = sh.wr[0];
      const int i = W.len;
      const int kind = sh.mkind[i];
      const uint32_t bb = mbrick(a.m, sh.ptn[i]);
      const int ob = __ldcg(a.m.occ + bb);
      bool ref = false;
      int cb = -1, ocb = 0;
      if (grid_on(a)) {
        cb = sh.cn[i];
        ocb = __ldcg(a.g.occ + cb);
        bool same_c = false;
        if (kind == 0) {
          const RW r = rw_of(a, sh, base - (uint64_t)i, sh.nprev, i, W.d[i]);
          same_c = r.co == cb;
        }
        ref = !same_c && ocb >= a.g.cap;
      }
      a.st->error = GCMC_CELL_OVERFLOW;
      a.st->err_a = ref ? cb : (int64_t)bb;
      a.st->err_b = ref ? ocb : ob;
      a.st->err_c = ref ? 0 : 1;
    }
  }
}

}  // namespace

// engine_mode 2, or 0 (auto) when at least kSmShare chains share the device:
// from there a CTA per chain beats 1/K of the device per chain (64k sweep:
// K = 8 engine2 10.2 M moves/s vs 9.2 M here, K = 16+ this engine,
// profiles/r02sm).
constexpr int kSmShare = 12;
bool engine_sm_supported(const Chain& c) {
  if (c.params.engine_mode != 2 && !(c.params.engine_mode == 0 && c.params.engine_share >= kSmShare))
    return false;
  if (c.params.max_displacement > 0.0) return false;
  if (c.grid.kind == GCMC_ALL_PAIRS) return false;
  return c.capn < (1ull << 31);
}

namespace {

SmArgs make_args(const Chain& c, uint64_t nmoves, gcmc_trace_rec* trace_d) {
  const gcmc_params& P = c.params;
  SmArgs a{};
  a.g = c.grid;
  a.m = c.mirror;
  a.b = c.box;
  a.s = Store{c.pos, c.rslot};
  a.ep = c.ep;
  a.st = c.st;
  a.props = c.props;
  a.trace = trace_d;
  a.nmoves = nmoves;
  a.capn = c.capn;
  a.beta = 1.0 / P.temperature;  // config.hpp:66
  a.mu = P.chemical_potential;
  a.lambda3 = P.lambda * P.lambda * P.lambda;
  a.vol = P.box_length * P.box_length * P.box_length;  // box.hpp:19
  a.temp = P.temperature;
  a.equil = P.equilibration_steps;
  a.interval = P.sampling_interval;
  a.tail = P.tail_corrections;
  const double sg = P.sigma, rc = P.r_cut;
  const double sr3 = (sg / rc) * (sg / rc) * (sg / rc);
  const double sr9 = sr3 * sr3 * sr3;
  const double pi = 3.141592653589793238462643383279502884;
  a.tail_cu = (8.0 / 3.0) * pi;
  a.tail_cp = (16.0 / 3.0) * pi;
  a.tail_s3 = sg * sg * sg;
  a.tail_bu = sr9 / 3.0 - sr3;
  a.tail_bp = 2.0 / 3.0 * sr9 - sr3;
  a.max_acc = kSAcc;
  return a;
}

// Dynamic shared memory for these chains: the engine's state plus the
// mirror-occupancy replica of every chain whose replica fits while a third of
// the SM's shared memory stays L1 (the call frames live there).
gcmc_status smem_plan(Chain* const* cs, int k, SmArgs* as, size_t& smem) {
  smem = (sizeof(SmShared) + 15) & ~size_t(15);
  int max_optin = 0, per_sm = 0;
  cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, cs[0]->device);
  cudaDeviceGetAttribute(&per_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, cs[0]->device);
  max_optin -= 1024;  // the static shared arguments
  // 256-thread build: two CTAs (chains) per SM, each within half the SM's
  // shared memory; 512 threads: one, with a third of it left to L1
  const size_t budget = kST <= 256 ? (size_t)per_sm / 2 - 2048 : (size_t)max_optin * 2 / 3;
  size_t occ = 0;
  for (int i = 0; i < k; ++i) {
    const size_t nb = ((size_t)cs[i]->mirror.nb + 15) & ~size_t(15);
    as[i].smem_occ = smem + nb <= budget ? 1 : 0;
    if (as[i].smem_occ) occ = occ > nb ? occ : nb;
  }
  smem += occ;
  if (smem > (size_t)max_optin) return set_error(GCMC_ARG, "engine_sm: shared memory");
  return GCMC_OK;
}

}  // namespace

gcmc_status engine_sm_run(Chain& c, uint64_t nmoves, gcmc_trace_rec* trace_d, cudaStream_t s) {
  if (nmoves == 0) return GCMC_OK;
  cudaError_t e;
  if (!c.e_valid) {
    gcmc_status st = epart_build(c, c.ep);
    if (st) return st;
    c.e_valid = true;
  }
  SmArgs a = make_args(c, nmoves, trace_d);
  static thread_local unsigned long long* diag = nullptr;
  const bool want_diag = std::getenv("GCMC_SM_PHASES") != nullptr;
  if (want_diag && !diag && cudaMalloc(&diag, 16 * sizeof(unsigned long long)) != cudaSuccess) diag = nullptr;
  if (want_diag) a.diag = diag;
  Chain* cp = &c;
  size_t smem = 0;
  gcmc_status st = smem_plan(&cp, 1, &a, smem);
  if (st) return st;
  if ((e = cudaFuncSetAttribute(k_engine_sm<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)))
    return cuda_error(e, "engine_sm smem");
  k_engine_sm<false><<<1, kST, smem, s>>>(a, nullptr);
  if ((e = cudaGetLastError())) return cuda_error(e, "engine_sm launch");
  if (std::getenv("GCMC_SM_PHASES")) {  // diagnostics: cycles per round by phase
    ChainState h;
    if (cudaMemcpyAsync(&h, c.st, sizeof h, cudaMemcpyDeviceToHost, s) == cudaSuccess &&
        cudaStreamSynchronize(s) == cudaSuccess && h.pad[8]) {
      const double r = (double)h.pad[8];
      std::fprintf(stderr,
                   "[engine_sm] smem %zu rounds %llu moves/round %.1f cycles/round: top %.0f eval %.0f "
                   "walk+verify %.0f commit1 %.0f commit2 %.0f\n",
                   smem, (unsigned long long)h.pad[8], h.moves_done / r, h.pad[0] / r, h.pad[1] / r,
                   h.pad[2] / r, h.pad[3] / r, h.pad[4] / r);
      unsigned long long d[16];
      if (diag && cudaMemcpy(d, diag, sizeof d, cudaMemcpyDeviceToHost) == cudaSuccess)
        std::fprintf(stderr,
                     "[engine_sm] role cycles/round (max over warps): eval %.0f walk %.0f verify %.0f "
                     "e-updates %.0f commit_loads %.0f ring %.0f statistics %.0f commit_stores %.0f "
                     "close %.0f\n",
                     d[0] / r, d[1] / r, d[2] / r, d[3] / r, d[4] / r, d[5] / r, d[6] / r, d[7] / r, d[8] / r);
      if (diag && cudaMemcpy(d, diag, sizeof d, cudaMemcpyDeviceToHost) == cudaSuccess)
        std::fprintf(stderr, "[engine_sm] steps (diagnostics build: -DGCMC_SM_STEPS energy updates: windows / occupancies+expansion / gather / stash; -DGCMC_SM_CL_STEPS commit loads): %.0f %.0f %.0f %.0f %.0f; commits/round %.2f ordered %.2f\n",
                     d[9] / r, d[10] / r, d[11] / r, d[12] / r, d[13] / r, d[15] / r, d[14] / r);
    }
  }
  return GCMC_OK;
}

gcmc_status engine_sm_run_many(Chain* const* cs, int k, const uint64_t* n, cudaStream_t s) {
  if (k <= 0) return GCMC_OK;
  cudaError_t e;
  std::vector<SmArgs> as(k);
  for (int i = 0; i < k; ++i) as[i] = make_args(*cs[i], n[i], nullptr);
  size_t smem = 0;
  gcmc_status st = smem_plan(cs, k, as.data(), smem);
  if (st) return st;
  if ((e = cudaFuncSetAttribute(k_engine_sm<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)))
    return cuda_error(e, "engine_sm smem");
  SmArgs* d = nullptr;
  if ((e = cudaMallocAsync(&d, k * sizeof(SmArgs), s))) return cuda_error(e, "engine_sm args");
  if ((e = cudaMemcpyAsync(d, as.data(), k * sizeof(SmArgs), cudaMemcpyHostToDevice, s)))
    return cuda_error(e, "engine_sm args");
  k_engine_sm<true><<<k, kST, smem, s>>>(SmArgs{}, d);
  if ((e = cudaGetLastError())) return cuda_error(e, "engine_sm launch");
  cudaFreeAsync(d, s);
  return GCMC_OK;
}

}  // namespace gcmcb
