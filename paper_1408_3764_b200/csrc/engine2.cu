// Maintained-energy engine: Simulation::step() x n (engine.hpp:293-308,
// 350-426) as exact multi-move speculation in which every move costs ONE
// evaluation slot, whatever N turns out to be.
//
// The per-window engine (engine.cu) pays a window evaluation for every
// distinct particle a displacement / deletion could pick over its candidate
// N: the old-position sum Σ_j u(x_pid, x_j) is what makes a move depend on N.
// Here every particle carries its current pair energy and virial
//   e[i] = Σ_{j != i, r_ij <= r_c} (u_ij, w_ij)
// maintained on the device across accepted moves, so
//   delete  pid:      ΔU = -e[pid]                                  (no window)
//   displace pid->n:  ΔU = (S(n) - pair(n, x_pid)) - e[pid]         (window of n)
//   insert  n:        ΔU = S(n)                                     (window of n)
// where S(n) = Σ_all pair(n, x_j) does not depend on N. A slot evaluates S(n)
// once with its whole group, then its leader warp resolves all 32 candidate N
// (offsets d = -16..15 around the round's starting N, one lane each: pid =
// index_from(pick, N + d), one load of x_pid and e[pid]) into accept bits.
// ΔU differs from the reference's Kahan sums only by rounding (parity bound
// 1e-10 relative, observed ~1e-15); the exclusion pair(n, x_pid) is a plain
// subtraction unless it is large enough to cost precision, in which case the
// warp re-sums the window without pid.
//
// A round: decision D_r (base, N, the previous round's accepted moves) ->
// each evaluator group takes slot s = move base + s (s < fit) -> the
// sequencer polls the slots' accept / stop / overflow masks, walks the moves
// tracking N, verifies that no consumed move read anything an earlier
// accepted move of the round changed (exact distances: a move reads the
// positions within r_c of its new point and e / x of its particle), and
// publishes D_{r+1}. Commits of round r run during round r+1:
//   * structural (positions, reference grid, brick mirror, e of the mover):
//     the sequencer's helper warp, then a release of flags[0] = r;
//   * pair-energy updates of the neighbours (e_j -= u(o, x_j), e_j += u(n,
//     x_j)): one reserved evaluator group per accepted move, after flags[0];
//     the sequencer waits for all of them before publishing D_{r+2}.
// An evaluation of round r+1 whose window overlaps a brick a round-r commit
// changes waits for flags[0] (it then reads the committed state); one whose
// particle might be touched by an in-flight commit or energy update (same
// index, or within r_c of a changed position) stops the walk there, and the
// move is re-evaluated in the next round.
//
// Supported: brick-window strategies (microcell, cell list) with whole-box
// displacements (max_displacement = 0, the bench and paper configuration).
// Otherwise engine.cu runs.
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "commit.cuh"
#include "internal.h"
#include "slot.cuh"
#include "sync.cuh"

namespace gcmcb {

namespace {

constexpr int kThreads = 512;
#ifndef GCMC_E2_MOVES
#define GCMC_E2_MOVES 384
#endif
constexpr int kMaxMoves = GCMC_E2_MOVES;  // moves per round
constexpr int kMH = kMaxMoves / 32;       // moves per walk lane
constexpr int kMaxAcc = 32;               // accepted moves per round (= reserved e-update groups)
constexpr int kRing = 2 * kMaxMoves;      // proposal ring (>= 2 * kMaxMoves)
constexpr int kHalf = 16;                 // N offsets d = -16..15 <-> bit d + 16
constexpr int kDecHdr = 4;
constexpr int kDecEnt = 4;
constexpr int kDecWords = kDecHdr + kDecEnt * kMaxAcc;  // 132
constexpr int kDecStride = 160;
constexpr int kResWords = 3;
constexpr int kPollWarps = 12;
constexpr int kMaxSlots = 768;            // buffer sizing: evaluator groups
constexpr double kHugeTerm = 1e4;
constexpr int kEBuf = 384;              // buffered energy updates per group in shared memory
constexpr int kEBig = 4096;             // ... and in global memory beyond that          // verify bitmap: up to 131072 bricks         // |pair(n, x_pid)| above this: re-sum without pid

struct OffRec {  // one candidate N offset of a slot (accepted offsets; all when tracing)
  double du, dw;  // ΔU, ΔW
  double su, sw;  // e of the mover after the move
  double pe;      // acceptance probability
  double pad;
};
struct SlotExt {
  OffRec off[32];
  uint64_t tag;
  uint64_t pad[3];
};
static_assert(sizeof(SlotExt) % 32 == 0, "SlotExt layout");

struct ATab {  // accepted move k of a round, exact (sequencer -> commit groups / evaluators)
  double ox, oy, oz, nx, ny, nz;
  int64_t ia, ib;
  uint64_t nn;     // store size before the move
  int32_t kind, slot, d;
  uint32_t deps;   // earlier accepted moves of the round this commit is ordered after
  uint64_t tag;    // round (stored last, release)
};
// flags[]: [kECount] energy updates done (cumulative); [kSFlag] last round whose
// accepted moves are committed (structural + the movers' e).
constexpr int kECount = 8;
constexpr int kSFlag = 9;   // same line as kECount (polled together)
constexpr int kGo = 24;      // last round whose evaluations are complete (commits may store)
constexpr int kETrav = 32;   // energy-update traversals done (cumulative)
constexpr int kFlagWords = 64;

struct EngineArgs {
  Grid g;
  Mirror m;
  Box b;
  Store s;
  double2* ep;
  ChainState* st;
  const Proposal* props;
  gcmc_trace_rec* trace;
  uint64_t nmoves;
  double beta, mu, lambda3, vol, temp;
  uint64_t equil, interval;
  int tail, nslots, fitmax;
  int max_acc;      // accepted moves per round = reserved energy-update groups (<= kMaxAcc)
  double tail_cu, tail_cp, tail_s3, tail_bu, tail_bp;
  uint64_t* dec;    // [kDecStride]
  uint64_t* res;    // [2][kResWords][nslots]
  SlotExt* ext;     // [2][nslots]
  ATab* atab;       // [2][kMaxAcc]
  uint64_t* flags;  // see kECount / kSFlag
  double4* ebig;    // [kMaxAcc][kEBig] energy-update overflow buffers
  int smem_occ;
  unsigned poll_ns, epoll_ns;
  int walk_reps;  // diagnostics: walk repeated (GCMC_WALK_REPS)
  unsigned long long* prof;
};

__device__ __forceinline__ int fit_of(const EngineArgs& a, uint64_t base) {
  if (base >= a.nmoves) return 0;
  const uint64_t left = a.nmoves - base;
  return left < (uint64_t)a.fitmax ? (int)left : a.fitmax;
}

__device__ __forceinline__ bool within_rc(const Box& b, double ax, double ay, double az, double bx,
                                          double by, double bz) {
  return min_image_dist2(ax, ay, az, bx, by, bz, b) <= b.rc2 * (1.0 + 1e-9);
}

// ----------------------------------------------------------------- decision
struct AccE {
  uint64_t pt0, pt1;  // brick points: new (displace / insert), old (displace / delete)
  int64_t ia, ib;     // particle (insert: its new index), last index (delete)
  int kind;
  int cn, co;         // reference cells of the new / old position (-1: none)
};
struct Dec {
  uint64_t base, n;
  uint64_t ctot;  // accepted moves through the listed round (cumulative, this launch)
  int nacc, stop;
  AccE acc[kMaxAcc];
};

__device__ __forceinline__ void ring_fill(const EngineArgs& a, Proposal* ring, uint64_t lo,
                                         uint64_t hi, int lane) {
  constexpr unsigned W = sizeof(Proposal) / 8;
  const unsigned cnt = (unsigned)(hi - lo) * W;
  for (unsigned k = lane; k < cnt; k += 32) {
    const uint64_t mv = lo + k / W;
    const unsigned w = k % W;
    cp_async8(reinterpret_cast<uint64_t*>(&ring[mv % kRing]) + w,
              reinterpret_cast<const uint64_t*>(a.props + mv) + w);
  }
  cp_async_commit();
}

// Warp: wait for D_r (self-validating tagged words) and decode it.
// The state D_r's evaluations read must be complete as well: the energy
// updates through round r - 2 (flags[kECount] >= ctot - nacc) and, when
// round r - 2 accepted moves, their commits (flags[kSFlag] >= r - 2). Both
// flags are polled with the decision words, so the sequencer publishes D_r
// without waiting for them.
__device__ __forceinline__ void poll_dec(const EngineArgs& a, uint32_t r, Dec& d, int lane, bool need_s) {
  constexpr int PER = (kDecWords + 31) / 32;  // 5
  uint64_t w[PER];
  const uint64_t* dec = a.dec;
#ifdef GCMC_PHASE_TIMERS
  unsigned long long t_tag = 0;  // first poll that saw the header words of D_r
#endif
  for (;;) {
    w[0] = ld_relaxed(dec + lane);
    w[1] = ld_relaxed(dec + 32 + lane);
    const uint64_t fl = lane < 2 ? ld_acquire(a.flags + (lane == 0 ? kECount : kSFlag)) : 0ull;
    const uint64_t h2 = __shfl_sync(0xffffffffu, w[0], 2);
    const uint64_t h3 = __shfl_sync(0xffffffffu, w[0], 3);
#ifdef GCMC_PHASE_TIMERS
    if (!t_tag && tagged(h2, r) && tagged(h3, r)) t_tag = gtimer();
#endif
    const uint64_t ecnt = __shfl_sync(0xffffffffu, fl, 0) & 0xffffffffull;
    const uint64_t sflg = __shfl_sync(0xffffffffu, fl, 1);
    const bool h2ok = tagged(h2, r) && tagged(h3, r) &&
                      ecnt + (h2 & 0xff) >= (h3 & kPay) && (!need_s || sflg + 2 >= (uint64_t)r);
    const int nacc = h2ok ? (int)(h2 & 0xff) : 0;
    const int need = kDecHdr + kDecEnt * nacc;
#pragma unroll
    for (int j = 2; j < PER; ++j) {
      const int idx = lane + 32 * j;
      w[j] = idx < need ? ld_relaxed(dec + idx) : 0;
    }
    bool ok = h2ok;
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      const int idx = lane + 32 * j;
      if (idx < need && !tagged(w[j], r)) ok = false;
    }
    if (__all_sync(0xffffffffu, ok)) break;
    __nanosleep(a.epoll_ns);
  }
#ifdef GCMC_PHASE_TIMERS
  if (a.prof && lane == 0 && r > 2 && t_tag) {  // decision visible vs state flags (ECount, SFlag) ready
    const unsigned long long pub = ld_relaxed(reinterpret_cast<uint64_t*>(a.prof + 3600 + (r & 1)));
    const unsigned long long now = gtimer();
    atomicAdd(a.prof + 3680, t_tag - pub);
    atomicAdd(a.prof + 3681, now - t_tag);
    atomicAdd(a.prof + 3682, 1ull);
    if (now - t_tag > 300) atomicAdd(a.prof + 3683, 1ull);
  }
#endif
  const uint64_t h2 = __shfl_sync(0xffffffffu, w[0], 2) & kPay;
  const int nacc = (int)(h2 & 0xff);
  const int need = kDecHdr + kDecEnt * nacc;
#pragma unroll
  for (int j = 0; j < PER; ++j) {
    const int idx = lane + 32 * j;
    if (idx >= need) continue;
    const uint64_t p = w[j] & kPay;
    if (idx == 0) d.base = p;
    else if (idx == 1) d.n = p;
    else if (idx == 2) {
      d.nacc = nacc;
      d.stop = (int)((p >> 9) & 1);
    } else if (idx == 3) {
      d.ctot = p;
    } else if (idx >= kDecHdr) {
      const int e = (idx - kDecHdr) / kDecEnt, f = (idx - kDecHdr) % kDecEnt;
      if (f == 0) {
        d.acc[e].pt0 = p & kNoPoint;
        d.acc[e].pt1 = (p >> 24) & kNoPoint;
      } else if (f == 1) {
        d.acc[e].kind = (int)(p >> 32) & 3;
        d.acc[e].ia = (int64_t)(uint32_t)p;
      } else if (f == 2) {
        const uint32_t ib = (uint32_t)p;
        d.acc[e].ib = ib == 0xffffffffu ? -1 : (int64_t)ib;
      } else {
        const int cn = (int)(p & 0xffffff), co = (int)((p >> 24) & 0xffffff);
        d.acc[e].cn = cn == 0xffffff ? -1 : cn;
        d.acc[e].co = co == 0xffffff ? -1 : co;
      }
    }
  }
  __syncwarp();
}

// 1 when both packed brick points exist and lie within r bricks of each
// other on every axis (cyclic), computed without branches.
__device__ __forceinline__ unsigned near_bits(uint32_t p, uint32_t q, int d, int r) {
  int dx = (int)(p & 0xffu) - (int)(q & 0xffu);
  int dy = (int)((p >> 8) & 0xffu) - (int)((q >> 8) & 0xffu);
  int dz = (int)((p >> 16) & 0xffu) - (int)((q >> 16) & 0xffu);
  dx = abs(dx);
  dy = abs(dy);
  dz = abs(dz);
  dx = min(dx, d - dx);
  dy = min(dy, d - dy);
  dz = min(dz, d - dz);
  return (unsigned)(p != (uint32_t)kNoPoint) & (unsigned)(q != (uint32_t)kNoPoint) & (unsigned)(dx <= r) &
         (unsigned)(dy <= r) & (unsigned)(dz <= r);
}

// The same test on packed bytes (all three axes at once) when dims <= 127:
// with t = |dp| < d per axis, u = |2t - d| <= 127, and
// min(t, d - t) <= reach  <=>  u >= d - 2 reach  (both branches of the min).
// near_ok adds 0x80 - max(d - 2 reach, 0) per byte (no carries: u <= 127) and
// wants bit 7 of all three bytes. Points must be valid (not kNoPoint).
struct NearK {
  uint32_t dd, add_r, add_2;
  bool simd;
};
__device__ __forceinline__ NearK near_k(int d, int reach) {
  const auto add = [d](int r) {
    const int k = d - 2 * r > 0 ? d - 2 * r : 0;
    const uint32_t b = (uint32_t)(0x80 - k);
    return b | (b << 8) | (b << 16);
  };
  return {(uint32_t)d | ((uint32_t)d << 8) | ((uint32_t)d << 16), add(reach), add(2), d <= 127};
}
__device__ __forceinline__ uint32_t near_u(uint32_t p, uint32_t q, uint32_t dd) {
  const uint32_t t = __vabsdiffu4(p, q);
  return __vabsdiffu4(t + t, dd);
}
__device__ __forceinline__ unsigned near_ok(uint32_t u, uint32_t add) {
  return ((u + add) & 0x808080u) == 0x808080u ? 1u : 0u;
}

// =================================================================== evaluator
template <int T>
struct EvalShared {
  Proposal ring[kRing];
  Dec d;
  struct EBuf {                   // buffered neighbour energy updates (energy_update)
    uint32_t id[kEBuf];            // particle | pass << 31
    double u[kEBuf], w[kEBuf];
    int n;
  } eb[kThreads / T];
  int nprev;                      // the previous decision's accepted moves (replica update)
  uint64_t nstore;                // particles in the store during this round (before the in-flight moves)
  uint32_t prev_pt0[kMaxAcc], prev_pt1[kMaxAcc];
  int prev_kind[kMaxAcc];
  WinWs<T> ws[kThreads / T];
  struct G {
    int task;        // 0 none, 1 evaluate move i, 2 energy update of accepted entry k
    int i, k, kind;
    double nx, ny, nz;
    double ox, oy, oz;
    int64_t excl;    // energy update: particle id excluded (the mover)
    int sgn0, sgn1;  // energy update: window signs
    uint32_t nearS;  // moves in flight whose changed points may be within r_c of n
  } gs[kThreads / T];
};

// The structural commits of the accepted moves of round rr (one warp, lane
// k = accepted move k): store, reference grid and brick mirror (commit.cuh).
// Everything is loaded while round rr + 1 is still being evaluated against
// the old state; stores start once its evaluations are complete (flags[kGo]).
// A commit whose cells, bricks or particles overlap an earlier one of the
// round is re-loaded and applied after it in move order (a later insertion
// reusing the index an earlier deletion vacated needs no order: the
// deletion's loads precede every store, unless it is itself ordered). The
// movers' e (set / relabel copy) are written in move order after the
// round's neighbour energy updates have been applied. Then flags[kSFlag] = rr.
// Branch-free form of touches() (commit.cuh): any shared cell, brick or particle.
__device__ __forceinline__ bool touches_bf(const Touch& a, const Touch& b) {
  unsigned hit = 0u;
#pragma unroll
  for (int x = 0; x < 3; ++x)
#pragma unroll
    for (int y = 0; y < 3; ++y)
      hit |= ((unsigned)(a.cell[x] >= 0) & (unsigned)(a.cell[x] == b.cell[y])) |
             ((unsigned)(a.brick[x] >= 0) & (unsigned)(a.brick[x] == b.brick[y]));
#pragma unroll
  for (int x = 0; x < 5; ++x)
#pragma unroll
    for (int y = 0; y < 5; ++y) hit |= (unsigned)(a.part[x] >= 0) & (unsigned)(a.part[x] == b.part[y]);
  return hit != 0u;
}

// Order test of this lane's commit against every earlier one of the round
// (one form): dep = must follow an earlier commit; exm = earlier deletions
// whose vacated index this insertion reuses. chain_form releases the relabel
// chains at the store's end (see commit_round).
__device__ __forceinline__ void touch_deps(const EngineArgs& a, const Touch& tc, int kind, int chain,
                                           int fsrc, bool mine, int lane, int nacc, bool chain_form,
                                           bool& dep, unsigned& exm) {
  Touch tme = tc;
  if (chain_form && (chain & 1)) tme.part[1] = -1;
  if (chain_form && (chain & 2)) tme.part[0] = -1;
  Touch tsh = tme;  // as seen by later lanes
#pragma unroll 1
  for (int j = 0; j < nacc - 1; ++j) {
    Touch tj;
#pragma unroll
    for (int x = 0; x < 3; ++x) {
      tj.cell[x] = __shfl_sync(0xffffffffu, tsh.cell[x], j);
      tj.brick[x] = __shfl_sync(0xffffffffu, tsh.brick[x], j);
    }
#pragma unroll
    for (int x = 0; x < 5; ++x) tj.part[x] = __shfl_sync(0xffffffffu, tsh.part[x], j);
    const int kj = __shfl_sync(0xffffffffu, kind, j);
    if (mine && j < lane) {
      Touch tm = tme;
      if (kind == 1 && kj == 2 && tm.part[0] >= 0 && tm.part[0] == tj.part[1]) {
        tm.part[0] = -1;
        exm |= 1u << j;
      }
      if (j == fsrc) {  // the forwarded particle's index, cell and record are expected
        tm.part[1] = -1;
        tm.cell[2] = -1;
        tm.brick[2] = -1;
      }
      if (touches_bf(tm, tj)) {
        dep = true;
#ifdef GCMC_PHASE_TIMERS
        if (a.prof && chain_form) {  // which pair of fields overlaps (diagnostics)
          int code = 63;
          for (int x = 0; x < 3 && code == 63; ++x)
            for (int y = 0; y < 3 && code == 63; ++y) {
              if (tm.cell[x] >= 0 && tm.cell[x] == tj.cell[y]) code = x * 3 + y;
              else if (tm.brick[x] >= 0 && tm.brick[x] == tj.brick[y]) code = 9 + x * 3 + y;
            }
          for (int x = 0; x < 5 && code == 63; ++x)
            for (int y = 0; y < 5 && code == 63; ++y)
              if (tm.part[x] >= 0 && tm.part[x] == tj.part[y]) code = 18 + x * 5 + y;
          atomicAdd(a.prof + 3660 + code, 1ull);
          atomicAdd(a.prof + 3730 + kind * 3 + kj, 1ull);
        }
#endif
      }
    }
  }
}

__device__ __noinline__ void commit_round(const EngineArgs& a, int nacc, uint32_t rr, uint64_t ctot,
                                          int lane) {
  const bool mine = lane < nacc;
  const ATab* t = a.atab + (size_t)(rr & 1) * kMaxAcc + lane;
  MoveData md{};
  CommitIn c{};
  Touch tc{};
  int kind = 0;
  uint64_t pid = 0, nn = 0;
  double esu = 0.0, esw = 0.0;
  PhaseClock cc;
  cc.start(a.prof && lane == 0);
  if (mine) {
    while (ld_acquire(&t->tag) != (uint64_t)rr) nap();
    cc.mark(0);
    kind = (int)__ldcg(&t->kind);
    nn = __ldcg(&t->nn);
    pid = kind == 1 ? 0 : (uint64_t)__ldcg(&t->ia);
    md.nx = __ldcg(&t->nx);
    md.ny = __ldcg(&t->ny);
    md.nz = __ldcg(&t->nz);
    md.rslot_pid = md.bslot_pid = -1;
    load_move(a.s, kind, pid, md);
    if (kind != 2) {
      const SlotExt* ex = a.ext + (size_t)(rr & 1) * a.nslots + __ldcg(&t->slot);
      while (ld_acquire(&ex->tag) != (uint64_t)rr) nap();
      const OffRec* o = &ex->off[__ldcg(&t->d) + kHalf];
      esu = __ldcg(&o->su);
      esw = __ldcg(&o->sw);
    }
    cc.mark(1);
    commit_load(a.g, a.m, a.s, kind, pid, nn, md, c);
    tc = touch_of(a.m, kind, pid, nn, c);
  }
  cc.mark(2);
  // Forwarding: a deletion that relabels a particle inserted earlier in this
  // round takes that particle's data (position, reference slot, record) from
  // the insertion's lane instead of waiting for its stores; its own stores
  // then follow the insertion's (pass B below).
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
  // Relabel chains at the store's end (insert at n, a deletion relabels it,
  // another insert at n, ...): a forwarded deletion never reads index q from
  // memory, and an insertion relabelled away by a later deletion of the
  // round need not write index n at all (skip_index). Without those
  // accesses the chain's commits are independent. This holds while no
  // member of a chain is ordered for another reason (an ordered forwarded
  // deletion re-loads q from memory); otherwise the round falls back to the
  // full ordering (dep1 below).
  const unsigned fwd_src = __reduce_or_sync(0xffffffffu, (mine && fsrc >= 0) ? (1u << fsrc) : 0u);
  const bool away = mine && kind == 1 && ((fwd_src >> lane) & 1u);
  const int chain = (fsrc >= 0 ? 1 : 0) | (away ? 2 : 0);
  bool dep = false;
  unsigned exm = 0;
  touch_deps(a, tc, kind, chain, fsrc, mine, lane, nacc, true, dep, exm);
  // an exempted / forwarded commit is ordered after its partner when the
  // partner itself is (it then loads or stores late)
#pragma unroll 1
  for (int it = 0; it < 32; ++it) {
    const unsigned b = __ballot_sync(0xffffffffu, dep);
    const bool nd = dep || (b & exm) || (fsrc >= 0 && ((b >> fsrc) & 1u));
    if (__ballot_sync(0xffffffffu, nd) == b) break;
    dep = nd;
  }
  const bool chains_free = !__any_sync(0xffffffffu, chain != 0 && dep);
  if (!chains_free) {  // full ordering (rare)
    dep = false;
    exm = 0u;
    touch_deps(a, tc, kind, chain, fsrc, mine, lane, nacc, false, dep, exm);
#pragma unroll 1
    for (int it = 0; it < 32; ++it) {
      const unsigned b = __ballot_sync(0xffffffffu, dep);
      const bool nd = dep || (b & exm) || (fsrc >= 0 && ((b >> fsrc) & 1u));
      if (__ballot_sync(0xffffffffu, nd) == b) break;
      dep = nd;
    }
  }
  const bool skip_index = chains_free && away;
  cc.mark(3);
  // stores only once the round being evaluated against the old state is
  // done, and the round's energy updates have found their neighbours
  if (lane == 0) {
    while (ld_acquire(a.flags + kGo) < (uint64_t)rr + 1) nap();
#ifdef GCMC_PHASE_TIMERS
    if (a.prof && rr > 2) {
      { const unsigned long long tn = gtimer(); a.prof[3655] += tn - ld_relaxed(reinterpret_cast<uint64_t*>(a.prof + 3640 + ((rr + 1) & 1))); }
      a.prof[3656] += 1;
    }
#endif
    while (ld_acquire(a.flags + kETrav) < ctot) nap();
  }
  __syncwarp();
  cc.mark(7);
  long long e1, e2, e3;
  if (mine && !dep && fsrc < 0)
    commit_store(a.g, a.m, a.s, &a.st->peak, kind, pid, nn, md, c, e1, e2, e3, skip_index);
  __syncwarp();  // pass B: forwarded deletions after their insertions
  if (mine && !dep && fsrc >= 0) commit_store(a.g, a.m, a.s, &a.st->peak, kind, pid, nn, md, c, e1, e2, e3);
  const unsigned deps = __ballot_sync(0xffffffffu, dep);
  cc.mark(4);
  if (deps) {
    __syncwarp();  // same warp: stores before the barrier are visible to loads after it
#pragma unroll 1
    for (int j = 0; j < nacc; ++j) {
      if (((deps >> j) & 1u) && lane == j) {
        load_move(a.s, kind, pid, md);
        commit_move(a.g, a.m, a.s, &a.st->peak, kind, pid, nn, md, e1, e2, e3);
      }
      __syncwarp();
    }
  }
  cc.mark(5);
  // the movers' e, after the neighbour updates of the round (a relabel copy
  // must carry them), in move order
  // Each lane writes e[x] (displace: pid, insert: its new index, delete: pid
  // <- e[q], q = n - 1). A deletion's source e[q] is the value the latest
  // earlier lane of the round wrote to index q, else memory (all loaded in
  // parallel, then resolved in move order by shuffles); the stores follow
  // move order (same-index writers: the last one wins).
  if (lane == 0) {
    while (ld_acquire(a.flags + kECount) < ctot) nap();
#ifdef GCMC_PHASE_TIMERS
    if (a.prof && rr > 2) {
      { const unsigned long long tn = gtimer(); a.prof[3653] += tn - ld_relaxed(reinterpret_cast<uint64_t*>(a.prof + 3640 + ((rr + 1) & 1))); }
      a.prof[3654] += 1;
    }
#endif
  }
  __syncwarp();
  const bool copies = mine && kind == 2 && pid != nn - 1;
  const int64_t ex = !mine ? -1 : (kind == 1 ? (int64_t)nn : (kind == 0 || copies ? (int64_t)pid : -1));
  const int64_t eq = copies ? (int64_t)(nn - 1) : -2;
  if (copies) {
    const double2 el = __ldcg(a.ep + (nn - 1));
    esu = el.x;
    esw = el.y;
  }
#pragma unroll 1
  for (int j = 0; j < nacc - 1; ++j) {  // lane j's value reaches later lanes copying index x_j
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
  __syncwarp();  // every lane's stores happen-before lane 0's (cumulative) release
  if (lane == 0) {
    // the release store alone (a separate fence first cost ~1.7 us per round
    // on the commit chain, profiles/r02/engine_variants.txt)
    st_release(a.flags + kSFlag, (uint64_t)rr);
#ifdef GCMC_PHASE_TIMERS
    if (a.prof && rr > 2) {
      { const unsigned long long tn = gtimer(); a.prof[3649] += tn - ld_relaxed(reinterpret_cast<uint64_t*>(a.prof + 3640 + ((rr + 1) & 1))); }
      a.prof[3650] += 1;
    }
#endif
  }
#ifdef GCMC_DBGDELAY
  __nanosleep(3000);  // robustness test: a committer that returns late
#endif
  cc.mark(6);
  const unsigned fwd_mask = __ballot_sync(0xffffffffu, fsrc >= 0 && !dep);
  (void)fwd_mask;
  if (cc.on) {
    for (int q = 0; q < 7; ++q) a.prof[80 + q] += cc.acc[q];
    a.prof[90] += cc.acc[7];
    a.prof[87] += 1;
    a.prof[88] += (unsigned long long)__popc(deps);
    a.prof[91] += (unsigned long long)__popc(fwd_mask);
    a.prof[89] += (unsigned long long)nacc;
  }
}

// Energy update of accepted move k of round r - 1 (a reserved group): the
// neighbours' e_j lose the pair with the old position and gain the pair with
// the new one. The neighbours are found on the state BEFORE the round's
// commits while round r is being evaluated (the round's accepted moves are
// more than 2 r_c apart, so none of them changes this move's neighbour set;
// the mover's own record is the one at its old position); the updates are
// buffered and applied (old window first, then new) once round r's
// evaluations are complete, before any relabel copy of the round.
template <int T>
__device__ __noinline__ void energy_update(const EngineArgs& a, EvalShared<T>& sh, WinWs<T>& ws, const uint8_t* occ_s,
                              uint32_t r, int g, int gt, int gw, int lane, int bar_id) {
  auto& G = sh.gs[g];
  auto& B = sh.eb[g];
  const uint32_t rr = r - 1;
  PhaseClock ec;
  ec.start(a.prof && G.k == 0 && gt == 0);
  if (gw == 0) {
    const ATab* t = a.atab + (size_t)(rr & 1) * kMaxAcc + G.k;
    if (lane == 0) {
      while (ld_acquire(&t->tag) != (uint64_t)rr) nap();
      ec.mark(0);
    }
    __syncwarp();
    const int kind = (int)__ldcg(&t->kind);
    const double ox = __ldcg(&t->ox), oy = __ldcg(&t->oy), oz = __ldcg(&t->oz);
    const double nx = __ldcg(&t->nx), ny = __ldcg(&t->ny), nz = __ldcg(&t->nz);
    int nent = 0, nent0 = 0;
    // window 0: new position (+), window 1: old position (-); a deletion has
    // only the old one (as window 0, sign -)
    if (kind != 2) nent = win_add<T>(a.m, a.b, ws, nent, nx, ny, nz, lane);
    nent0 = nent;
    if (kind != 1) nent = win_add<T>(a.m, a.b, ws, nent, ox, oy, oz, lane);
    if (kind == 2) nent0 = nent;
    win_finish<T>(a.m, ws, occ_s, nent, nent0, lane);  // replica = the state before the round's commits
    if (lane == 0) {
      G.kind = kind;
      G.nx = kind == 2 ? ox : nx;
      G.ny = kind == 2 ? oy : ny;
      G.nz = kind == 2 ? oz : nz;
      G.ox = ox;
      G.oy = oy;
      G.oz = oz;
      G.sgn0 = kind == 2 ? -1 : 1;
      G.sgn1 = -1;
      B.n = 0;
    }
  }
  group_sync(bar_id, T);
  ec.mark(1);
  const int total = ws.total;
  if (gt == 0) atomicAdd(&a.st->pair_evals, (unsigned long long)total);
  const double c0x = G.nx, c0y = G.ny, c0z = G.nz, c1x = G.ox, c1y = G.oy, c1z = G.oz;
  const double s0 = (double)G.sgn0, s1 = (double)G.sgn1;
  const bool has_old = G.kind != 1;
  for (int f = gt; f < total; f += T) {
    int e, k;
    if (f < kCandMax) {
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
    const bool w1 = e >= ws.nent0;
    const int idx = (int)ws.brick[e] * a.m.cap + k;
    const double rx = __ldcg(a.m.rx + idx), ry = __ldcg(a.m.ry + idx), rz = __ldcg(a.m.rz + idx);
    if (has_old && rx == c1x && ry == c1y && rz == c1z) continue;  // the mover itself
    const double r2 = w1 ? min_image_dist2(c1x, c1y, c1z, rx, ry, rz, a.b)
                         : min_image_dist2(c0x, c0y, c0z, rx, ry, rz, a.b);
    if (r2 <= a.b.rc2) {
      double u, w;
      lj_pair_clamped(r2, a.b, u, w);
      const double sg = w1 ? s1 : s0;
      const int32_t rid = __ldcg(a.m.rid + idx);
      const int q = atomicAdd(&B.n, 1);
      const int pass = (w1 || G.kind == 2) ? 0 : 1;  // old window first
      if (q < kEBuf) {
        B.id[q] = (uint32_t)rid | ((uint32_t)pass << 31);
        B.u[q] = __dmul_rn(sg, u);
        B.w[q] = __dmul_rn(sg, w);
      } else {
        if (q - kEBuf < kEBig) a.ebig[(size_t)G.k * kEBig + (q - kEBuf)] = make_double4(__longlong_as_double((long long)rid | ((long long)pass << 40)), __dmul_rn(sg, u), __dmul_rn(sg, w), 0.0);
      }
    }
  }
  __threadfence();
  group_sync(bar_id, T);
  if (gt == 0) {
    atomicAdd(reinterpret_cast<unsigned long long*>(a.flags + kETrav), 1ull);
    while (ld_acquire(a.flags + kGo) < (uint64_t)r) nap();
  }
  group_sync(bar_id, T);
  ec.mark(2);
  const int nb = B.n;
  // old window first (a particle near both positions gets two updates)
  for (int pass = 0; pass < 2; ++pass) {
    if (pass == 1) {
      __threadfence();
      group_sync(bar_id, T);
    }
    for (int q = gt; q < nb; q += T) {
      uint32_t id;
      double du, dw;
      int ps;
      if (q < kEBuf) {
        id = B.id[q] & 0x7fffffffu;
        ps = (int)(B.id[q] >> 31);
        du = B.u[q];
        dw = B.w[q];
      } else {
        const double4 v = ld_cg(a.ebig + (size_t)G.k * kEBig + (q - kEBuf));
        const long long bits = __double_as_longlong(v.x);
        id = (uint32_t)(bits & 0x7fffffffll);
        ps = (int)(bits >> 40);
        du = v.y;
        dw = v.z;
      }
      if (ps != pass) continue;
      atomicAdd(&a.ep[id].x, du);
      atomicAdd(&a.ep[id].y, dw);
    }
  }
  __threadfence();
  group_sync(bar_id, T);
  if (gt == 0) atomicAdd(reinterpret_cast<unsigned long long*>(a.flags + kECount), 1ull);
#ifdef GCMC_PHASE_TIMERS
  if (a.prof && gt == 0 && r > 3) {  // ns after go_r: this group's updates applied
    atomicAdd(a.prof + 3651, gtimer() - ld_relaxed(reinterpret_cast<uint64_t*>(a.prof + 3640 + (r & 1))));
    atomicAdd(a.prof + 3652, 1ull);
  }
#endif
  ec.mark(3);
  if (ec.on)
    for (int q = 0; q < 4; ++q) atomicAdd(a.prof + 64 + q, ec.acc[q]);
  if (ec.on) atomicAdd(a.prof + 68, 1ull);
}

// Change of Σ pair(x, ·) caused by the in-flight accepted move t: minus the
// pair with its old position, plus the pair with its new one (each only
// within r_c), as its commit and energy update will apply them.
__device__ __noinline__ void pair_delta(const EngineArgs& a, const ATab* t, double x, double y,
                                        double z, double& cu, double& cw) {
  cu = cw = 0.0;
  const int k = (int)__ldcg(&t->kind);
  if (k != 1) {
    const double r2 = min_image_dist2(x, y, z, __ldcg(&t->ox), __ldcg(&t->oy), __ldcg(&t->oz), a.b);
    if (r2 <= a.b.rc2) {
      double u, w;
      lj_pair_clamped(r2, a.b, u, w);
      cu = __dsub_rn(cu, u);
      cw = __dsub_rn(cw, w);
    }
  }
  if (k != 2) {
    const double r2 = min_image_dist2(x, y, z, __ldcg(&t->nx), __ldcg(&t->ny), __ldcg(&t->nz), a.b);
    if (r2 <= a.b.rc2) {
      double u, w;
      lj_pair_clamped(r2, a.b, u, w);
      cu = __dadd_rn(cu, u);
      cw = __dadd_rn(cw, w);
    }
  }
}

// S(n) after the in-flight moves in `near`, without particle xp (-1: none),
// re-summed by one warp in a fixed order: the window's records except xp and
// the old positions of those moves, plus the pairs with their new positions.
// Used when a pair to subtract is too large to subtract without losing
// precision (the mover's own pair, or an in-flight move's old position).
template <int T>
__device__ __noinline__ void resum_excl(const EngineArgs& a, const WinWs<T>& ws, double px, double py,
                                        double pz, int64_t xp, unsigned near, const ATab* tab,
                                        int lane, double& au, double& aw) {
  au = 0.0;
  aw = 0.0;
  for (int f = lane; f < ws.total; f += 32) {
    int e, k;
    if (f < kCandMax) {
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
    const int idx = (int)ws.brick[e] * a.m.cap + k;
    if ((int64_t)__ldcg(a.m.rid + idx) == xp) continue;
    const double rx = __ldcg(a.m.rx + idx), ry = __ldcg(a.m.ry + idx), rz = __ldcg(a.m.rz + idx);
    bool gone = false;
    for (unsigned m = near; m; m &= m - 1) {
      const ATab* t = tab + (__ffs(m) - 1);
      if (__ldcg(&t->kind) != 1 && rx == __ldcg(&t->ox) && ry == __ldcg(&t->oy) && rz == __ldcg(&t->oz))
        gone = true;
    }
    if (gone) continue;
    const double r2 = min_image_dist2(px, py, pz, rx, ry, rz, a.b);
    if (r2 <= a.b.rc2) lj_accum(a.b, r2, 1.0, au, aw);
  }
  double cu = 0.0, cw = 0.0;
  if ((near >> lane) & 1u) {
    const ATab* t = tab + lane;
    if (__ldcg(&t->kind) != 2) {
      const double r2 = min_image_dist2(px, py, pz, __ldcg(&t->nx), __ldcg(&t->ny), __ldcg(&t->nz), a.b);
      if (r2 <= a.b.rc2) lj_accum(a.b, r2, 1.0, cu, cw);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    au = __dadd_rn(au, __shfl_xor_sync(0xffffffffu, au, o));
    aw = __dadd_rn(aw, __shfl_xor_sync(0xffffffffu, aw, o));
    cu = __dadd_rn(cu, __shfl_xor_sync(0xffffffffu, cu, o));
    cw = __dadd_rn(cw, __shfl_xor_sync(0xffffffffu, cw, o));
  }
  au = __dadd_rn(au, cu);
  aw = __dadd_rn(aw, cw);
}

template <int T>
__device__ void evaluator(const EngineArgs& a, uint8_t* smem) {
  constexpr int MG = kThreads / T;
  constexpr int kGW = T / 32;
  auto& sh = *reinterpret_cast<EvalShared<T>*>(smem);
  uint8_t* occ_s = a.smem_occ ? smem + ((sizeof(EvalShared<T>) + 15) & ~size_t(15)) : nullptr;
  uint32_t* occ_w = reinterpret_cast<uint32_t*>(occ_s);
  const int tid = threadIdx.x, lane = tid & 31;
  const int g = tid / T, gt = tid % T, gw = gt >> 5;
  const int bar_id = 1 + g;
  const int slot = (blockIdx.x - 1) * MG + g;
  const int eslot0 = a.nslots - a.max_acc;  // groups reserved for energy updates
  WinWs<T>& ws = sh.ws[g];
  auto& G = sh.gs[g];
  const bool grid = a.g.kind != GCMC_ALL_PAIRS;
  const bool tracing = a.trace != nullptr;

  if (occ_s)
    for (uint32_t i = tid; i < a.m.nb; i += kThreads) occ_s[i] = (uint8_t)__ldcg(a.m.occ + i);
  if (tid == 0) sh.nprev = 0;
  uint64_t ring_hi = a.nmoves < (uint64_t)kRing ? a.nmoves : (uint64_t)kRing;
  if (tid < 32) {
    ring_fill(a, sh.ring, 0, ring_hi, lane);
    cp_async_wait();
  }
  __syncwarp();
    __syncthreads();
  PhaseClock pc;
  pc.start(a.prof && blockIdx.x == 1 && tid == 0);
  for (uint32_t r = 1;; ++r) {
    pc.mark(0);
    if (tid < 32) {
      poll_dec(a, r, sh.d, lane, sh.nprev > 0);
#ifdef GCMC_PHASE_TIMERS
      if (a.prof && lane == 0 && r > 2) {
        const unsigned long long dt = gtimer() - ld_relaxed(reinterpret_cast<uint64_t*>(a.prof + 3600 + (r & 1)));
        atomicAdd(a.prof + 3610, dt);
        atomicMax(a.prof + 3611, dt);
        atomicAdd(a.prof + 3612, 1ull);
      }
#endif
      const Dec& d = sh.d;
      // replica = memory: the commits of the moves the PREVIOUS decision
      // listed have landed (a--, b++); this decision's run after this
      // round's evaluations
      if (occ_s && lane < sh.nprev) {
        const int k = sh.prev_kind[lane];
        if (k != 1) {
          const uint32_t ba = mbrick(a.m, sh.prev_pt1[lane]);
          atomicSub(occ_w + (ba >> 2), 1u << (8 * (ba & 3)));
        }
        if (k != 2) {
          const uint32_t bb = mbrick(a.m, sh.prev_pt0[lane]);
          atomicAdd(occ_w + (bb >> 2), 1u << (8 * (bb & 3)));
        }
      }
      __syncwarp();
      if (lane < d.nacc) {
        sh.prev_kind[lane] = d.acc[lane].kind;
        sh.prev_pt0[lane] = (uint32_t)d.acc[lane].pt0;
        sh.prev_pt1[lane] = (uint32_t)d.acc[lane].pt1;
      }
      {  // the store still holds the state before the in-flight moves (all-pairs scans it)
        const int kd = lane < d.nacc ? d.acc[lane].kind : 0;
        const int dn = __reduce_add_sync(0xffffffffu, kd == 1 ? 1 : (kd == 2 ? -1 : 0));
        if (lane == 0) sh.nstore = (uint64_t)((int64_t)d.n - dn);
      }
      if (lane == 0) sh.nprev = d.nacc;
      if (lane < MG) {
        const int s = slot - g + lane;
        const int fit = d.stop ? 0 : fit_of(a, d.base);
        auto& Gl = sh.gs[lane];
        Gl.task = 0;
        if (s < fit) {
          Gl.task = 1;
          Gl.i = s;
        } else if (s >= eslot0 && s - eslot0 < d.nacc) {
          Gl.task = 2;
          Gl.k = s - eslot0;
        } else if (s == eslot0 - 1 && d.nacc > 0) {
          Gl.task = 3;  // structural commits of the previous round
        }
      }
      cp_async_wait();
    }
    __syncwarp();
    __syncthreads();
    pc.mark(1);
    const Dec& d = sh.d;
    const bool stop_r = d.stop;  // this round's decision (sh.d is rewritten by the next decode)
    if (G.task == 3 && gt < 32) commit_round(a, d.nacc, r - 1, d.ctot, lane);
    if (G.task == 2) energy_update<T>(a, sh, ws, occ_s, r, g, gt, gw, lane, bar_id);
    if (stop_r) break;
    if (G.task == 1) {
      const int lw = g % (kGW < 4 ? kGW : 4);  // leader warp (groups on different sub-partitions)
      const uint64_t mv = d.base + (uint64_t)G.i;
      const Proposal& pr = sh.ring[mv % kRing];
      const int kind = pr.kind;
      uint64_t* rw = a.res + (size_t)(r & 1) * kResWords * a.nslots + slot;
      SlotExt* ex = a.ext + (size_t)(r & 1) * a.nslots + slot;
      // per-lane candidate state (leader warp only)
      const int dd = lane - kHalf;
      const int64_t nd = (int64_t)d.n + dd;
      const bool valid = kind == 1 ? nd >= 0 : nd >= 1;  // kinds 0/2 at N <= 0: counted rejection
      uint64_t pid = 0;
      double xox = 0.0, xoy = 0.0, xoz = 0.0, eu = 0.0, ew = 0.0, fpre = 1.0;
      int ocb = 0, ob = 0;
      bool cf = false;
      if (gw == lw) {
        // candidate particles: one L2 hop for x_pid and e[pid], issued first
        if (kind != 1 && valid) {
          pid = index_from(pr.pick, (uint64_t)nd);
          const double* op = reinterpret_cast<const double*>(a.s.pos + pid);
          xox = __ldcg(op);
          xoy = __ldcg(op + 1);
          xoz = __ldcg(op + 2);
          const double2 e2 = __ldcg(a.ep + pid);
          eu = e2.x;
          ew = e2.y;
        }
        // the exchange ratio's prefactor for this lane's N (engine.hpp:28-59,
        // same operations), computed while the loads above are in flight
        {
          const double nn = (double)nd;
          fpre = kind == 1 ? __ddiv_rn(a.vol, __dmul_rn(a.lambda3, __dadd_rn(nn, 1.0)))
                           : (kind == 2 ? __ddiv_rn(__dmul_rn(a.lambda3, nn), a.vol) : 1.0);
        }
        int nent = 0;
        pc.mark(6);
        // The previous round's accepted moves (this decision's list) are not
        // committed yet: the state read here is the one before them, and
        // their effect is added exactly (pair terms of their changed
        // positions, occupancy counts); a candidate particle whose index they
        // touch stops the walk.
        uint64_t pn = kNoPoint;
        if (kind != 2) {
          if (pr.wmask != kNoMask) nent = window_bricks_mask(a.m, pr.wmask, pr.bpt, ws.brick, lane);
          else nent = win_add<T>(a.m, a.b, ws, 0, pr.x, pr.y, pr.z, lane);
          pn = pr.wmask != kNoMask ? (uint64_t)pr.bpt : mpoint(a.m, pr.x, pr.y, pr.z);
          const int cb = grid ? (pr.wmask != kNoMask ? pr.cell : cell_of(a.g, pr.x, pr.y, pr.z)) : -1;
          const uint32_t bb = mbrick(a.m, pn);
          // occupancy corrections and S(n) neighbours among the moves in flight
          int dob = 0, docb = 0;
          bool nearS = false;
          if (lane < d.nacc) {
            const AccE& A = d.acc[lane];
            if (A.kind != 1 && mbrick(a.m, A.pt1) == bb) --dob;
            if (A.kind != 2 && mbrick(a.m, A.pt0) == bb) ++dob;
            if (grid && A.kind != 1 && A.co == cb) --docb;
            if (grid && A.kind != 2 && A.cn == cb) ++docb;
            nearS = mnear(a.m, pn, A.pt0) || mnear(a.m, pn, A.pt1);
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            dob += __shfl_xor_sync(0xffffffffu, dob, o);
            docb += __shfl_xor_sync(0xffffffffu, docb, o);
          }
          const unsigned nm = __ballot_sync(0xffffffffu, nearS);
          if (lane == 0) {
            ob = (occ_s ? (int)occ_s[bb] : __ldcg(a.m.occ + bb)) + dob;
            if (grid) ocb = __ldcg(a.g.occ + cb) + docb;
            G.nearS = nm;
          }
          pc.mark(7);
          win_finish<T>(a.m, ws, occ_s, nent, nent, lane);
        }
        if (lane == 0) {
          G.kind = kind;
          ws.excl = -1;
          ws.nwin = 1;
          ws.sign1 = 1;
          ws.cx[0] = pr.x;
          ws.cy[0] = pr.y;
          ws.cz[0] = pr.z;
          if (kind == 2) {
            ws.total = 0;
            G.nearS = 0u;
          }
        }
        pc.mark(8);
        // the candidate particle's position / e vs the moves in flight
        if (kind != 1) {
          // branch-free scan of the moves in flight (uniform trip count), then
          // the rare brick-near ones exactly, in move order
          const uint32_t po = valid ? (uint32_t)mpoint(a.m, xox, xoy, xoz) : (uint32_t)kNoPoint;
          const int ip = valid ? (int)pid : -7;
          const int dm = a.m.dims, rch = a.m.reach;
          unsigned hit = 0u, nearm = 0u;
          const NearK nk = near_k(dm, rch);
          if (nk.simd) {
            const unsigned pv = po != (uint32_t)kNoPoint ? 1u : 0u;
#pragma unroll 2
            for (int k = 0; k < d.nacc; ++k) {
              const AccE& A = d.acc[k];
              const uint32_t p0 = (uint32_t)A.pt0, p1 = (uint32_t)A.pt1;
              hit |= ((unsigned)(ip == (int)A.ia) | (unsigned)(ip == (int)A.ib)) << k;
              const unsigned n0 = near_ok(near_u(po, p0, nk.dd), nk.add_r) & (unsigned)(p0 != (uint32_t)kNoPoint);
              const unsigned n1 = near_ok(near_u(po, p1, nk.dd), nk.add_r) & (unsigned)(p1 != (uint32_t)kNoPoint);
              nearm |= (pv & (n0 | n1)) << k;
            }
          } else {
#pragma unroll 2
            for (int k = 0; k < d.nacc; ++k) {
              const AccE& A = d.acc[k];
              hit |= ((unsigned)(ip == (int)A.ia) | (unsigned)(ip == (int)A.ib)) << k;
              nearm |= (near_bits(po, (uint32_t)A.pt0, dm, rch) | near_bits(po, (uint32_t)A.pt1, dm, rch)) << k;
            }
          }
          cf = valid && hit != 0u;
          if (valid && !cf) {
            for (unsigned m = nearm; m; m &= m - 1) {
              const int k = __ffs(m) - 1;
              const ATab* t = a.atab + (size_t)((r - 1) & 1) * kMaxAcc + k;
              while (ld_acquire(&t->tag) != (uint64_t)(r - 1)) nap();
              double cu = 0.0, cw = 0.0;
              pair_delta(a, t, xox, xoy, xoz, cu, cw);
              eu = __dadd_rn(eu, cu);
              ew = __dadd_rn(ew, cw);
            }
          }
        }
      }
      pc.mark(9);
      group_sync(bar_id, T);
      pc.mark(2);
      // ---- S(n): the whole group
      double su = 0.0, sw = 0.0;
      // all-pairs strategy (strategy.hpp:64-116): S(n) over the whole store,
      // in-flight moves corrected below like the brick window's
      const bool allp = a.g.kind == GCMC_ALL_PAIRS;
      if (kind != 2) {
        if (allp) allpairs_sums<T>(a.b, a.s.pos, sh.nstore, ws, -1, gt, su, sw);
        else win_sums<T>(a.m, a.b, ws, gt, su, sw);
      }
      if (gt == 0 && kind != 2)
        atomicAdd(&a.st->pair_evals, (unsigned long long)(allp ? sh.nstore : (uint64_t)ws.total));
      group_reduce<T>(ws, su, sw, bar_id, gt, 32 * lw);
      pc.mark(3);
      if (gw == lw) {
        su = __shfl_sync(0xffffffffu, su, 0);
        sw = __shfl_sync(0xffffffffu, sw, 0);
        const ATab* tabr = a.atab + (size_t)((r - 1) & 1) * kMaxAcc;
        if (G.nearS) {  // S(n) after the moves in flight (fixed-order sum of their pair changes)
          double cu = 0.0, cw = 0.0;
          bool huge = false;
          if ((G.nearS >> lane) & 1u) {
            const ATab* t = tabr + lane;
            while (ld_acquire(&t->tag) != (uint64_t)(r - 1)) nap();
            pair_delta(a, t, pr.x, pr.y, pr.z, cu, cw);
            huge = fabs(cu) > kHugeTerm || fabs(cw) > kHugeTerm;
          }
          if (__any_sync(0xffffffffu, huge)) {
            resum_excl<T>(a, ws, pr.x, pr.y, pr.z, -1, G.nearS, tabr, lane, su, sw);
          } else {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
              cu = __dadd_rn(cu, __shfl_xor_sync(0xffffffffu, cu, o));
              cw = __dadd_rn(cw, __shfl_xor_sync(0xffffffffu, cw, o));
            }
            su = __dadd_rn(su, cu);
            sw = __dadd_rn(sw, cw);
          }
        }
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
            slow = fabs(tu) > kHugeTerm || fabs(tw) > kHugeTerm;
            mu_ = __dsub_rn(su, tu);
            mw = __dsub_rn(sw, tw);
          } else {
            du = -eu;
            dw = -ew;
          }
        }
        // rare: the mover's own pair is large -> S(n) without pid, re-summed (warp, fixed order)
        unsigned sl = __ballot_sync(0xffffffffu, slow);
        while (sl) {
          const int src = __ffs(sl) - 1;
          sl &= sl - 1;
          const int64_t xp = (int64_t)__shfl_sync(0xffffffffu, (unsigned long long)pid, src);
          double au, aw;
          resum_excl<T>(a, ws, pr.x, pr.y, pr.z, xp, G.nearS, tabr, lane, au, aw);
          if (lane == src) {
            mu_ = au;
            mw = aw;
          }
        }
        if (kind == 0) {
          du = __dsub_rn(mu_, eu);
          dw = __dsub_rn(mw, ew);
        }
        {  // engine.hpp:28-59 with one exponential (same operation order)
          const double x = kind == 0 ? __dmul_rn(-a.beta, du)
                         : (kind == 1 ? __dmul_rn(a.beta, __dsub_rn(a.mu, du))
                                      : __dmul_rn(-a.beta, __dadd_rn(a.mu, du)));
          const double ex = exp(x);
          if (valid) p = metropolis(kind == 0 ? ex : __dmul_rn(fpre, ex));
        }
        const bool acc = valid && pr.acc < p;
        // overflow of the commit (exact: occupancies after the previous round)
        ob = __shfl_sync(0xffffffffu, ob, 0);
        ocb = __shfl_sync(0xffffffffu, ocb, 0);
        bool ovf = false;
        if (valid && kind != 2) {
          const uint32_t bb = mbrick(a.m, pr.wmask != kNoMask ? (uint64_t)pr.bpt : mpoint(a.m, pr.x, pr.y, pr.z));
          const bool same_b = kind == 0 && mbrick(a.m, mpoint(a.m, xox, xoy, xoz)) == bb;
          if (!same_b && ob >= a.m.cap) ovf = true;
          if (grid) {
            const int cb = pr.wmask != kNoMask ? pr.cell : cell_of(a.g, pr.x, pr.y, pr.z);
            const bool same_c = kind == 0 && cell_of(a.g, xox, xoy, xoz) == cb;
            if (!same_c && ocb >= a.g.cap) ovf = true;
          }
        }
        const uint32_t accm = __ballot_sync(0xffffffffu, acc);
        const uint32_t cfm = __ballot_sync(0xffffffffu, cf);
        const uint32_t ovm = __ballot_sync(0xffffffffu, ovf);
        if (lane < kResWords) {
          const uint64_t pw = lane == 0 ? ((uint64_t)kind | ((uint64_t)accm << 8))
                                        : (lane == 1 ? (uint64_t)cfm : (uint64_t)ovm);
          st_relaxed(rw + (size_t)lane * a.nslots, tagw(r, pw));
#ifdef GCMC_PHASE_TIMERS
          if (a.prof && lane == 0 && r > 2) {
            const unsigned long long dt = gtimer() - ld_relaxed(reinterpret_cast<uint64_t*>(a.prof + 3600 + (r & 1)));
            atomicAdd(a.prof + 3613, dt);
            atomicAdd(a.prof + 3614, 1ull);
            atomicMax(reinterpret_cast<unsigned long long*>(a.prof + 3620 + (r & 7)), dt);
          }
#endif
        }
        pc.mark(4);
        // payload for commits / statistics / trace (off the critical path)
        if (acc || tracing) {
          OffRec o;
          o.du = du;
          o.dw = dw;
          o.su = mu_;
          o.sw = mw;
          o.pe = valid ? p : 0.0;
          o.pad = 0.0;
          ex->off[lane] = o;
          __threadfence();
        }
        __syncwarp();
        if (lane == 0) {
          fence_gpu();
          st_relaxed(&ex->tag, (uint64_t)r);
        }
      }
    }
    // ring refill (off the critical path)
    if (tid < 32) {
      const uint64_t want = d.base + kRing < a.nmoves ? d.base + kRing : a.nmoves;
      if (want > ring_hi) {
        ring_fill(a, sh.ring, ring_hi, want, lane);
        ring_hi = want;
      }
    }
    pc.mark(5);
    // every warp of the CTA is done with this round's decision, tasks and
    // shared state before warp 0 decodes the next one (a late group would
    // otherwise read the next decision's stop flag / task)
    __syncwarp();
    __syncthreads();
  }
  if (a.prof && blockIdx.x == 1 && tid == 0) pc.flush(a.prof + 16);
}

// =================================================================== sequencer
struct Round {  // a decided round, handed to the helper warps
  uint64_t base, n;
  uint32_t r;
  int len, nacc, par;
  int acc_i[kMaxAcc], acc_d[kMaxAcc], acc_kind[kMaxAcc];
  int64_t acc_ia[kMaxAcc], acc_ib[kMaxAcc];
  double acc_nx[kMaxAcc], acc_ny[kMaxAcc], acc_nz[kMaxAcc];
  int res_d[kMaxMoves];
  uint8_t kind[kMaxMoves];
};

enum Stop { kStopEnd, kStopRange, kStopPrev, kStopVerify, kStopFull, kStopOverflow, kNStop };

struct AccV {  // an accepted move's write set, packed for the verify
  int j, ia, ib;
  uint32_t an, ao, bn, bo;
  int cn, co;
};

struct SeqShared {
  Proposal ring[kRing];
  AccV av[kMaxAcc];
  alignas(16) uint32_t macc[kMaxMoves];
  alignas(16) uint32_t mcf[kMaxMoves];
  alignas(16) uint32_t movf[kMaxMoves];
  alignas(16) uint8_t mkind[kMaxMoves];
  int len, nacc, err, cmin, why, dend, arrived, plen;
  unsigned long long vmax, vsum;  // diagnostics
  unsigned viters, vcalls;
  int wscr_i[kMaxAcc], wscr_d[kMaxAcc];  // walk dry runs (discarded)
  int8_t wscr_k[kMaxMoves];
  // the previous round's masks, the dry walk's input (the live masks are
  // being written by the poll while it runs)
  uint32_t pacc[kMaxMoves], pcf[kMaxMoves], povf[kMaxMoves];
  uint8_t pkind[kMaxMoves];
  int acc_i[kMaxAcc], acc_d[kMaxAcc];
  int res_d[kMaxMoves];
  // read / write sets of the consumed moves (verify)
  double xo[kMaxMoves][3];
  uint32_t pto[kMaxMoves], ptn[kMaxMoves];
  int32_t co[kMaxMoves], cn[kMaxMoves];
  int64_t ia[kMaxMoves], ib[kMaxMoves];
  Round done;
  double acc_du[kMaxAcc], acc_dw[kMaxAcc];
  double st_e[kMaxAcc + 1], st_w[kMaxAcc + 1];
  uint64_t st_n[kMaxAcc + 1];
  double st_v[kMaxAcc + 1][4];
  unsigned long long stops[kNStop];
  unsigned smp[kMH];          // statistics: sampled steps of the round
  int8_t acck[kMaxMoves];     // accepted index of a consumed move (-1: rejected)
  uint8_t nbef[kMaxMoves];    // accepted moves before a consumed move
  uint64_t dw[kDecWords];
  int dneed;
  ChainState ks;
};

struct Observables {
  double rep_u, pres;
};

// reported_energy() and pressure() (engine.hpp:277-291) with the tail terms
// of tail_corrections() (potential.hpp:63-72), same operation order.
__device__ __noinline__ Observables observables(const EngineArgs& a, uint64_t n, double u,
                                                   double w) {
  const double rho = __ddiv_rn((double)n, a.vol);
  double p = __dadd_rn(__dmul_rn(rho, a.temp), __ddiv_rn(w, __dmul_rn(3.0, a.vol)));
  double ru = u;
  if (a.tail) {
    const double tu = __dmul_rn(
        __dmul_rn(__dmul_rn(__dmul_rn(a.tail_cu, rho), a.b.eps), a.tail_s3), a.tail_bu);
    const double tp = __dmul_rn(
        __dmul_rn(__dmul_rn(__dmul_rn(__dmul_rn(a.tail_cp, rho), rho), a.b.eps), a.tail_s3),
        a.tail_bp);
    p = __dadd_rn(p, tp);
    ru = __dadd_rn(ru, __dmul_rn((double)n, tu));
  }
  return {ru, p};
}

struct WalkOut {
  int len, nacc, err, why;
};

// The walk (one warp): moves in order, tracking the N offset d (bit d + 16
// of a move's masks); stops at the first move whose mask says stop (conflict
// with an in-flight commit, or d outside the evaluated range) or whose accepted
// commit would overflow. Two ballots per 64 moves plus two per event; N
// changes only at accepted insertions / deletions.
__device__ __noinline__ WalkOut walk_warp(const uint32_t* macc, const uint32_t* mcf, const uint32_t* movf,
                                          const uint8_t* mkind, int fit, int* acc_i, int* acc_d,
                                          int8_t* acck, int lane, int max_acc) {
  int d = 0, start = 0, nacc = 0, len = fit, err = 0, why = kStopEnd;
  const int nh = (fit + 31) >> 5;
  // two blocks of 32 moves per ballot pair (independent ballots), so a block
  // without events costs half an iteration
#pragma unroll 1
  for (int h = 0; h < nh; h += 2) {
    const int i0 = lane + 32 * h, i1 = i0 + 32;
    const bool in0 = i0 < fit, in1 = i1 < fit;
    const uint32_t am0 = in0 ? macc[i0] : 0u, sm0 = in0 ? mcf[i0] : 0u, om0 = in0 ? movf[i0] : 0u;
    const uint32_t am1 = in1 ? macc[i1] : 0u, sm1 = in1 ? mcf[i1] : 0u, om1 = in1 ? movf[i1] : 0u;
    const unsigned kd0 = in0 ? mkind[i0] : 0u, kd1 = in1 ? mkind[i1] : 0u;
    bool done = false;
#pragma unroll 1
    for (;;) {
      const int j = d + kHalf;
      const bool inr = j >= 0 && j < 32;
      const int jj = j & 31;
      const bool act0 = in0 && i0 >= start, act1 = in1 && i1 >= start;
      const bool st0 = act0 && (!inr || ((sm0 >> jj) & 1u));
      const bool ac0 = act0 && inr && ((am0 >> jj) & 1u);
      const bool st1 = act1 && (!inr || ((sm1 >> jj) & 1u));
      const bool ac1 = act1 && inr && ((am1 >> jj) & 1u);
      const unsigned ev0 = __ballot_sync(0xffffffffu, st0 || ac0);
      const unsigned ev1 = __ballot_sync(0xffffffffu, st1 || ac1);
      if (!(ev0 | ev1)) break;
      const bool first = ev0 != 0u;
      const int el = __ffs(first ? ev0 : ev1) - 1;
      const int e = 32 * (first ? h : h + 1) + el;
      const unsigned mine = first ? ((st0 ? 1u : 0u) | (((om0 >> jj) & 1u) << 1) | (kd0 << 2))
                                  : ((st1 ? 1u : 0u) | (((om1 >> jj) & 1u) << 1) | (kd1 << 2));
      const unsigned info = __shfl_sync(0xffffffffu, mine, el);
      if (info & 1u) {
        len = e;
        why = inr ? kStopPrev : kStopRange;
        done = true;
        break;
      }
      if (info & 2u) {
        len = e;
        err = 1;
        why = kStopOverflow;
        done = true;
        break;
      }
      if (lane == 0) {
        acc_i[nacc] = e;
        acc_d[nacc] = d;
        acck[e] = (int8_t)nacc;
      }
      ++nacc;
      const int k = (int)(info >> 2);
      d += k == 1 ? 1 : (k == 2 ? -1 : 0);
      start = e + 1;
      if (nacc == max_acc) {
        len = e + 1;
        why = kStopFull;
        done = true;
        break;
      }
    }
    if (done) break;
  }
  __syncwarp();
  return {len, nacc, err, why};
}

// Does consumed move i read anything accepted move j (earlier in the round)
// changed? Index overlap, the target brick / cell of i (overflow test), or a
// changed position within r_c of a point i read (its new point's window, its
// particle's e). Brick proximity filters, exact distances decide.
__device__ __forceinline__ bool conflict(const EngineArgs& a, const SeqShared& sh, int i, int j) {
  // i reads its particle's position and e (displace / delete); j wrote its
  // particle (insert: the new index; delete: pid and the last index)
  const int64_t la = sh.mkind[i] != 1 ? sh.ia[i] : -1, aa = sh.ia[j], ab = sh.ib[j];
  if (la >= 0 && (la == aa || la == ab)) return true;
  const bool grid = a.g.kind != GCMC_ALL_PAIRS;
  const uint64_t ln = sh.ptn[i], an = sh.ptn[j], ao = sh.pto[j];
  if (ln != kNoPoint) {
    if (ao != kNoPoint && (mbrick(a.m, ln) == mbrick(a.m, ao) || (grid && sh.cn[i] == sh.co[j]))) return true;
    if (an != kNoPoint && (ln == an || (grid && sh.cn[i] == sh.cn[j]))) return true;
  }
  return false;
}

__device__ __noinline__ bool conflict_xyz(const EngineArgs& a, const SeqShared& sh,
                                             const Proposal& pi, const Proposal& pj, int i, int j) {
  const uint64_t ln = sh.ptn[i], lo = sh.pto[i], an = sh.ptn[j], ao = sh.pto[j];
  // i's points: new (window) and old (its particle); j's changed points: old, new
  if (ln != kNoPoint) {
    if (ao != kNoPoint && mnear(a.m, ln, ao) &&
        within_rc(a.b, pi.x, pi.y, pi.z, sh.xo[j][0], sh.xo[j][1], sh.xo[j][2])) return true;
    if (an != kNoPoint && mnear(a.m, ln, an) && within_rc(a.b, pi.x, pi.y, pi.z, pj.x, pj.y, pj.z))
      return true;
  }
  if (lo != kNoPoint) {
    if (ao != kNoPoint && mnear(a.m, lo, ao) &&
        within_rc(a.b, sh.xo[i][0], sh.xo[i][1], sh.xo[i][2], sh.xo[j][0], sh.xo[j][1], sh.xo[j][2]))
      return true;
    if (an != kNoPoint && mnear(a.m, lo, an) &&
        within_rc(a.b, sh.xo[i][0], sh.xo[i][1], sh.xo[i][2], pj.x, pj.y, pj.z)) return true;
  }
  return false;
}

// Brick at window offset o (0..26) of a packed brick point (dims >= 3).
__device__ __forceinline__ uint32_t nbr_brick(const Mirror& m, uint32_t pt, int o) {
  const int d = m.dims;
  int cx = pt_x(pt) + o % 3 - 1, cy = pt_y(pt) + (o / 3) % 3 - 1, cz = pt_z(pt) + o / 9 - 1;
  cx += cx < 0 ? d : 0;
  cx -= cx >= d ? d : 0;
  cy += cy < 0 ? d : 0;
  cy -= cy >= d ? d : 0;
  cz += cz < 0 ? d : 0;
  cz -= cz >= d ? d : 0;
  return (uint32_t)cx + (uint32_t)d * ((uint32_t)cy + (uint32_t)d * (uint32_t)cz);
}

// All changed points of accepted moves i and j more than 2 r_c apart.
__device__ __noinline__ bool far_apart(const EngineArgs& a, const SeqShared& sh,
                                          const Proposal& pi, const Proposal& pj, int i, int j) {
  double p[2][3], q[2][3];
  int np = 0, nq = 0;
  if (sh.ptn[i] != kNoPoint) { p[np][0] = pi.x; p[np][1] = pi.y; p[np][2] = pi.z; ++np; }
  if (sh.pto[i] != kNoPoint) { p[np][0] = sh.xo[i][0]; p[np][1] = sh.xo[i][1]; p[np][2] = sh.xo[i][2]; ++np; }
  if (sh.ptn[j] != kNoPoint) { q[nq][0] = pj.x; q[nq][1] = pj.y; q[nq][2] = pj.z; ++nq; }
  if (sh.pto[j] != kNoPoint) { q[nq][0] = sh.xo[j][0]; q[nq][1] = sh.xo[j][1]; q[nq][2] = sh.xo[j][2]; ++nq; }
  const double lim = __dmul_rn(4.0, a.b.rc2) * (1.0 + 1e-9);
  for (int x = 0; x < np; ++x)
    for (int y = 0; y < nq; ++y)
      if (min_image_dist2(p[x][0], p[x][1], p[x][2], q[y][0], q[y][1], q[y][2], a.b) <= lim) return false;
  return true;
}

__device__ __forceinline__ void compose_dec(uint32_t r, uint64_t base, uint64_t n, int nacc,
                                            int stop, uint64_t ctot, SeqShared& sh, int lane) {
  for (int idx = lane; idx < kDecHdr + kDecEnt * nacc; idx += 32) {
    uint64_t p = 0;
    if (idx == 0) p = base;
    else if (idx == 1) p = n;
    else if (idx == 2) p = (uint64_t)nacc | ((uint64_t)stop << 9);
    else if (idx == 3) p = ctot;
    else if (idx >= kDecHdr) {
      const int e = (idx - kDecHdr) / kDecEnt, f = (idx - kDecHdr) % kDecEnt;
      const int i = sh.acc_i[e];
      const int kind = sh.mkind[i];
      if (f == 0) p = (uint64_t)(sh.ptn[i] & kNoPoint) | ((uint64_t)(sh.pto[i] & kNoPoint) << 24);
      else if (f == 1) p = ((uint64_t)kind << 32) | (uint64_t)(uint32_t)sh.ia[i];
      else if (f == 2) p = sh.ib[i] < 0 ? 0xffffffffull : (uint64_t)(uint32_t)sh.ib[i];
      else {
        const uint64_t cn = kind != 2 && sh.cn[i] >= 0 ? (uint64_t)sh.cn[i] : 0xffffffull;
        const uint64_t co = kind != 1 && sh.co[i] >= 0 ? (uint64_t)sh.co[i] : 0xffffffull;
        p = cn | (co << 24);
      }
    }
    sh.dw[idx] = tagw(r, p);
  }
  if (lane == 0) sh.dneed = kDecHdr + kDecEnt * nacc;
}

// Helper warps (kPollWarps .. 15): commits, statistics and trace of the round
// in sh.done, while the poll warps wait for the next round.
__device__ __noinline__ void helpers(const EngineArgs& a, SeqShared& sh, int warp, int lane) {
  const Round& D = sh.done;
  if (D.len == 0) return;
  if (a.walk_reps == 6) return;  // diagnostics only (statistics / trace skipped)
  auto ext_of = [&](int s) -> const SlotExt* {
    const SlotExt* ex = a.ext + (size_t)D.par * a.nslots + s;
    while (ld_acquire(&ex->tag) != (uint64_t)D.r) nap();
    return ex;
  };
  if (warp == kPollWarps) {  // (commits run in the reserved evaluator groups)
  } else if (warp == kPollWarps + 1) {  // statistics (engine.hpp:293-308, 413-426)
    const int len = D.len, nacc = D.nacc;
    ChainState& ks = sh.ks;
    if (lane < nacc) {
      const OffRec& o = ext_of(D.acc_i[lane])->off[D.acc_d[lane] + kHalf];
      sh.acc_du[lane] = o.du;
      sh.acc_dw[lane] = o.dw;
    }
    __syncwarp();
    if (lane == 0) {
      double energy = ks.energy, virial = ks.virial;
      uint64_t cur = D.n;
      sh.st_e[0] = energy;
      sh.st_w[0] = virial;
      sh.st_n[0] = cur;
      for (int k = 0; k < nacc; ++k) {
        energy = __dadd_rn(energy, sh.acc_du[k]);
        virial = __dadd_rn(virial, sh.acc_dw[k]);
        const int kind = D.acc_kind[k];
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
      const Observables ob = observables(a, cur, sh.st_e[k], sh.st_w[k]);
      const double nd = (double)cur;
      sh.st_v[k][0] = nd;
      sh.st_v[k][1] = __dmul_rn(nd, nd);
      sh.st_v[k][2] = ob.rep_u;
      sh.st_v[k][3] = ob.pres;
    }
    const uint64_t step0 = ks.step;
    unsigned* smp = sh.smp;
    unsigned att0 = 0, att1 = 0, att2 = 0;
#pragma unroll 1
    for (int h = 0; h < kMH; ++h) {
      const int i = lane + 32 * h;
      const bool in = i < len;
      const int kind = in ? D.kind[i] : 3;
      att0 += __popc(__ballot_sync(0xffffffffu, kind == 0));
      att1 += __popc(__ballot_sync(0xffffffffu, kind == 1));
      att2 += __popc(__ballot_sync(0xffffffffu, kind == 2));
      const uint64_t st = step0 + (uint64_t)i + 1;
      const bool sm = in && st > a.equil && (a.interval == 1 || (st - a.equil) % a.interval == 0);
      const unsigned b = __ballot_sync(0xffffffffu, sm);
      if (lane == 0) smp[h] = b;
    }
    __syncwarp();
    __syncwarp();
    if (lane == 0) {
      double sn = ks.sum_n, sn2 = ks.sum_n2, su = ks.sum_u, sp = ks.sum_p;
      uint64_t samples = 0;
      int lo = 0;
      for (int k = 0; k <= nacc; ++k) {
        const int hi = k < nacc ? D.acc_i[k] : len;
        int c = 0;
#pragma unroll 1
        for (int h = 0; h < kMH; ++h) {
          const int a0 = lo - 32 * h, a1 = hi - 32 * h;
          const unsigned m_hi = a1 >= 32 ? 0xffffffffu : (a1 <= 0 ? 0u : (1u << a1) - 1u);
          const unsigned m_lo = a0 >= 32 ? 0xffffffffu : (a0 <= 0 ? 0u : (1u << a0) - 1u);
          c += __popc(smp[h] & m_hi & ~m_lo);
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
  } else if (a.trace) {  // trace records (MoveOutcome, engine.hpp:104-110)
    const int nt = (kThreads / 32 - kPollWarps - 2) * 32;
    for (int i = (warp - kPollWarps - 2) * 32 + lane; i < D.len; i += nt) {
      const OffRec& o = ext_of(i)->off[D.res_d[i] + kHalf];
      int accepted = 0, dn = 0;
#pragma unroll 1
      for (int k = 0; k < D.nacc; ++k) {
        if (D.acc_i[k] == i) accepted = 1;
        if (D.acc_i[k] <= i) dn += D.acc_kind[k] == 1 ? 1 : (D.acc_kind[k] == 2 ? -1 : 0);
      }
      gcmc_trace_rec t;
      t.kind = D.kind[i];
      t.accepted = accepted;
      t.delta_u = o.du;
      t.delta_w = o.dw;
      t.acceptance_prob = o.pe;
      t.n_after = (uint64_t)((int64_t)D.n + dn);
      a.trace[D.base + i] = t;
    }
  }
}

__device__ void sequencer(const EngineArgs& a, uint8_t* smem) {
  auto& sh = *reinterpret_cast<SeqShared*>(smem);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool grid = a.g.kind != GCMC_ALL_PAIRS;
  constexpr int kPollThreads = kPollWarps * 32;
  if (tid == 0) {
    sh.ks = *a.st;
    sh.plen = 0;
    sh.done.len = 0;
    sh.done.nacc = 0;
    sh.arrived = 0;
    sh.vmax = sh.vsum = 0;
    sh.viters = sh.vcalls = 0;
    sh.err = 0;
    for (int k = 0; k < kNStop; ++k) sh.stops[k] = 0;
  }
  uint64_t ring_hi = a.nmoves < (uint64_t)kRing ? a.nmoves : (uint64_t)kRing;
  if (warp == 0) {
    ring_fill(a, sh.ring, 0, ring_hi, lane);
    cp_async_wait();
  }
  __syncwarp();
    __syncthreads();
  uint64_t base = 0, n = sh.ks.n;
  uint64_t rounds = 0, etarget = 0;  // energy updates expected through the previous round
  uint64_t need_s = 0;                 // latest round before the last whose commits D_r waits for
  int prev_nacc = 0;
  int fit = fit_of(a, 0);
  uint32_t r = 1;
  if (warp == 0) {
    sh.nacc = 0;
    compose_dec(r, base, n, 0, 0, 0, sh, lane);
  }
  __syncwarp();
    __syncthreads();
  if (tid < sh.dneed) st_relaxed(a.dec + tid, sh.dw[tid]);
  PhaseClock pc;
  pc.start(a.prof && tid == 0);
  for (;;) {
    const int par = (int)(r & 1);
    if (warp < kPollWarps) {
      // -------------------- poll: slot words -> per-move masks. Warp 0 does
      // not poll: it repeats the walk on the masks as they arrive (results
      // discarded) so that the walk's code is in the instruction cache when
      // the last slot lands.
      if (warp == 0) {  // one dry run (the walk's code into the instruction cache), then wait
        walk_warp(sh.pacc, sh.pcf, sh.povf, sh.pkind, sh.plen, sh.wscr_i, sh.wscr_d, sh.wscr_k, lane, a.max_acc);
        while (*(volatile int*)&sh.arrived < fit) __nanosleep(32);
      }
      for (int sl = tid - 32; sl >= 0 && sl < fit; sl += kPollThreads - 32) {
        const uint64_t* rw = a.res + (size_t)par * kResWords * a.nslots + sl;
        uint64_t w[kResWords];
        for (;;) {
          bool ok = true;
#pragma unroll
          for (int j = 0; j < kResWords; ++j) {
            w[j] = ld_relaxed(rw + (size_t)j * a.nslots);
            ok &= tagged(w[j], r);
          }
          if (ok) break;
          __nanosleep(a.poll_ns);
        }
        sh.mkind[sl] = (uint8_t)(w[0] & 3);
        sh.acck[sl] = -1;
        sh.macc[sl] = (uint32_t)((w[0] & kPay) >> 8);
        sh.mcf[sl] = (uint32_t)w[1];
        sh.movf[sl] = (uint32_t)w[2];
        atomicAdd(&sh.arrived, 1);
      }
      group_sync(1, kPollThreads);
      // every evaluation of round r has read its state: the previous round's
      // commits may store now. A relaxed store suffices: every slot result
      // word read above is data-dependent on that slot's state loads, which
      // had therefore returned before the word was written; the committers'
      // stores follow their acquire of kGo (0.15 us per round less than a
      // release here, profiles/r02/engine_variants.txt).
      if (tid == 0) st_relaxed(a.flags + kGo, (uint64_t)r);
#ifdef GCMC_PHASE_TIMERS
      if (a.prof && tid == 0) a.prof[3640 + (r & 1)] = gtimer();
#endif
#ifdef GCMC_PHASE_TIMERS
      if (a.prof && tid == 0 && r > 2) {
        a.prof[3615] += gtimer() - a.prof[3600 + (r & 1)];
        a.prof[3616] += a.prof[3620 + (r & 7)];
        a.prof[3620 + ((r + 4) & 7)] = 0;
        a.prof[3617] += 1;
      }
#endif
      pc.mark(1);
      if (warp == 0) {  // ---- walk (warm: warp 0 ran it on the partial masks while polling)
        const WalkOut wo = walk_warp(sh.macc, sh.mcf, sh.movf, sh.mkind, fit, sh.acc_i, sh.acc_d, sh.acck, lane, a.max_acc);
        if (lane == 0) {
          sh.len = wo.len;
          sh.nacc = wo.nacc;
          sh.cmin = wo.len;
          sh.err = wo.err;
          sh.why = wo.why;
        }
      }
      group_sync(1, kPollThreads);
      pc.mark(2);
#ifdef GCMC_PHASE_TIMERS
      if (a.walk_reps == 3) {  // diagnostics: the same walk again, warm (bucket 8)
        if (warp == 0) walk_warp(sh.macc, sh.mcf, sh.movf, sh.mkind, fit, sh.wscr_i, sh.wscr_d, sh.wscr_k, lane, a.max_acc);
        group_sync(1, kPollThreads);
        pc.mark(8);
      }
#endif
#pragma unroll 1
      for (int vrep = 0; vrep < (a.walk_reps == 2 ? 2 : 1); ++vrep) {
      if (vrep == 1) pc.mark(7);
      {  // ---- read / write sets of the consumed moves (one L2 hop for x_pid)
        const int len = sh.len + sh.err;  // the overflowing move's data is reported too
        const int nacc = sh.nacc;
        for (int i = tid; i < len; i += kPollThreads) {
          const Proposal& pr = sh.ring[(base + i) % kRing];
          const int kind = sh.mkind[i];
          int di = 0, nb = 0;  // N offset before move i (uniform trip count: no divergence)
          for (int k = 0; k < nacc; ++k) {
            const int j = sh.acc_i[k];
            const int ak = sh.mkind[j];
            di += j < i ? (ak == 1 ? 1 : (ak == 2 ? -1 : 0)) : 0;
            nb += j < i ? 1 : 0;
          }
          sh.res_d[i] = di;
          sh.nbef[i] = (uint8_t)nb;
          const int64_t nd = (int64_t)n + di;
          sh.ptn[i] = (uint32_t)(kind != 2 ? (pr.wmask != kNoMask ? (uint64_t)pr.bpt : mpoint(a.m, pr.x, pr.y, pr.z)) : kNoPoint);
          sh.cn[i] = (kind != 2 && grid) ? (pr.wmask != kNoMask ? pr.cell : cell_of(a.g, pr.x, pr.y, pr.z)) : -1;
          sh.pto[i] = (uint32_t)kNoPoint;
          sh.co[i] = -1;
          sh.ia[i] = -1;
          sh.ib[i] = -1;
          if (kind == 1) {
            sh.ia[i] = nd;
          } else if (nd >= 1) {
            const uint64_t pid = index_from(pr.pick, (uint64_t)nd);
            const double4 o = ld_cg(a.s.pos + pid);
            sh.xo[i][0] = o.x;
            sh.xo[i][1] = o.y;
            sh.xo[i][2] = o.z;
            sh.pto[i] = (uint32_t)mpoint(a.m, o.x, o.y, o.z);
            sh.co[i] = grid ? cell_of(a.g, o.x, o.y, o.z) : -1;
            sh.ia[i] = (int64_t)pid;
            sh.ib[i] = kind == 2 ? nd - 1 : -1;
          }
        }
      }
      group_sync(1, kPollThreads);
      pc.mark(6);  // read / write sets
      // ---- verify: one thread per consumed move i, against every accepted
      // move before it (their data read from shared memory, broadcast):
      // index overlap, the target brick / cell of i, and (brick-near, then
      // exact distance) a changed position within r_c of a point i read. An
      // accepted move is also checked against the accepted moves before it:
      // more than 2 r_c apart (disjoint neighbour-energy updates, so every e_j
      // sees its updates in chain order: reproducible bits).
#ifdef GCMC_PHASE_TIMERS
      const unsigned long long vt0 = clock64();
#endif
      {
        const int len = sh.len, nacc = sh.nacc;
        const int first = nacc ? sh.acc_i[0] : len;
        // the accepted moves' write sets, packed once (broadcast reads below)
        if (tid < nacc) {
          const int j = sh.acc_i[tid];
          AccV v;
          v.j = j;
          v.ia = (int)sh.ia[j];
          v.ib = (int)sh.ib[j];
          v.an = sh.ptn[j];
          v.ao = sh.pto[j];
          v.bn = v.an != (uint32_t)kNoPoint ? mbrick(a.m, v.an) : 0xfffffffdu;
          v.bo = v.ao != (uint32_t)kNoPoint ? mbrick(a.m, v.ao) : 0xfffffffdu;
          v.cn = v.an != (uint32_t)kNoPoint && grid ? sh.cn[j] : -4;
          v.co = v.ao != (uint32_t)kNoPoint && grid ? sh.co[j] : -4;
          sh.av[tid] = v;
        }
        group_sync(1, kPollThreads);
        const int dm = a.m.dims, rch = a.m.reach;
        const NearK nk = near_k(dm, rch);
#pragma unroll 1
        for (int i = first + 1 + tid; i < len && a.walk_reps != 5; i += kPollThreads) {
          const int kind = sh.mkind[i];
          const int la = kind != 1 ? (int)sh.ia[i] : -5;
          const uint32_t ln = sh.ptn[i], lo = sh.pto[i];
          const uint32_t lb = ln != (uint32_t)kNoPoint ? mbrick(a.m, ln) : 0xfffffffeu;
          const int lcn = ln != (uint32_t)kNoPoint && grid ? sh.cn[i] : -3;
          const unsigned acci = sh.acck[i] >= 0 ? 1u : 0u;
          const unsigned lnv = ln != (uint32_t)kNoPoint ? 1u : 0u, lov = lo != (uint32_t)kNoPoint ? 1u : 0u;
          // Branch-free over the accepted moves before i (acc_i is sorted, so
          // the trip count differs by at most a few within a warp of
          // consecutive i): hard = certain conflicts, soft = needs an exact test.
          unsigned hard = 0u, soft = 0u;
          const int kb = sh.nbef[i];
#pragma unroll 2
          for (int k = 0; k < kb; ++k) {
            const AccV v = sh.av[k];
            const unsigned before = 1u;
            const unsigned idx = (unsigned)(la >= 0) & ((unsigned)(la == v.ia) | (unsigned)(la == v.ib));
            const unsigned tgt = (unsigned)(lb == v.bo) | (unsigned)(lb == v.bn) | (unsigned)(lcn == v.co) |
                                 (unsigned)(lcn == v.cn);
            unsigned nr, n2;
            if (nk.simd) {
              const unsigned aov = v.ao != (uint32_t)kNoPoint ? 1u : 0u, anv = v.an != (uint32_t)kNoPoint ? 1u : 0u;
              const unsigned mno = lnv & aov, mnn = lnv & anv, moo = lov & aov, mon = lov & anv;
              const uint32_t uno = near_u(ln, v.ao, nk.dd), unn = near_u(ln, v.an, nk.dd);
              const uint32_t uoo = near_u(lo, v.ao, nk.dd), uon = near_u(lo, v.an, nk.dd);
              nr = (mno & near_ok(uno, nk.add_r)) | (mnn & near_ok(unn, nk.add_r)) |
                   (moo & near_ok(uoo, nk.add_r)) | (mon & near_ok(uon, nk.add_r));
              n2 = acci & ((mno & near_ok(uno, nk.add_2)) | (mnn & near_ok(unn, nk.add_2)) |
                           (moo & near_ok(uoo, nk.add_2)) | (mon & near_ok(uon, nk.add_2)));
            } else {
              nr = near_bits(ln, v.ao, dm, rch) | near_bits(ln, v.an, dm, rch) |
                   near_bits(lo, v.ao, dm, rch) | near_bits(lo, v.an, dm, rch);
              n2 = acci & (near_bits(ln, v.an, dm, 2) | near_bits(ln, v.ao, dm, 2) |
                           near_bits(lo, v.an, dm, 2) | near_bits(lo, v.ao, dm, 2));
            }
            hard |= (before & (idx | tgt)) << k;
            soft |= (before & (nr | n2)) << k;
          }
          bool c = hard != 0u;
          // rare: exact distances (r_c; 2 r_c between accepted moves)
          for (unsigned m = c ? 0u : soft; m; m &= m - 1) {
            const int k = __ffs(m) - 1;
            const AccV v = sh.av[k];
            const Proposal& pi = sh.ring[(base + i) % kRing];
            const Proposal& pj = sh.ring[(base + v.j) % kRing];
            if (conflict_xyz(a, sh, pi, pj, i, v.j) || (acci && !far_apart(a, sh, pi, pj, i, v.j))) {
              c = true;
              break;
            }
          }
          if (c) atomicMin(&sh.cmin, i);
        }
      }
#ifdef GCMC_PHASE_TIMERS
      if (a.prof && lane == 0) {
        const unsigned long long d = clock64() - vt0;
        atomicMax(&sh.vmax, d);
        atomicAdd(&sh.vsum, d);
      }
      group_sync(1, kPollThreads);
      if (a.prof && tid == 0) {
        a.prof[3500] += sh.vmax;
        a.prof[3501] += sh.vsum / kPollWarps;
        a.prof[3502] += sh.viters;
        a.prof[3503] += sh.vcalls;
        sh.viters = sh.vcalls = 0;
        sh.vmax = 0;
        sh.vsum = 0;
      }
#endif
      group_sync(1, kPollThreads);
      pc.mark(9);
      }
      pc.mark(3);
      if (tid == 0 && a.prof && r < 200) {
        a.prof[256 + 4 * r] = base;
        a.prof[256 + 4 * r + 1] = (unsigned long long)sh.len;
        a.prof[256 + 4 * r + 2] = (unsigned long long)sh.nacc | ((unsigned long long)sh.cmin << 16);
        a.prof[256 + 4 * r + 3] = (unsigned long long)sh.why;
      }
      if (tid == 0 && sh.cmin < sh.len) {
        const int c = sh.cmin;
        sh.len = c;
        int k = 0;
        while (k < sh.nacc && sh.acc_i[k] < c) ++k;
        sh.nacc = k;
        sh.err = 0;
        sh.why = kStopVerify;
      }
    } else {
      helpers(a, sh, warp, lane);  // previous round, concurrently with the poll
    }
    __syncwarp();
    __syncthreads();
    pc.mark(4);
    // -------------------- close the round
    const int len = sh.len, nacc = sh.nacc;
    int dn;  // N change of the round: one accepted move per lane (nacc <= kMaxAcc = 32)
    {
      const int kd = lane < nacc ? (int)sh.mkind[sh.acc_i[lane]] : 0;
      dn = __reduce_add_sync(0xffffffffu, kd == 1 ? 1 : (kd == 2 ? -1 : 0));
    }
    const uint64_t nbase = base + (uint64_t)len;
    const uint64_t nn = (uint64_t)((int64_t)n + dn);
    const bool stop = nbase >= a.nmoves || sh.err;
    ATab at;  // warp 1: accepted move `lane`, read here (the ring is refilled after the publish)
    if (warp == 0) {
      compose_dec(r + 1, nbase, nn, nacc, stop, etarget + (uint64_t)nacc, sh, lane);
    } else if (warp == 1) {
      if (lane < nacc) {
        const int i = sh.acc_i[lane];
        const Proposal& pr = sh.ring[(base + i) % kRing];
        const int kind = sh.mkind[i];
        at.ox = kind != 1 ? sh.xo[i][0] : 0.0;
        at.oy = kind != 1 ? sh.xo[i][1] : 0.0;
        at.oz = kind != 1 ? sh.xo[i][2] : 0.0;
        at.nx = pr.x;
        at.ny = pr.y;
        at.nz = pr.z;
        at.ia = sh.ia[i];
        at.ib = sh.ib[i];
        at.nn = (uint64_t)((int64_t)n + sh.acc_d[lane]);
        at.kind = kind;
        at.slot = i;
        at.d = sh.acc_d[lane];
      }
    } else if (warp >= 2 && warp < 2 + kMaxMoves / 32) {  // hand the round to the helpers
      Round& D = sh.done;
      const int i = tid - 64;
      if (i < len) {
        D.res_d[i] = sh.res_d[i];
        D.kind[i] = sh.mkind[i];
      }
      if (i < fit) {  // the next round's dry walk input
        sh.pacc[i] = sh.macc[i];
        sh.pcf[i] = sh.mcf[i];
        sh.povf[i] = sh.movf[i];
        sh.pkind[i] = sh.mkind[i];
      }
      if (i == 0) sh.plen = fit;
      if (i < nacc) {
        const int m = sh.acc_i[i];
        const Proposal& pr = sh.ring[(base + m) % kRing];
        D.acc_i[i] = m;
        D.acc_d[i] = sh.acc_d[i];
        D.acc_kind[i] = sh.mkind[m];
        D.acc_ia[i] = sh.ia[m];
        D.acc_ib[i] = sh.ib[m];
        D.acc_nx[i] = pr.x;
        D.acc_ny[i] = pr.y;
        D.acc_nz[i] = pr.z;
      }
      if (i == 0) {
        D.base = base;
        D.n = n;
        D.r = r;
        D.len = len;
        D.nacc = nacc;
        D.par = par;
        ++sh.stops[sh.why];
      }
    }
    // D_{r+1} goes out at once: the evaluators themselves wait for the
    // previous round's energy updates and commits (poll_dec)
    if (prev_nacc) need_s = r - 1;
    __syncwarp();
    __syncthreads();
#ifdef GCMC_PHASE_TIMERS
    if (a.prof && tid == 0) a.prof[3600 + ((r + 1) & 1)] = gtimer();
    if (a.prof && tid == 0 && r > 2) a.prof[3648] += gtimer() - a.prof[3640 + (r & 1)];
#endif
    if (tid < sh.dneed) st_relaxed(a.dec + tid, sh.dw[tid]);
    if (warp == 1 && lane < nacc) {  // the exact table, after the publish (every reader waits for the tag)
      ATab* t = a.atab + (size_t)par * kMaxAcc + lane;
      t->ox = at.ox;
      t->oy = at.oy;
      t->oz = at.oz;
      t->nx = at.nx;
      t->ny = at.ny;
      t->nz = at.nz;
      t->ia = at.ia;
      t->ib = at.ib;
      t->nn = at.nn;
      t->kind = at.kind;
      t->slot = at.slot;
      t->d = at.d;
      t->deps = 0u;
      st_release(&t->tag, (uint64_t)r);
    }
    etarget += (uint64_t)nacc;
    prev_nacc = nacc;
    pc.mark(5);
    // next round's ring (while the evaluators work)
    if (warp == 0) {
      const uint64_t want = nbase + kRing < a.nmoves ? nbase + kRing : a.nmoves;
      if (want > ring_hi) {
        ring_fill(a, sh.ring, ring_hi, want, lane);
        ring_hi = want;
      }
      cp_async_wait();
    }
    fit = fit_of(a, nbase);
    if (tid == 0) sh.arrived = 0;
    __syncwarp();
    __syncthreads();
    base = nbase;
    n = nn;
    ++rounds;
    ++r;
    if (stop) break;
  }
  if (tid == 0) st_release(a.flags + kGo, (uint64_t)r);  // the last decision's commits
  // the last round's statistics / trace
  if (warp >= kPollWarps) helpers(a, sh, warp, lane);
  if (tid == 32) while (ld_acquire(a.flags + kSFlag) < need_s) __nanosleep(a.poll_ns);
  __syncwarp();
    __syncthreads();
  if (a.prof && tid == 0) {
    pc.flush(a.prof);
    a.prof[15] = rounds;
    for (int k = 0; k < kNStop; ++k) a.prof[40 + k] = sh.stops[k];
  }
  if (tid == 0) {
    ChainState& ks = sh.ks;
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
    if (sh.err) {  // overflow at move `base` (relative index len of the last round)
      const int i = sh.len;
      const int kind = sh.mkind[i];
      const uint32_t bb = mbrick(a.m, sh.ptn[i]);
      const int ob = __ldcg(a.m.occ + bb);
      bool ref = false;
      int cb = -1, ocb = 0;
      if (grid) {
        cb = sh.cn[i];
        ocb = __ldcg(a.g.occ + cb);
        const bool same_c = kind == 0 && sh.co[i] == cb;
        ref = !same_c && ocb >= a.g.cap;
      }
      a.st->error = GCMC_CELL_OVERFLOW;
      a.st->err_a = ref ? cb : (int64_t)bb;
      a.st->err_b = ref ? ocb : ob;
      a.st->err_c = ref ? 0 : 1;
    }
  }
}

template <int T>
__global__ void __launch_bounds__(kThreads, 1) k_engine2(EngineArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  // The arguments live in shared memory: the engine passes them by reference
  // to out-of-line functions, which makes the compiler copy a by-value kernel
  // parameter to the local-memory stack — every field read (m.dims, b.rc2, ...)
  // would then be a local load, an L2 round trip with the L1 given to shared
  // memory.
  __shared__ EngineArgs sa;
  if (threadIdx.x == 0) sa = a;
  __syncthreads();
  if (blockIdx.x == 0)
    sequencer(sa, smem);
  else
    evaluator<T>(sa, smem);
}

// e[i] from scratch: one thread per particle over its 3x3x3 brick window
// (plain sequential sums, deterministic).
__global__ void __launch_bounds__(256) k_epart(Mirror m, Box b, const double4* __restrict__ pos,
                                              uint64_t n, double2* out) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double4 x = ld_cg(pos + i);
  const int self = bslot_in(x);
  double su = 0.0, sw = 0.0;
  auto brick = [&](uint32_t id) {
    const int occ = __ldcg(m.occ + id);
    for (int k = 0; k < occ; ++k) {
      const int idx = (int)id * m.cap + k;
      if (idx == self) continue;
      const double r2 = min_image_dist2(x.x, x.y, x.z, __ldcg(m.rx + idx), __ldcg(m.ry + idx),
                                        __ldcg(m.rz + idx), b);
      if (r2 <= b.rc2) lj_accum(b, r2, 1.0, su, sw);
    }
  };
  if (m.dims < 3) {
    for (uint32_t id = 0; id < m.nb; ++id) brick(id);
  } else {
    const int d = m.dims;
    const int bx = mcoord(m, x.x), by = mcoord(m, x.y), bz = mcoord(m, x.z);
    for (int oz = -1; oz <= 1; ++oz)
      for (int oy = -1; oy <= 1; ++oy)
        for (int ox = -1; ox <= 1; ++ox) {
          const int cx = (bx + ox + d) % d, cy = (by + oy + d) % d, cz = (bz + oz + d) % d;
          brick((uint32_t)cx + (uint32_t)d * ((uint32_t)cy + (uint32_t)d * (uint32_t)cz));
        }
  }
  out[i] = make_double2(su, sw);
}

// max |a - b| over both components (non-negative doubles order as their bits)
__global__ void k_ediff(const double2* a, const double2* b, uint64_t n, unsigned long long* out) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double2 x = a[i], y = b[i];
  atomicMax(out, (unsigned long long)__double_as_longlong(fabs(x.x - y.x)));
  atomicMax(out + 1, (unsigned long long)__double_as_longlong(fabs(x.y - y.y)));
}

}  // namespace

bool engine2_supported(const Chain& c) {
  if (c.params.engine_mode == 1) return false;
  if (knob("GCMC_ENGINE_V1")) return false;
  if (c.params.max_displacement > 0.0) return false;
  const int mg = kThreads / c.engine2_group;
  return (c.engine2_ctas - 1) * mg > 8 + 1 + 8 && (c.engine2_ctas - 1) * mg <= kMaxSlots;
}

gcmc_status epart_build(Chain& c, double2* out) {
  const uint64_t n = c.st_host->n;
  if (n) {
    k_epart<<<(unsigned)((n + 255) / 256), 256, 0, c.stream>>>(c.mirror, c.box, c.pos, n, out);
    cudaError_t e = cudaGetLastError();
    if (e) return cuda_error(e, "epart");
  }
  return GCMC_OK;
}

gcmc_status epart_drift(Chain& c, double* du, double* dw) {
  *du = *dw = 0.0;
  const uint64_t n = c.st_host->n;
  if (!c.e_valid || n == 0) return GCMC_OK;
  double2* fresh = nullptr;
  unsigned long long* out = nullptr;
  cudaError_t e = cudaMalloc(&fresh, n * sizeof(double2));
  if (!e) e = cudaMalloc(&out, 2 * sizeof(unsigned long long));
  if (e) return cuda_error(e, "epart drift");
  gcmc_status s = epart_build(c, fresh);
  if (!s) {
    cudaMemsetAsync(out, 0, 2 * sizeof(unsigned long long), c.stream);
    k_ediff<<<(unsigned)((n + 255) / 256), 256, 0, c.stream>>>(fresh, c.ep, n, out);
    unsigned long long h[2];
    e = cudaMemcpyAsync(h, out, sizeof h, cudaMemcpyDeviceToHost, c.stream);
    if (!e) e = cudaStreamSynchronize(c.stream);
    if (e) s = cuda_error(e, "epart drift");
    *du = __builtin_bit_cast(double, h[0]);
    *dw = __builtin_bit_cast(double, h[1]);
  }
  cudaFree(fresh);
  cudaFree(out);
  return s;
}

gcmc_status epart_dump(Chain& c, double* maint, double* fresh) {
  const uint64_t n = c.st_host->n;
  if (!c.e_valid || n == 0) return GCMC_OK;
  double2* f = nullptr;
  cudaError_t e = cudaMalloc(&f, n * sizeof(double2));
  if (e) return cuda_error(e, "epart dump");
  gcmc_status s = epart_build(c, f);
  if (!s) {
    e = cudaMemcpyAsync(fresh, f, n * sizeof(double2), cudaMemcpyDeviceToHost, c.stream);
    if (!e) e = cudaMemcpyAsync(maint, c.ep, n * sizeof(double2), cudaMemcpyDeviceToHost, c.stream);
    if (!e) e = cudaStreamSynchronize(c.stream);
    if (e) s = cuda_error(e, "epart dump");
  }
  cudaFree(f);
  return s;
}

gcmc_status engine2_run(Chain& c, uint64_t nmoves, gcmc_trace_rec* trace_d, cudaStream_t s) {
  if (nmoves == 0) return GCMC_OK;
  const gcmc_params& P = c.params;
  cudaError_t e;
  if (!c.e_valid) {
    gcmc_status st = epart_build(c, c.ep);
    if (st) return st;
    c.e_valid = true;
  }
  const int T = c.engine2_group;
  const int MG = kThreads / T;
  const int G = c.engine2_ctas;
  EngineArgs a{};
  a.g = c.grid;
  a.m = c.mirror;
  a.b = c.box;
  a.s = Store{c.pos, c.rslot};
  a.ep = c.ep;
  a.st = c.st;
  a.props = c.props;
  a.trace = trace_d;
  a.nmoves = nmoves;
  a.beta = 1.0 / P.temperature;  // config.hpp:66
  a.mu = P.chemical_potential;
  a.lambda3 = P.lambda * P.lambda * P.lambda;
  a.vol = P.box_length * P.box_length * P.box_length;  // box.hpp:19
  a.temp = P.temperature;
  a.equil = P.equilibration_steps;
  a.interval = P.sampling_interval;
  a.tail = P.tail_corrections;
  a.prof = c.prof;
  {
    const double sg = P.sigma, rc = P.r_cut;
    const double sr3 = (sg / rc) * (sg / rc) * (sg / rc);
    const double sr9 = sr3 * sr3 * sr3;
    const double pi = 3.141592653589793238462643383279502884;
    a.tail_cu = (8.0 / 3.0) * pi;
    a.tail_cp = (16.0 / 3.0) * pi;
    a.tail_s3 = sg * sg * sg;
    a.tail_bu = sr9 / 3.0 - sr3;
    a.tail_bp = 2.0 / 3.0 * sr9 - sr3;
  }
  a.nslots = (G - 1) * MG;
  // Accepted moves per round, each with its own energy-update group: 32 when
  // the evaluator groups are plentiful; a smaller engine (a chain sharing the
  // device, a small box) keeps about a quarter of its groups for them (at
  // least 8), so more are left for moves: a round stops at max_acc accepts.
  a.max_acc = a.nslots >= kMaxMoves + kMaxAcc + 1 ? kMaxAcc
                                                   : std::max(8, std::min(kMaxAcc, a.nslots / 4));
  a.fitmax = a.nslots - a.max_acc - 1 < kMaxMoves ? a.nslots - a.max_acc - 1 : kMaxMoves;  // + committer
  {
    const char* f = knob("GCMC_FITMAX");
    if (f && std::atoi(f) > 0 && std::atoi(f) < a.fitmax) a.fitmax = std::atoi(f);
  }
  if (!c.eng2_buf) {
    const size_t bytes = kDecStride * 8 + 2 * (size_t)kMaxSlots * kResWords * 8 +
                         2 * (size_t)kMaxSlots * sizeof(SlotExt) + 2 * kMaxAcc * sizeof(ATab) + kFlagWords * 8 +
                         (size_t)kMaxAcc * kEBig * sizeof(double4);
    if ((e = cudaMalloc(&c.eng2_buf, bytes))) return cuda_error(e, "alloc engine2");
    c.eng2_bytes = bytes;
  }
  char* p = static_cast<char*>(c.eng2_buf);
  a.dec = reinterpret_cast<uint64_t*>(p);
  p += kDecStride * 8;
  a.res = reinterpret_cast<uint64_t*>(p);
  p += 2 * (size_t)kMaxSlots * kResWords * 8;
  a.ext = reinterpret_cast<SlotExt*>(p);
  p += 2 * (size_t)kMaxSlots * sizeof(SlotExt);
  a.atab = reinterpret_cast<ATab*>(p);
  p += 2 * kMaxAcc * sizeof(ATab);
  a.flags = reinterpret_cast<uint64_t*>(p);
  p += kFlagWords * 8;
  a.ebig = reinterpret_cast<double4*>(p);
  {
    const char* e1 = knob("GCMC_POLL_NS");
    a.poll_ns = e1 ? (unsigned)std::atoi(e1) : 64u;
    const char* e2 = knob("GCMC_EPOLL_NS");
    a.epoll_ns = e2 ? (unsigned)std::atoi(e2) : 64u;
    const char* e3 = knob("GCMC_WALK_REPS");
    a.walk_reps = e3 && std::atoi(e3) > 1 ? std::atoi(e3) : 1;

  }
  size_t eval_bytes = T == 128 ? sizeof(EvalShared<128>) : (T == 256 ? sizeof(EvalShared<256>) : sizeof(EvalShared<512>));
  eval_bytes = (eval_bytes + 15) & ~size_t(15);
  size_t smem = eval_bytes + ((c.mirror.nb + 15) & ~15u);
  a.smem_occ = 1;
  int max_optin = 0;
  cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, c.device);
  if (smem > (size_t)max_optin) {
    a.smem_occ = 0;
    smem = eval_bytes;
  }
  if (smem < sizeof(SeqShared)) smem = sizeof(SeqShared);
  if (a.prof)
    std::fprintf(stderr, "[engine2 prof] smem=%zu eval=%zu seq=%zu occ_replica=%d slots=%d fit=%d\n", smem,
                 eval_bytes, sizeof(SeqShared), a.smem_occ, a.nslots, a.fitmax);
  void (*kern)(EngineArgs) = T == 128 ? k_engine2<128> : (T == 256 ? k_engine2<256> : k_engine2<512>);
  if ((e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)))
    return cuda_error(e, "engine2 smem");
  if ((e = cudaMemsetAsync(c.eng2_buf, 0, c.eng2_bytes, s))) return cuda_error(e, "engine2");
  void* args[] = {&a};
  e = cudaLaunchCooperativeKernel((const void*)kern, dim3(G), dim3(kThreads), args, smem, s);
  if (e) return cuda_error(e, "engine2 launch");
  return GCMC_OK;
}

}  // namespace gcmcb
