// Persistent on-device Metropolis loop: Simulation::step() x n
// (engine.hpp:293-308, 350-426), executed as exact multi-move speculation
// across the whole GPU.
//
// Why speculation is exact. Every move's random draws are fixed before its ΔE
// is known (engine.hpp:207-213, 352-354), so proposals are precomputed
// (gen.cu). Only two things couple a move to its predecessors: the state its
// ΔE reads, and N, which picks the particle (pid = index_from(pick, N)) and
// enters the exchange acceptance ratios. A round evaluates a window of
// upcoming moves against the current state S in parallel — pid-based moves
// once per candidate N ("variant") — then a single sequencer walks the window
// in order, tracking N, and keeps the longest prefix in which every move's
// evaluation provably equals what the serial chain computes:
//   * the variant for the move's true N was evaluated,
//   * no earlier accepted move of this round, and no move committed in the
//     previous round (whose stores may still be in flight), changed anything
//     the evaluation read: no changed position within reach of its windows,
//     no changed particle slot it loaded (mirror.cuh, conflict()).
// Every decision in that prefix is the reference's decision; the first move
// that fails the test starts the next round. Accepted moves of one round are
// pairwise independent, so their commits (commit.cuh) run concurrently.
//
// Roles (one persistent CTA per SM, cooperative launch):
//   CTA 0        sequencer: polls the slot results of round r, walks, verifies,
//                publishes decision D_{r+1}; helper warps commit round r's
//                accepted moves, do the RunStatistics bookkeeping (same
//                sequential double adds as Simulation::sample) and the trace
//                while round r+1 is being evaluated.
//   CTAs 1..G-1  evaluators: MG groups of T threads, one slot (move, variant)
//                per group per round (slot.cuh), against a shared-memory
//                replica of the mirror occupancy.
// Communication is through L2 with self-validating tagged 64-bit words
// (round tag in the top 16 bits, payload below), so neither side needs a
// fence on the critical path; the one release/acquire pair orders the
// commits before the next-but-one round reads them.
#include <cstdlib>

#ifndef GCMC_KMAXMOVES
#define GCMC_KMAXMOVES 64
#endif
#include "commit.cuh"
#include <cstdio>
#include "internal.h"
#include "slot.cuh"
#include "sync.cuh"

namespace gcmcb {

namespace {

constexpr int kThreads = 512;
constexpr int kMaxMoves = GCMC_KMAXMOVES;   // moves per round
constexpr int kMH = kMaxMoves / 32;  // moves per walk lane
constexpr int kMaxAcc = 32;      // accepted moves per round
constexpr int kRing = GCMC_KMAXMOVES * 4;       // proposal ring (moves)
constexpr int kPre = 2 * kMaxMoves + 2;  // slot prefix entries
constexpr int kDecHdr = 4;
constexpr int kDecEnt = 2;
constexpr int kDecWords = kDecHdr + kDecEnt * kMaxAcc;  // 68
constexpr int kDecStride = 80;
constexpr int kMaxCtas = 1;
constexpr int kResWords = 3;     // tagged words per slot result (dense per-word arrays)
constexpr int kPollWarps = 12;   // sequencer warps that poll / walk / verify
constexpr int kSlotsPerPoller = 2;
constexpr int kMaxSlots = kPollWarps * 32 * kSlotsPerPoller;
constexpr int kInsSpan = 32;     // insertion accept mask covers d in [-16, 15]


enum SlotFlag : uint32_t {
  kFKindMask = 3u,   // 0 displace, 1 insert, 2 delete
  kFConflict = 4u,   // overlaps a commit of the previous round
  kFOverflow = 8u,   // accepted commit would overflow a cell / brick
  kFEmpty = 16u,     // N == 0: counted rejection (engine.hpp:355, 399)
};

struct SlotExt {  // untagged per-slot payload, published with its own tag
  double du, dw, pe;  // ΔU, ΔW, p (insert: exp factor E)
  MoveData md;
  int32_t cb, ocb, bb, obb;  // cell / brick entered and occupancy (overflow report)
  uint64_t tag;
  uint64_t pad;
};
static_assert(sizeof(SlotExt) % 16 == 0, "SlotExt layout");

struct EngineArgs {
  Grid g;
  Mirror m;
  Box b;
  Store s;
  ChainState* st;
  const Proposal* props;
  gcmc_trace_rec* trace;
  uint64_t nmoves;
  double beta, mu, lambda3, vol, temp, max_disp;
  uint64_t equil, interval;
  int tail, nslots;  // nslots = (gridDim.x - 1) * MG
  double tail_cu, tail_cp, tail_s3, tail_bu, tail_bp;
  uint64_t* dec;     // [kDecStride] decision words
  uint64_t* res;     // [2][kResWords][nslots]
  SlotExt* ext;      // [2][nslots]
  int smem_occ;      // mirror occupancy replicated in shared memory
  int bias0;         // initial variant bias (+1 / -1)
  int nvar;          // variants per displace / delete proposal (move index >= 1)
  unsigned poll_ns;  // back-off between polls (sequencer)
  unsigned epoll_ns;  // back-off between polls (evaluators)
  unsigned long long* prof;
  unsigned long long* stamp;  // profiling: [0] publish time, [1 + slot] (seen, done) pairs
};

// ----------------------------------------------------------------- variants
// Variant v of a pid-based move evaluates N + off(v): 0, +bias, -bias,
// +2 bias, -2 bias, ...
__device__ __forceinline__ int var_off(int v, int bias) {
  if (v == 0) return 0;
  const int k = (v + 1) >> 1;
  return (v & 1) ? bias * k : -bias * k;
}
// Centre of the candidate N offsets at move i: the expected drift rate*i
// (rate in 1/256 per move, published by the sequencer), rounded.
__device__ __forceinline__ int var_centre(int rate, int i) { return (rate * i + 128) >> 8; }
__device__ __forceinline__ int var_of(int d, int bias) {
  if (d == 0) return 0;
  const int k = d < 0 ? -d : d;
  return ((d > 0) == (bias > 0)) ? 2 * k - 1 : 2 * k;
}

// Slot layout of a round with base B: slot 0 is move 0 (its true N is known);
// move i >= 1 takes need(i) consecutive slots, 1 for an insertion and nvar
// (one per candidate N) otherwise. Moves are included while all of their
// slots fit in nslots, up to kMaxMoves and the end of the batch. Both sides
// derive it from the prefix Q[k] = sum_{m<k} need(B0 + m) over the proposal
// ring, so an evaluator can place its slot for any base B = B0 + len with one
// binary search (no assignment step after the decision arrives).
// Candidate N of a displacement / deletion at window position i: nvar
// consecutive values centred on the expected drift (just npub for i = 0,
// whose N is exact).
__device__ __forceinline__ void n_window(int64_t npub, int rate, int i, int nvar, int64_t& nlo,
                                         int& cnt) {
  if (i == 0) {
    nlo = npub;
    cnt = 1;
  } else {
    nlo = npub + var_centre(rate, i) - (nvar - 1) / 2;
    cnt = nvar;
  }
}
// The particle a proposal picks depends on N only through
// pid = index_from(pick, N); over nvar consecutive N it takes at most
// floor(pick (nvar - 1)) + 2 distinct values, one evaluation slot each.
__device__ __forceinline__ int pid_slots(double pick, int nvar) {
  return (int)__dmul_rn(pick, (double)(nvar - 1)) + 2;
}
// First particle of the window (lowest N >= 1), or -1 if every N <= 0.
__device__ __forceinline__ int64_t pid_lo(double pick, int64_t nlo, int cnt) {
  const int64_t n1 = nlo < 1 ? 1 : nlo;
  if (n1 > nlo + cnt - 1) return -1;
  return (int64_t)index_from(pick, (uint64_t)n1);
}

__device__ __forceinline__ int need_of(const EngineArgs& a, const Proposal* ring, uint64_t mv) {
  if (mv >= a.nmoves) return 1 << 16;
  const Proposal& p = ring[mv % kRing];
  return p.kind == 1 ? 1 : pid_slots(p.pick, a.nvar);
}

// One warp: Q[0..kPre) over moves B0, B0+1, ...
__device__ __forceinline__ void prefix_warp(const EngineArgs& a, const Proposal* ring, uint64_t b0,
                                           int* Q, int lane) {
  constexpr int PER = (kPre + 31) / 32;  // 5
  int v[PER], run = 0;
#pragma unroll
  for (int j = 0; j < PER; ++j) {
    const int k = lane * PER + j;
    v[j] = k < kPre - 1 ? need_of(a, ring, b0 + (uint64_t)k) : 0;
    run += v[j];
  }
  int incl = run;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  int ex = incl - run;
#pragma unroll
  for (int j = 0; j < PER; ++j) {
    const int k = lane * PER + j;
    if (k < kPre) Q[k] = ex;
    ex += v[j];
  }
}

// Moves / slots of the round at base B0 + len (Q relative to B0).
__device__ __forceinline__ void round_shape(const EngineArgs& a, const int* Q, int len,
                                            uint64_t b, int& fit, int& used) {
  if (b >= a.nmoves) {
    fit = used = 0;
    return;
  }
  // largest f with 1 + Q[len+f] - Q[len+1] <= nslots, f <= kMaxMoves, b+f <= nmoves
  int lo = 1, hi = kMaxMoves;
  const uint64_t left = a.nmoves - b;
  if ((uint64_t)hi > left) hi = (int)left;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (1 + Q[len + mid] - Q[len + 1] <= a.nslots) lo = mid; else hi = mid - 1;
  }
  fit = lo;
  used = 1 + Q[len + lo] - Q[len + 1];
}

// Slot s of the round at base B0 + len -> (move i, variant v); false if unused.
__device__ __forceinline__ bool slot_move(const int* Q, int len, int s, int fit, int& i, int& v) {
  if (s == 0) {
    i = 0;
    v = 0;
    return fit > 0;
  }
  const int target = Q[len + 1] + (s - 1);
  int lo = len + 1, hi = len + fit - 1;  // k with Q[k] <= target
  if (hi < lo) return false;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (Q[mid] <= target) lo = mid; else hi = mid - 1;
  }
  i = lo - len;
  v = target - Q[lo];
  return Q[lo + 1] > target;  // inside move lo (the last move may be partial -> beyond used)
}

// Slot of move i resolved at N offset dd (sequencer; fs = first slot of i).
__device__ __forceinline__ int resolved_slot(const EngineArgs& a, const Proposal& pr, int i, int fs,
                                             int64_t npub, int rate, int dd) {
  if (pr.kind == 1) return fs;
  int64_t nlo;
  int cnt;
  n_window(npub, rate, i, a.nvar, nlo, cnt);
  const int64_t nn = npub + dd;
  if (nn <= 0) return fs;
  const int64_t plo = pid_lo(pr.pick, nlo, cnt);
  return fs + (int)((int64_t)index_from(pr.pick, (uint64_t)nn) - plo);
}

// ----------------------------------------------------------------- conflicts
struct RW {  // what an evaluation read / a commit wrote
  uint64_t pt[3];  // brick points: new, old, last particle (delete)
  int64_t ia, ib;  // particle indices: pid / insert index, q
};

// Read set of move i (later) vs write set of accepted move j (earlier).
__device__ __forceinline__ bool conflict(const Mirror& m, bool all_pairs, const RW& r,
                                         const RW& w) {
  if (all_pairs) return true;
  if (r.ia >= 0 && (r.ia == w.ia || r.ia == w.ib)) return true;
  if (r.ib >= 0 && (r.ib == w.ia || r.ib == w.ib)) return true;
  // points: new (0) and old (1); pt[2] is unused since deletions no longer
  // read the last particle during evaluation
  return mnear(m, r.pt[0], w.pt[0]) || mnear(m, r.pt[0], w.pt[1]) ||
         mnear(m, r.pt[1], w.pt[0]) || mnear(m, r.pt[1], w.pt[1]);
}

// ----------------------------------------------------------------- decision
struct Dec {
  uint64_t base, n;
  int nacc, bias, stop, rate;
  RW acc[kMaxAcc];
  int kind[kMaxAcc];
};

// Ring refill by one warp: proposals [lo, hi) (8-byte async copies).
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

// Warp: wait for D_r and decode it. The D words are self-validating (round
// tag per word); the loads that follow go to L2 (ld.cg), which holds every
// commit the sequencer's helpers completed (and fenced) before D_r was
// written.
__device__ __forceinline__ void poll_dec(const EngineArgs& a, uint32_t r, Dec& d, int lane) {
  constexpr int PER = (kDecWords + 31) / 32;
  uint64_t w[PER];
  const uint64_t* dec = a.dec;  // one copy, polled by every evaluator CTA
  for (;;) {
    w[0] = ld_relaxed(dec + lane);
    w[1] = ld_relaxed(dec + 32 + lane);
    const uint64_t h2 = __shfl_sync(0xffffffffu, w[0], 2);
    const bool h2ok = tagged(h2, r);
    const int nacc = h2ok ? (int)(h2 & 0xff) : 0;
    const int need = kDecHdr + kDecEnt * nacc;
    if (need > 64) {
#pragma unroll
      for (int j = 2; j < PER; ++j) {
        const int idx = lane + 32 * j;
        w[j] = idx < need ? ld_relaxed(dec + idx) : 0;
      }
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
      d.bias = (p >> 8) & 1 ? 1 : -1;
      d.stop = (int)((p >> 9) & 1);
      d.rate = (int)(int16_t)(uint16_t)((p >> 10) & 0xffff);
    } else if (idx >= kDecHdr) {
      const int e = (idx - kDecHdr) / kDecEnt, f = (idx - kDecHdr) % kDecEnt;
      if (f == 0) {
        d.acc[e].pt[0] = p & kNoPoint;
        d.acc[e].pt[1] = (p >> 24) & kNoPoint;
        d.acc[e].pt[2] = kNoPoint;
      } else {
        d.kind[e] = (int)(p >> 32) & 3;
        const uint32_t ia = (uint32_t)p;
        d.acc[e].ia = ia == 0xffffffffu ? -1 : (int64_t)ia;
        d.acc[e].ib = -1;
      }
    }
  }
  __syncwarp();
}

// =================================================================== evaluator
template <int T>
struct EvalShared {
  Proposal ring[kRing];
  Dec d;
  int Q[kPre];
  int16_t stab[kMaxMoves + 1][kThreads / T];  // slot of group g for a round of length len: i | v << 8
  WinWs<T> ws[kThreads / T];
  struct G {
    int i, v, kind, empty, cf;
    uint32_t cov;    // candidate N (window-relative bits) this slot decides
    long long nlo;   // lowest candidate N
    uint64_t pid, q, nv;
    MoveData md;
    double acc;
    int pre, cell;   // new position precomputed (k_annotate): its brick point and grid cell
    uint32_t bpt;
  } gs[kThreads / T];
};

// Warp: for every possible length of the round in progress (next base =
// b0 + len), the (move, variant) of this CTA's MG slots.
template <int MG>
__device__ __forceinline__ void slot_table_warp(const EngineArgs& a, const int* Q, uint64_t b0,
                                                int cta_slot0, int16_t (*stab)[MG], int lane) {
  for (int len = lane; len <= kMaxMoves; len += 32) {
    int fit, used;
    round_shape(a, Q, len, b0 + (uint64_t)len, fit, used);
#pragma unroll
    for (int g = 0; g < MG; ++g) {
      int i = -1, v = 0;
      const int s = cta_slot0 + g;
      if (!(s < used && slot_move(Q, len, s, fit, i, v))) i = -1;
      stab[len][g] = (int16_t)(i < 0 ? -1 : (i | (v << 8)));
    }
  }
}

template <int T>
__device__ void evaluator(const EngineArgs& a, uint8_t* smem) {
  constexpr int MG = kThreads / T;
  auto& sh = *reinterpret_cast<EvalShared<T>*>(smem);
  uint8_t* occ_s = a.smem_occ ? smem + ((sizeof(EvalShared<T>) + 15) & ~size_t(15)) : nullptr;
  uint32_t* occ_w = reinterpret_cast<uint32_t*>(occ_s);
  const int tid = threadIdx.x, lane = tid & 31;
  const int g = tid / T, gt = tid % T, gw = gt >> 5;
  const int bar_id = 1 + g;
  const int cta_slot0 = (blockIdx.x - 1) * MG;  // slots >= nslots are never used
  WinWs<T>& ws = sh.ws[g];
  auto& G = sh.gs[g];
  const bool all_pairs = a.g.kind == GCMC_ALL_PAIRS;

  // initial replica, ring, slot prefix
  if (occ_s)
    for (uint32_t i = tid; i < a.m.nb; i += kThreads) occ_s[i] = (uint8_t)__ldcg(a.m.occ + i);
  uint64_t ring_hi = a.nmoves < (uint64_t)kRing ? a.nmoves : (uint64_t)kRing;
  if (tid < 32) {
    ring_fill(a, sh.ring, 0, ring_hi, lane);
    cp_async_wait();
    __syncwarp();
    prefix_warp(a, sh.ring, 0, sh.Q, lane);
    __syncwarp();
    slot_table_warp<MG>(a, sh.Q, 0, cta_slot0, sh.stab, lane);
  }
  __syncwarp();
    __syncthreads();
  uint64_t b0 = 0;  // base the prefix Q / slot table refer to
  uint32_t r = 1;
  PhaseClock pc;
  pc.start(a.prof && blockIdx.x == 1 && tid == 0);
  for (;; ++r) {
    pc.mark(0);
    if (tid < 32) {
      poll_dec(a, r, sh.d, lane);
      pc.mark(1);  // D observed
      if (a.stamp && lane == 0) {
        const unsigned long long t = gtimer();
        atomicMin(a.stamp + 8 * (r & 8191) + 1, t);  // first CTA sees D_r
        atomicMax(a.stamp + 8 * (r & 8191) + 2, t);  // last CTA sees D_r
      }
      const Dec& d = sh.d;
      // replica: the previous round's commits (a--, b++)
      if (occ_s && lane < d.nacc) {
        const int k = d.kind[lane];
        const RW& e = d.acc[lane];
        if (k != 1) {
          const uint32_t ba = mbrick(a.m, e.pt[1]);
          atomicSub(occ_w + (ba >> 2), 1u << (8 * (ba & 3)));
        }
        if (k != 2) {
          const uint32_t bb = mbrick(a.m, e.pt[0]);
          atomicAdd(occ_w + (bb >> 2), 1u << (8 * (bb & 3)));
        }
      }
      // slots of this CTA (precomputed for every round length)
      if (lane < MG && !d.stop) {
        const int t = sh.stab[(int)(d.base - b0)][lane];
        sh.gs[lane].i = t < 0 ? -1 : (t & 0xff);
        sh.gs[lane].v = t < 0 ? 0 : (t >> 8);
      }
      cp_async_wait();
    }
    __syncwarp();
    __syncthreads();
    const Dec& d = sh.d;
    if (d.stop) break;
    pc.mark(2);  // replica + slot
    uint64_t* rw = a.res + (size_t)(r & 1) * kResWords * a.nslots + cta_slot0 + g;  // + j * nslots
    SlotExt* ex = a.ext + (size_t)(r & 1) * a.nslots + cta_slot0 + g;
    if (G.i >= 0) {
      constexpr int kGW = T / 32;                 // warps per group
      const int lw = g % (kGW < 4 ? kGW : 4);     // leader warp
      const int lw2 = kGW > 1 ? (lw + 1) % kGW : lw;
      int ocb = 0;
      int setup_nent = 0, setup_nent0 = 0;
      const int bar_pair = 1 + MG + g;  // leader and second warp of the group
      // ---- setup (the group's leader warp: warp g % 4 of group g, so the
      // groups' serial chains run on different SM sub-partitions)
      if (gw == lw) {
        const uint64_t mv = d.base + (uint64_t)G.i;
        const Proposal& pr = sh.ring[mv % kRing];
        const int kind = pr.kind;
        int empty = 0;
        int64_t nv = (int64_t)d.n;
        uint64_t pid = 0, q = 0;
        uint32_t cov = 0;  // candidate N (window-relative bits) this slot decides
        int64_t nlo = 0;
        if (kind != 1) {
          int cnt;
          n_window((int64_t)d.n, d.rate, G.i, a.nvar, nlo, cnt);
          const int64_t plo = pid_lo(pr.pick, nlo, cnt);
          const int64_t p = plo + G.v;
          bool real = false;
          if (lane < cnt) {
            const int64_t nl = nlo + lane;
            bool c = false;
            if (nl <= 0) c = G.v == 0;  // empty store: counted rejection (engine.hpp:355, 399)
            else if (plo >= 0 && (int64_t)index_from(pr.pick, (uint64_t)nl) == p) {
              c = true;
              real = true;
            }
            cov = c ? 1u : 0u;
          }
          cov = __ballot_sync(0xffffffffu, cov != 0);
          const bool any_real = __any_sync(0xffffffffu, real);
          empty = !any_real;   // nothing to evaluate (rejection-only or no coverage)
          nv = any_real ? p + 1 : 0;  // any N that maps to p (only for the loads below)
        }
        pc.mark(7);  // s_prop
        MoveData md;
        md.nx = pr.x;
        md.ny = pr.y;
        md.nz = pr.z;
        md.rslot_pid = md.bslot_pid = -1;
        md.ox = md.oy = md.oz = 0.0;
        const bool loads = kind != 1 && !empty;
        if (loads) pid = (uint64_t)(nv - 1);  // the slot's particle p (nv = p + 1 above)
        q = 0;
        // The mover's position and back-pointer: one L2 hop, issued by every
        // lane (one broadcast transaction) and unconditionally (record 0 when
        // unused), so that no register merge waits on it before the windows.
        // (four 64-bit loads: a quad destination invites an early register
        // move that waits on the load)
        const double* op = reinterpret_cast<const double*>(a.s.pos + (loads ? pid : 0));
        double4 o;
        o.x = __ldcg(op);
        o.y = __ldcg(op + 1);
        o.z = __ldcg(op + 2);
        o.w = __ldcg(op + 3);
        // windows, one call site: [0] the new position before the mover load
        // lands (it does not need the mover unless max_displacement), [1] the
        // new position after it (max_displacement), [2] the old position
        const bool early = kind != 2 && !empty && !(kind == 0 && a.max_disp > 0.0) && !all_pairs;
        const bool pre = early && pr.wmask != kNoMask;  // window precomputed (k_annotate)
        if (lane == 0 && early)  // reference cell entered
          ocb = __ldcg(a.g.occ + (pre ? pr.cell : cell_of(a.g, md.nx, md.ny, md.nz)));
        int nent = 0, nent0 = 0;
#pragma unroll 1
        for (int w = 0; w < 3; ++w) {
          if (w == 1) {
            pc.mark(8);  // s_neww
            if (loads) {
              md.ox = o.x;
              md.oy = o.y;
              md.oz = o.z;
              md.rslot_pid = -1;  // the commit loads the reference slot itself
              md.bslot_pid = bslot_in(o);
              if (kind == 0 && a.max_disp > 0.0) {  // engine.hpp:359-365
                const double c = a.max_disp;
                md.nx = wrap_axis(__dadd_rn(md.ox, __dmul_rn(__dsub_rn(__dmul_rn(2.0, pr.x), 1.0), c)), a.b.l);
                md.ny = wrap_axis(__dadd_rn(md.oy, __dmul_rn(__dsub_rn(__dmul_rn(2.0, pr.y), 1.0), c)), a.b.l);
                md.nz = wrap_axis(__dadd_rn(md.oz, __dmul_rn(__dsub_rn(__dmul_rn(2.0, pr.z), 1.0), c)), a.b.l);
                if (lane == 0 && !all_pairs) ocb = __ldcg(a.g.occ + cell_of(a.g, md.nx, md.ny, md.nz));
              }
            }
            pc.mark(9);  // s_load
          }
          const bool want = w == 0 ? early
                          : (!all_pairs && !empty &&
                             (w == 1 ? (kind == 0 && !early) : kind != 1));
          if (want) {
            if (w == 0 && pre) {
              nent = window_bricks_mask(a.m, pr.wmask, pr.bpt, ws.brick, lane);
            } else {
              const double cx = w == 2 ? md.ox : md.nx, cy = w == 2 ? md.oy : md.ny,
                           cz = w == 2 ? md.oz : md.nz;
              nent = win_add<T>(a.m, a.b, ws, nent, cx, cy, cz, lane);
            }
            if (w < 2 || kind == 2) nent0 = nent;
          }
        }
        pc.mark(10);  // s_oldw
        setup_nent = nent;
        setup_nent0 = nent0;
        if (lane == 0) {
          G.kind = kind;
          G.empty = empty;
          G.cov = cov;
          G.nlo = nlo;
          G.pid = pid;
          G.q = q;
          G.nv = (uint64_t)(nv < 0 ? 0 : nv);
          G.md = md;
          G.acc = pr.acc;
          G.pre = pre;
          G.bpt = pr.bpt;
          G.cell = pr.cell;
          ws.excl = loads ? md.bslot_pid : -1;
          if (kind == 2) {
            ws.nwin = 1;
            ws.sign1 = 1;
            ws.cx[0] = md.ox;
            ws.cy[0] = md.oy;
            ws.cz[0] = md.oz;
          } else {
            ws.nwin = kind == 0 ? 2 : 1;
            ws.sign1 = -1;
            ws.cx[0] = md.nx;
            ws.cy[0] = md.ny;
            ws.cz[0] = md.nz;
            ws.cx[1] = md.ox;
            ws.cy[1] = md.oy;
            ws.cz[1] = md.oz;
          }
          if (empty) ws.total = 0;
        }
        group_sync(bar_pair, 64);  // G published to warp 1
        if (!all_pairs && !G.empty) win_finish<T>(a.m, ws, occ_s, setup_nent, setup_nent0, lane);
        pc.mark(11);  // s_finish
      } else if (gw == lw2) {
        // read set and conflicts with the previous round's commits, in
        // parallel with warp 0's window finish
        group_sync(bar_pair, 64);
        const int kind = G.kind;
        const MoveData& md = G.md;
        const bool loads = kind != 1 && !G.empty;
        RW rs;
        rs.pt[0] = kind != 2 ? (G.pre ? (uint64_t)G.bpt : mpoint(a.m, md.nx, md.ny, md.nz)) : kNoPoint;
        rs.pt[1] = loads ? mpoint(a.m, md.ox, md.oy, md.oz) : kNoPoint;
        rs.pt[2] = kNoPoint;
        rs.ia = loads ? (int64_t)G.pid : -1;
        rs.ib = -1;
        bool cf = false;
        if (!G.empty && lane < d.nacc) cf = conflict(a.m, all_pairs, rs, d.acc[lane]);
        cf = __any_sync(0xffffffffu, cf);
        if (lane == 0) G.cf = cf;
      }
      group_sync(bar_id, T);
      pc.mark(3);  // setup (pid hop + window)
      // ---- sums
      double du = 0.0, dw = 0.0;
      if (!G.empty) {
        if (all_pairs)
          allpairs_sums<T>(a.b, a.s.pos, d.n, ws, G.kind == 1 ? -1 : (long long)G.pid, gt, du, dw);
        else
          win_sums<T>(a.m, a.b, ws, gt, du, dw);
        if (gt == 0)
          atomicAdd(&a.st->pair_evals,
                    (unsigned long long)(all_pairs ? d.n * (uint64_t)ws.nwin : (uint64_t)ws.total));
      }
      group_reduce<T>(ws, du, dw, bar_id, gt, 32 * lw);
      pc.mark(4);  // sums + reduce
      // ---- acceptance bits, conflicts, publish (leader warp)
      if (gw == lw) {
        const int kind = G.kind;
        const MoveData& md = G.md;
        RW rs;
        rs.pt[0] = kind != 2 ? (G.pre ? (uint64_t)G.bpt : mpoint(a.m, md.nx, md.ny, md.nz)) : kNoPoint;
        rs.pt[1] = kind != 1 && !G.empty ? mpoint(a.m, md.ox, md.oy, md.oz) : kNoPoint;
        rs.pt[2] = kNoPoint;
        rs.ia = kind != 1 && !G.empty ? (int64_t)G.pid : -1;
        rs.ib = -1;
        const bool cf = G.cf;
        du = __shfl_sync(0xffffffffu, du, 0);
        dw = __shfl_sync(0xffffffffu, dw, 0);
        uint32_t bits = 0;
        double pe = 0.0;
        double rdu = du, rdw = dw;
        if (G.empty) {
          rdu = rdw = 0.0;
        } else {
          if (kind == 2) {
            rdu = -du;
            rdw = -dw;
          }
          // the one exponential of each kind (engine.hpp:28-59, same operation order)
          const double x = kind == 1 ? __dmul_rn(a.beta, __dsub_rn(a.mu, du))
                         : (kind == 0 ? __dmul_rn(-a.beta, du)
                                      : __dmul_rn(-a.beta, __dadd_rn(a.mu, rdu)));
          const double ex = exp(x);
          if (kind == 1) {
            pe = ex;
            const int64_t nj = (int64_t)d.n + lane - kInsSpan / 2;
            bool ok = false;
            if (nj >= 0) {
              const double p = metropolis(__dmul_rn(
                  __ddiv_rn(a.vol, __dmul_rn(a.lambda3, (double)(nj + 1))), ex));
              ok = G.acc < p;
            }
            bits = __ballot_sync(0xffffffffu, ok);
          } else if (kind == 0) {
            pe = metropolis(ex);
            bits = G.acc < pe ? G.cov : 0u;  // N-independent
            // rejection-only bits (N <= 0) never accept: offsets l <= -nlo
            if (G.nlo <= 0) {
              const int64_t k = 1 - G.nlo;  // bits 0..k-1
              bits &= k >= 32 ? 0u : ~((1u << k) - 1u);
            }
          } else {
            // deletion_acceptance with each candidate N mapping to this particle
            const int64_t nl = G.nlo + lane;
            bool ok = false;
            double pl = 0.0;
            if (((G.cov >> lane) & 1u) && nl > 0) {
              pl = metropolis(__dmul_rn(__ddiv_rn(__dmul_rn(a.lambda3, (double)nl), a.vol), ex));
              ok = G.acc < pl;
            }
            bits = __ballot_sync(0xffffffffu, ok);
            // the trace reports p for the N the walk resolves; publish the one at
            // the lowest covered N (recomputed by the trace writer otherwise)
            pe = __shfl_sync(0xffffffffu, pl, __ffs(G.cov & 0x7fffffffu) ? __ffs(G.cov) - 1 : 0);
          }
        }
        // overflow of the commit (occupancies read this round; exact unless cf)
        bool ovf = false;
        int cb = -1, bb = -1, ob = 0;
        if (lane == 0 && !G.empty && kind != 2) {
          bb = (int)mbrick(a.m, rs.pt[0]);
          const bool same_b = kind == 0 && (uint32_t)bb == mbrick(a.m, rs.pt[1]);
          ob = occ_s ? (int)occ_s[bb] : __ldcg(a.m.occ + bb);
          if (!same_b && ob >= a.m.cap) ovf = true;
          if (!all_pairs) {
            cb = G.pre ? G.cell : cell_of(a.g, md.nx, md.ny, md.nz);
            const bool same_c = kind == 0 && cb == cell_of(a.g, md.ox, md.oy, md.oz);
            if (!same_c && ocb >= a.g.cap) ovf = true;
          }
        }
        ovf = __shfl_sync(0xffffffffu, ovf, 0);
        const uint32_t flags = (uint32_t)kind | (cf ? kFConflict : 0u) | (ovf ? kFOverflow : 0u) |
                               (G.empty ? kFEmpty : 0u);
        if (lane < kResWords) {
          uint64_t p;
          if (lane == 0)
            p = kind == 1 ? (uint64_t)flags | ((uint64_t)bits << 8)
                          : (uint64_t)flags | ((uint64_t)(bits & 0xffffu) << 8) |
                                ((uint64_t)(G.cov & 0xffffu) << 24);
          else if (lane == 1) p = (rs.pt[0] & kNoPoint) | ((rs.pt[1] & kNoPoint) << 24);
          else
            p = (uint64_t)(rs.ia < 0 ? 0xffffffffu : (uint32_t)rs.ia) | ((uint64_t)G.i << 32) |
                ((uint64_t)G.v << 39);
          st_relaxed(rw + (size_t)lane * a.nslots, tagw(r, p));
        }
        if (a.stamp && lane == 0) {
          const unsigned long long t = gtimer();
          unsigned long long* e = a.stamp + 8 * (r & 8191);
          atomicMax(e + 3, t);  // last result
          atomicMin(e + 5, t);  // first result
          atomicAdd(e + 6, t - e[0]);  // mean result time (after the publish)
          atomicAdd(e + 7, 1ull);
        }
        pc.mark(5);  // bits + publish
        // off the critical path: payload, then its own tag after a release
        if (lane == 0) {
          ex->du = rdu;
          ex->dw = rdw;
          ex->pe = pe;
          ex->md = md;
          ex->cb = cb;
          ex->ocb = ocb;
          ex->bb = bb;
          ex->obb = ob;
          fence_gpu();
          st_relaxed(&ex->tag, (uint64_t)r);
        }
      }
    }
    // warp 0: prefix for the next round and ring refill (off the critical path)
    if (tid < 32) {
      b0 = d.base;
      const uint64_t want = b0 + kRing < a.nmoves ? b0 + kRing : a.nmoves;
      prefix_warp(a, sh.ring, b0, sh.Q, lane);
      __syncwarp();
      slot_table_warp<MG>(a, sh.Q, b0, cta_slot0, sh.stab, lane);
      if (want > ring_hi) {
        ring_fill(a, sh.ring, ring_hi, want, lane);
        ring_hi = want;
      }
    }
    pc.mark(6);
  }
  if (a.prof && blockIdx.x == 1 && tid == 0) {
    pc.flush(a.prof + 16);
    a.prof[16 + 15] = r;
  }
}

// =================================================================== sequencer
struct Round {  // a decided round, handed to the helper warps
  uint64_t base, n;
  uint32_t r;
  int len, nacc, par;
  int acc_i[kMaxAcc], acc_s[kMaxAcc], acc_n[kMaxAcc], acc_kind[kMaxAcc];
  uint32_t acc_pid[kMaxAcc];
  int res_s[kMaxMoves], res_d[kMaxMoves];
  uint8_t kind[kMaxMoves], empty[kMaxMoves];
};

enum Stop { kStopEnd, kStopVariant, kStopPrev, kStopVerify, kStopFull, kStopOverflow, kNStop };

struct SeqShared {
  Proposal ring[kRing];
  uint64_t sw[kMaxSlots][kResWords];  // slot words of the current round (payload)
  int Q[kPre];
  int fit, used;
  // per-move masks built by the pollers
  uint32_t macc[kMaxMoves], mcov[kMaxMoves], mcf[kMaxMoves], mov[kMaxMoves];
  uint8_t mkind[kMaxMoves];
  // walk output
  int len, nacc, err, cmin, err_slot, why;
  int acc_i[kMaxAcc], acc_s[kMaxAcc], acc_d[kMaxAcc];
  int res_s[kMaxMoves];  // resolved slot of each consumed move
  int res_d[kMaxMoves];  // N offset at each consumed move
  Round done;            // previous round, processed by the helpers
  double acc_du[kMaxAcc], acc_dw[kMaxAcc];
  double st_e[kMaxAcc + 1], st_w[kMaxAcc + 1];  // statistics: states of the round
  uint64_t st_n[kMaxAcc + 1];
  double st_v[kMaxAcc + 1][4];
  unsigned long long stops[kNStop];
  unsigned long long lat[6];
  uint64_t dw[kDecWords];  // decision words being broadcast
  int dneed;
  ChainState ks;
};

__device__ __forceinline__ RW rw_of(const uint64_t* w) {
  RW x;
  x.pt[0] = w[1] & kNoPoint;
  x.pt[1] = (w[1] >> 24) & kNoPoint;
  x.pt[2] = kNoPoint;
  const uint32_t ia = (uint32_t)w[2];
  x.ia = ia == 0xffffffffu ? -1 : (int64_t)ia;
  x.ib = -1;
  return x;
}

struct Observables {
  double rep_u, pres;
};

// reported_energy() and pressure() (engine.hpp:277-291) with the tail terms
// of tail_corrections() (potential.hpp:63-72), same operation order.
__device__ __forceinline__ Observables observables(const EngineArgs& a, uint64_t n, double u,
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

// Decision D_r (base, N, the previous round's accepted moves): one warp
// composes the words in shared memory, then one thread per word stores them. No fence here: the helpers fenced their commit
// stores before the barrier that precedes the broadcast, so every commit is
// in L2 before any D word is.
__device__ __forceinline__ void compose_dec(uint32_t r, uint64_t base, uint64_t n, int nacc,
                                            int bias, int stop, int rate, SeqShared& sh,
                                            int lane) {
  for (int idx = lane; idx < kDecHdr + kDecEnt * nacc; idx += 32) {
    uint64_t p = 0;
    if (idx == 0) p = base;
    else if (idx == 1) p = n;
    else if (idx == 2)
      p = (uint64_t)nacc | ((uint64_t)(bias > 0) << 8) | ((uint64_t)stop << 9) |
          ((uint64_t)(uint16_t)(int16_t)rate << 10);
    else if (idx >= kDecHdr) {
      const int e = (idx - kDecHdr) / kDecEnt, f = (idx - kDecHdr) % kDecEnt;
      const uint64_t* w = sh.sw[sh.acc_s[e]];
      const int kind = (int)(w[0] & 3);
      if (f == 0) p = w[1];
      else p = ((uint64_t)kind << 32) | (kind == 1 ? (uint32_t)sh.acc_d[e] : (uint32_t)w[2]);
    }
    sh.dw[idx] = tagw(r, p);
  }
  if (lane == 0) sh.dneed = kDecHdr + kDecEnt * nacc;
}
__device__ __forceinline__ void broadcast_dec(const EngineArgs& a, const SeqShared& sh, int tid) {
  if (tid < sh.dneed) st_relaxed(a.dec + tid, sh.dw[tid]);
}

// Helper warps (kPollWarps .. 15): commits, statistics and trace of the
// round in sh.done, while the poll warps wait for the next round.
__device__ void helpers(const EngineArgs& a, SeqShared& sh, int warp, int lane) {
  const Round& D = sh.done;
  if (D.len == 0) return;
  auto ext_of = [&](int s) -> const SlotExt* {
    const SlotExt* ex = a.ext + (size_t)D.par * a.nslots + s;
    while (ld_acquire(&ex->tag) != (uint64_t)D.r) nap();
    return ex;
  };
  if (warp == kPollWarps) {  // commits (commit.cuh): one lane per accepted move
    // All lanes load their commit's inputs in parallel; a commit whose
    // cells / bricks / particles overlap an earlier one of the round is
    // re-loaded and applied after it, in move order; the rest apply at once.
    const bool mine = lane < D.nacc;
    MoveData md{};
    CommitIn c{};
    Touch t{};
    int kind = 0;
    uint64_t pid = 0, nn = 0;
    if (mine) {
      const SlotExt* ex = ext_of(D.acc_s[lane]);
      md = ex->md;
      kind = D.acc_kind[lane];
      pid = D.acc_pid[lane];
      nn = (uint64_t)D.acc_n[lane];
      commit_load(a.g, a.m, a.s, kind, pid, nn, md, c);
      t = touch_of(a.m, kind, pid, nn, c);
    }
    bool dep = false;
    for (int j = 0; j < D.nacc - 1; ++j) {  // does my commit overlap commit j < lane?
      Touch tj;
#pragma unroll
      for (int x = 0; x < 3; ++x) {
        tj.cell[x] = __shfl_sync(0xffffffffu, t.cell[x], j);
        tj.brick[x] = __shfl_sync(0xffffffffu, t.brick[x], j);
      }
#pragma unroll
      for (int x = 0; x < 5; ++x) tj.part[x] = __shfl_sync(0xffffffffu, t.part[x], j);
      if (mine && j < lane && touches(t, tj)) dep = true;
    }
    long long e1, e2, e3;
    if (mine && !dep) commit_store(a.g, a.m, a.s, &a.st->peak, kind, pid, nn, md, c, e1, e2, e3);
    const unsigned deps = __ballot_sync(0xffffffffu, dep);
    if (deps) {
      __threadfence();  // independent commits are in L2 before the ordered ones reload
      __syncwarp();
      for (int j = 0; j < D.nacc; ++j) {
        if (((deps >> j) & 1u) && lane == j)
          commit_move(a.g, a.m, a.s, &a.st->peak, kind, pid, nn, md, e1, e2, e3);
        __syncwarp();
      }
    }
    if (mine) fence_gpu();  // every commit is in L2 before the next decision is published
  } else if (warp == kPollWarps + 1) {  // statistics (engine.hpp:293-308, 413-426)
#ifdef GCMC_EXP_NOSTATS
    return;
#endif
    // Warp-parallel form of the reference's per-step loop with its exact
    // operation order: the energy/virial chain over the accepted moves and
    // the running sums over the sampled steps stay sequential double adds
    // (lane 0), everything else is per lane.
    const int len = D.len, nacc = D.nacc;
    ChainState& ks = sh.ks;
    if (lane < nacc) {
      const SlotExt* ex = ext_of(D.acc_s[lane]);
      sh.acc_du[lane] = ex->du;
      sh.acc_dw[lane] = ex->dw;
    }
    __syncwarp();
    if (lane == 0) {  // state k = after the k-th accepted move of the round
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
    for (int k = lane; k <= nacc; k += 32) {  // sampled values of each state
      const uint64_t cur = sh.st_n[k];
      const Observables ob = observables(a, cur, sh.st_e[k], sh.st_w[k]);
      const double nd = (double)cur;
      sh.st_v[k][0] = nd;
      sh.st_v[k][1] = __dmul_rn(nd, nd);
      sh.st_v[k][2] = ob.rep_u;
      sh.st_v[k][3] = ob.pres;
    }
    // attempted moves by kind; sampled steps (move i ends step step0 + i + 1)
    const uint64_t step0 = ks.step;
    unsigned smp[kMH];
    unsigned att0 = 0, att1 = 0, att2 = 0;
#pragma unroll
    for (int h = 0; h < kMH; ++h) {
      const int i = lane + 32 * h;
      const bool in = i < len;
      const int kind = in ? D.kind[i] : 3;
      att0 += __popc(__ballot_sync(0xffffffffu, kind == 0));
      att1 += __popc(__ballot_sync(0xffffffffu, kind == 1));
      att2 += __popc(__ballot_sync(0xffffffffu, kind == 2));
      const uint64_t st = step0 + (uint64_t)i + 1;
      const bool sm = in && st > a.equil && (a.interval == 1 || (st - a.equil) % a.interval == 0);
      smp[h] = __ballot_sync(0xffffffffu, sm);
    }
    __syncwarp();
    if (lane == 0) {  // running sums in step order; state k holds for moves [acc_i[k-1], acc_i[k])
      double sn = ks.sum_n, sn2 = ks.sum_n2, su = ks.sum_u, sp = ks.sum_p;
      uint64_t samples = 0;
      int lo = 0;
      for (int k = 0; k <= nacc; ++k) {
        const int hi = k < nacc ? D.acc_i[k] : len;
        int c = 0;
#pragma unroll
        for (int h = 0; h < kMH; ++h) {
          const int a0 = lo - 32 * h, a1 = hi - 32 * h;  // bit range [a0, a1) of word h
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
      const int s = D.res_s[i];
      const SlotExt* ex = ext_of(s);
      const int kind = D.kind[i];
      int accepted = 0, dn = 0;
      for (int k = 0; k < D.nacc; ++k) {
        if (D.acc_i[k] == i) accepted = 1;
        if (D.acc_i[k] <= i) dn += D.acc_kind[k] == 1 ? 1 : (D.acc_kind[k] == 2 ? -1 : 0);
      }
      const uint64_t nm = (uint64_t)((int64_t)D.n + D.res_d[i]);
      gcmc_trace_rec t;
      t.kind = kind;
      t.accepted = accepted;
      t.delta_u = ex->du;
      t.delta_w = ex->dw;
      double p = ex->pe;
      if (kind == 1)
        p = metropolis(__dmul_rn(__ddiv_rn(a.vol, __dmul_rn(a.lambda3, (double)(nm + 1))), ex->pe));
      if (kind == 2 && (int64_t)nm > 0)
        p = deletion_acceptance(ex->du, nm, a.vol, a.beta, a.mu, a.lambda3);
      if (D.empty[i] || (kind != 1 && (int64_t)nm <= 0)) p = 0.0;
      t.acceptance_prob = p;
      t.n_after = (uint64_t)((int64_t)D.n + dn);
      a.trace[D.base + i] = t;
    }
  }
}

__device__ void sequencer(const EngineArgs& a, uint8_t* smem) {
  auto& sh = *reinterpret_cast<SeqShared*>(smem);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool all_pairs = a.g.kind == GCMC_ALL_PAIRS;
  constexpr int kPollThreads = kPollWarps * 32;
  if (tid == 0) {
    sh.ks = *a.st;
    sh.done.len = 0;
    sh.err = 0;
    for (int k = 0; k < kNStop; ++k) sh.stops[k] = 0;
    for (int k = 0; k < 6; ++k) sh.lat[k] = 0;
  }
  if (tid < kMaxMoves) {
    sh.macc[tid] = sh.mcov[tid] = sh.mcf[tid] = sh.mov[tid] = 0;
  }
  uint64_t ring_hi = a.nmoves < (uint64_t)kRing ? a.nmoves : (uint64_t)kRing;
  if (warp == 0) {
    ring_fill(a, sh.ring, 0, ring_hi, lane);
    cp_async_wait();
    __syncwarp();
    prefix_warp(a, sh.ring, 0, sh.Q, lane);
    __syncwarp();
    if (lane == 0) round_shape(a, sh.Q, 0, 0, sh.fit, sh.used);
  }
  __syncwarp();
    __syncthreads();
  uint64_t base = 0, n = sh.ks.n;
  int bias = a.bias0;
  uint64_t rounds = 0;
  uint32_t r = 1;
  int rate = 0;         // drift of N per move, 1/256 units
  float rate_f = 0.0f;
  if (warp == 0) compose_dec(r, base, n, 0, bias, 0, rate, sh, lane);
  __syncwarp();
    __syncthreads();
  broadcast_dec(a, sh, tid);
  PhaseClock pc, ph;
  pc.start(a.prof && tid == 0);
  ph.start(a.prof && tid == kPollWarps * 32);
  for (;;) {
    const int par = (int)(r & 1);
    if (warp < kPollWarps) {
      // -------------------- poll: slot words + per-move masks
      const int used = sh.used;
      for (int sl = tid; sl < used; sl += kPollThreads) {
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
#pragma unroll
        for (int j = 0; j < kResWords; ++j) sh.sw[sl][j] = w[j] & kPay;
        const uint32_t w0 = (uint32_t)w[0];
        const uint32_t bits = (uint32_t)((w[0] & kPay) >> 8);
        const int i = (int)((w[2] >> 32) & 127), v = (int)((w[2] >> 39) & 31);
        const int kind = (int)(w0 & 3);
        if (v == 0) sh.mkind[i] = (uint8_t)kind;
        // walk masks indexed by the N offset: bit j <-> d = j - kInsSpan/2
        if (kind == 1) {  // one slot, an accept bit per N
          const bool cf = (w0 & kFConflict) != 0;
          sh.macc[i] = bits;
          sh.mcov[i] = cf ? 0u : 0xffffffffu;
          sh.mcf[i] = cf ? 0xffffffffu : 0u;
          sh.mov[i] = (w0 & kFOverflow) ? 0xffffffffu : 0u;
        } else {  // a particle's slot: bits over its candidate N window
          int64_t nlo;
          int cnt;
          n_window((int64_t)n, rate, i, a.nvar, nlo, cnt);
          const int j0 = (int)(nlo - (int64_t)n) + kInsSpan / 2;
          const uint32_t acc16 = bits & 0xffffu, cov16 = (bits >> 16) & 0xffffu;
          auto place = [&](uint32_t m) -> uint32_t {
            if (j0 >= 32 || j0 <= -32) return 0u;
            return j0 >= 0 ? (m << j0) : (m >> -j0);
          };
          const uint32_t cw = place(cov16), aw = place(acc16);
          if (aw) atomicOr(&sh.macc[i], aw);
          if (cw) {
            if (w0 & kFConflict) atomicOr(&sh.mcf[i], cw);
            else atomicOr(&sh.mcov[i], cw);
            if (w0 & kFOverflow) atomicOr(&sh.mov[i], cw);
          }
        }
      }
      group_sync(1, kPollThreads);
      pc.mark(1);  // poll (waiting for the evaluators)
      if (a.stamp && tid == 0) a.stamp[8 * (r & 8191) + 4] = gtimer();  // sequencer has all
      if (warp == 0) {  // ---- walk (table-driven: bit j of a mask <-> d = j - 16)
        const int fit = sh.fit;
        uint32_t accm[kMH], stopm[kMH], ovfm[kMH], cfmk[kMH];
        unsigned kins[kMH], kdel[kMH];
#pragma unroll
        for (int h = 0; h < kMH; ++h) {
          const int i = lane + 32 * h;
          const bool in = i < fit;
          const int kd = in ? sh.mkind[i] : 0;
          accm[h] = in ? sh.macc[i] : 0u;
          stopm[h] = in ? ~sh.mcov[i] : 0xffffffffu;
          cfmk[h] = in ? sh.mcf[i] : 0u;
          ovfm[h] = in ? sh.mov[i] : 0u;
          kins[h] = __ballot_sync(0xffffffffu, kd == 1);
          kdel[h] = __ballot_sync(0xffffffffu, kd == 2);
        }
        pc.mark(6);  // walk: masks
        int d = 0, start = 0, nacc = 0, len = fit, err = 0, why = kStopEnd;
        int di[kMH];
#pragma unroll
        for (int h = 0; h < kMH; ++h) di[h] = 0;  // N offset at my moves
        int acc_e = -1, acc_dd = 0;  // lane k < nacc holds accepted move k and its d
        for (;;) {
          const int j = d + kInsSpan / 2;
          const bool inr = j >= 0 && j < kInsSpan;
          int e = -1, eh = 0;
          bool est = false, eov = false, ecf = false;
#pragma unroll
          for (int h = 0; h < kMH; ++h) {
            if (e >= 0) break;
            const int i = lane + 32 * h;
            const bool act = i >= start && i < fit;
            const bool st = act && (!inr || ((stopm[h] >> j) & 1u));
            const bool ac = act && inr && ((accm[h] >> j) & 1u);
            const unsigned b = __ballot_sync(0xffffffffu, st || ac);
            if (b) {
              const int el = __ffs(b) - 1;
              e = 32 * h + el;
              eh = h;
              const unsigned bit = 1u << el;
              est = (__ballot_sync(0xffffffffu, st) & bit) != 0;
              eov = (__ballot_sync(0xffffffffu, ac && ((ovfm[h] >> j) & 1u)) & bit) != 0;
              ecf = (__ballot_sync(0xffffffffu, act && inr && ((cfmk[h] >> j) & 1u)) & bit) != 0;
            }
          }
          if (e < 0) {
            len = fit;
            why = kStopEnd;
            break;
          }
          if (est) {
            len = e;
            why = ecf ? kStopPrev : kStopVariant;
            break;
          }
          if (eov) {
            len = e;  // the reference throws inside the commit of move e
            err = 1;
            why = kStopOverflow;
            break;
          }
          if (lane == nacc) {
            acc_e = e;
            acc_dd = d;
          }
          ++nacc;
          const unsigned bit = 1u << (e & 31);
          int delta = 0;
#pragma unroll
          for (int h = 0; h < kMH; ++h)
            if (h == eh) delta = (kins[h] & bit) ? 1 : ((kdel[h] & bit) ? -1 : 0);
#pragma unroll
          for (int h = 0; h < kMH; ++h)
            if (lane + 32 * h > e) di[h] += delta;
          d += delta;
          start = e + 1;
          if (nacc == kMaxAcc) {
            len = e + 1;
            why = kStopFull;
            break;
          }
        }
        pc.mark(7);  // walk: iterations
        // resolved slots of the consumed moves, accepted list
#pragma unroll
        for (int h = 0; h < kMH; ++h) {
          const int i = lane + 32 * h;
          if (i < len) {
            const int k = sh.mkind[i];
            const int dd = di[h];
            const int fs = i == 0 ? 0 : 1 + sh.Q[i] - sh.Q[1];
            sh.res_s[i] = resolved_slot(a, sh.ring[(base + i) % kRing], i, fs, (int64_t)n, rate, dd);
            (void)k;
            sh.res_d[i] = dd;
          }
        }
        if (lane < nacc) {
          const int i = acc_e;
          const int k = sh.mkind[i];
          const int fs = i == 0 ? 0 : 1 + sh.Q[i] - sh.Q[1];
          sh.acc_i[lane] = i;
          sh.acc_s[lane] = resolved_slot(a, sh.ring[(base + i) % kRing], i, fs, (int64_t)n, rate, acc_dd);
          (void)k;
          sh.acc_d[lane] = (int)((int64_t)n + acc_dd);  // store size before move i
        }
        if (err) {  // the overflowing move's slot
          const int i = len;
          const int k = sh.mkind[i];
          const int fs = i == 0 ? 0 : 1 + sh.Q[i] - sh.Q[1];
          if (lane == 0) sh.err_slot = resolved_slot(a, sh.ring[(base + i) % kRing], i, fs, (int64_t)n, rate, d);
          (void)k;
        }
        if (lane == 0) {
          sh.len = len;
          sh.nacc = nacc;
          sh.cmin = len;
          sh.err = err;
          sh.why = why;
        }
      }
      group_sync(1, kPollThreads);
      pc.mark(2);  // walk
      {  // ---- verify: every consumed move against the accepted moves before it
        const int len = sh.len, nacc = sh.nacc;
        const int i = tid % kMaxMoves;
        if (i < len)
          for (int j = tid / kMaxMoves; j < nacc; j += kPollThreads / kMaxMoves) {
            if (i <= sh.acc_i[j]) continue;
            const RW ri = rw_of(sh.sw[sh.res_s[i]]);
            RW wj = rw_of(sh.sw[sh.acc_s[j]]);
            if ((sh.sw[sh.acc_s[j]][0] & 3) == 1) wj.ia = sh.acc_d[j];  // insertion index
            if (conflict(a.m, all_pairs, ri, wj)) atomicMin(&sh.cmin, i);
          }
      }
      group_sync(1, kPollThreads);
      pc.mark(3);  // verify
      if (tid == 0 && sh.cmin < sh.len) {
        const int c = sh.cmin;
        sh.len = c;
        int k = 0;
        while (k < sh.nacc && sh.acc_i[k] < c) ++k;
        sh.nacc = k;
        sh.err = 0;  // the overflowing move is not reached this round
        sh.why = kStopVerify;
      }
    } else {
      helpers(a, sh, warp, lane);  // previous round, concurrently with the poll
      ph.mark(0);
    }
    __syncwarp();
    __syncthreads();
    pc.mark(4);  // wait for helpers
    // -------------------- close the round
    const int len = sh.len, nacc = sh.nacc;
    int dn = 0;
    for (int k = 0; k < nacc; ++k) {
      const int kd = (int)(sh.sw[sh.acc_s[k]][0] & 3);
      dn += kd == 1 ? 1 : (kd == 2 ? -1 : 0);
    }
    const uint64_t nbase = base + (uint64_t)len;
    const uint64_t nn = (uint64_t)((int64_t)n + dn);
    if (dn != 0) bias = dn > 0 ? 1 : -1;
    if (len > 0) {  // exponential average of the drift of N per move
      rate_f = 0.9f * rate_f + 0.1f * (float)dn / (float)len;
      int rr = __float2int_rn(rate_f * 256.0f);
      rate = rr < -128 ? -128 : (rr > 128 ? 128 : rr);
    }
    const bool stop = nbase >= a.nmoves || sh.err;
    if (warp == 0) {
      compose_dec(r + 1, nbase, nn, nacc, bias, stop, rate, sh, lane);
    } else if (warp >= 1 && warp <= kMaxMoves / 32) {  // hand the round to the helpers
      Round& D = sh.done;
      const int i = tid - 32;
      if (i < len) {
        D.res_s[i] = sh.res_s[i];
        D.res_d[i] = sh.res_d[i];
        const uint64_t w0 = sh.sw[sh.res_s[i]][0];
        D.kind[i] = (uint8_t)(w0 & 3);
        D.empty[i] = (uint8_t)((w0 & kFEmpty) ? 1 : 0);
      }
      if (i < nacc) {
        const uint64_t* w = sh.sw[sh.acc_s[i]];
        D.acc_i[i] = sh.acc_i[i];
        D.acc_s[i] = sh.acc_s[i];
        D.acc_n[i] = sh.acc_d[i];
        D.acc_kind[i] = (int)(w[0] & 3);
        D.acc_pid[i] = (uint32_t)w[2];
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
    __syncwarp();
    __syncthreads();
    if (a.stamp && tid == 0) a.stamp[8 * ((r + 1) & 8191)] = gtimer();  // publish of D_{r+1}
    broadcast_dec(a, sh, tid);
    pc.mark(8);  // close until the publish
    // next round's shape, masks, ring (while the evaluators work)
    if (warp == 0) {
      const uint64_t want = nbase + kRing < a.nmoves ? nbase + kRing : a.nmoves;
      prefix_warp(a, sh.ring, nbase, sh.Q, lane);
      __syncwarp();
      if (lane == 0) round_shape(a, sh.Q, 0, nbase, sh.fit, sh.used);
      if (want > ring_hi) {
        ring_fill(a, sh.ring, ring_hi, want, lane);
        ring_hi = want;
      }
      cp_async_wait();
    } else if (tid < 32 + kMaxMoves) {
      sh.macc[tid - 32] = sh.mcov[tid - 32] = sh.mcf[tid - 32] = sh.mov[tid - 32] = 0;
    }
    __syncwarp();
    __syncthreads();
    pc.mark(5);  // next shape (after the publish)
    ph.mark(1);
    base = nbase;
    n = nn;
    ++rounds;
    ++r;
    if (stop) break;
  }
  // the last round's commits / statistics / trace
  if (warp >= kPollWarps) helpers(a, sh, warp, lane);
  __syncwarp();
    __syncthreads();
  if (a.prof && tid == 0) {
    pc.flush(a.prof);
    a.prof[15] = rounds;
    for (int k = 0; k < kNStop; ++k) a.prof[40 + k] = sh.stops[k];
    for (int k = 0; k < 6; ++k) a.prof[48 + k] = sh.lat[k];
  }
  if (a.prof && tid == kPollWarps * 32) {
    a.prof[32] = ph.acc[0];
    a.prof[33] = ph.acc[1];
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
    if (sh.err) {  // overflow at move `base`: report the cell as insert_id would
      const SlotExt* ex = a.ext + (size_t)((r - 1) & 1) * a.nslots + sh.err_slot;
      while (ld_acquire(&ex->tag) != (uint64_t)(r - 1)) nap();
      const bool ref = ex->cb >= 0 && ex->ocb >= a.g.cap;
      a.st->error = GCMC_CELL_OVERFLOW;
      a.st->err_a = ref ? ex->cb : ex->bb;
      a.st->err_b = ref ? ex->ocb : ex->obb;
      a.st->err_c = ref ? 0 : 1;
    }
  }
}

template <int T>
__global__ void __launch_bounds__(kThreads, 1) k_engine(EngineArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  if (blockIdx.x == 0)
    sequencer(a, smem);
  else
    evaluator<T>(a, smem);
}

}  // namespace

gcmc_status engine_run(Chain& c, uint64_t nmoves, gcmc_trace_rec* trace_d, cudaStream_t s) {
  if (nmoves == 0) return GCMC_OK;
  if (engine_sm_supported(c)) {
    c.last_engine = 3;
    return engine_sm_run(c, nmoves, trace_d, s);
  }
  if (engine2_supported(c)) {
    c.last_engine = 2;
    return engine2_run(c, nmoves, trace_d, s);
  }
  c.last_engine = 1;
  c.e_valid = false;  // this engine does not maintain the per-particle energies
  const gcmc_params& P = c.params;
  EngineArgs a{};
  a.g = c.grid;
  a.m = c.mirror;
  a.b = c.box;
  a.s = Store{c.pos, c.rslot};
  a.st = c.st;
  a.props = c.props;
  a.trace = trace_d;
  a.nmoves = nmoves;
  a.beta = 1.0 / P.temperature;  // config.hpp:66
  a.mu = P.chemical_potential;
  a.lambda3 = P.lambda * P.lambda * P.lambda;
  a.vol = P.box_length * P.box_length * P.box_length;  // box.hpp:19
  a.temp = P.temperature;
  a.max_disp = P.max_displacement;
  a.equil = P.equilibration_steps;
  a.interval = P.sampling_interval;
  a.tail = P.tail_corrections;
  a.prof = c.prof;
  a.stamp = c.stamp;
  {
    // potential.hpp:63-72 factored into constants with the same rounding:
    // u = (8/3)*pi * rho * eps * s3 * (sr9/3 - sr3)
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
  const int T = c.engine_group;  // threads per slot
  const int MG = kThreads / T;
  const int G = c.engine_ctas;   // total CTAs (1 sequencer + evaluators)
  a.nslots = (G - 1) * MG;
  if (a.nslots > kMaxSlots) a.nslots = kMaxSlots;  // (G is clamped in api.cu)
  a.dec = c.eng_dec;
  a.res = c.eng_res;
  a.ext = reinterpret_cast<SlotExt*>(c.eng_ext);
  a.bias0 = c.engine_bias;
  a.nvar = c.engine_variants;
  {
    const char* e = knob("GCMC_POLL_NS");
    a.poll_ns = e ? (unsigned)std::atoi(e) : 64u;
    const char* f = knob("GCMC_EPOLL_NS");
    a.epoll_ns = f ? (unsigned)std::atoi(f) : 64u;
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
    std::fprintf(stderr, "[engine prof] smem=%zu eval=%zu seq=%zu occ_replica=%d nb=%u\n", smem,
                 eval_bytes, sizeof(SeqShared), a.smem_occ, c.mirror.nb);
  void (*kern)(EngineArgs) = T == 128 ? k_engine<128> : (T == 256 ? k_engine<256> : k_engine<512>);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e) return cuda_error(e, "engine smem");
  const size_t res_bytes = 2 * (size_t)a.nslots * kResWords * sizeof(uint64_t);
  if ((e = cudaMemsetAsync(c.eng_dec, 0, (size_t)kMaxCtas * kDecStride * sizeof(uint64_t), s)))
    return cuda_error(e, "engine");
  if ((e = cudaMemsetAsync(c.eng_res, 0, res_bytes, s))) return cuda_error(e, "engine");
  if ((e = cudaMemsetAsync(c.eng_ext, 0, 2 * (size_t)a.nslots * sizeof(SlotExt), s))) return cuda_error(e, "engine");
  void* args[] = {&a};
  e = cudaLaunchCooperativeKernel((const void*)kern, dim3(G), dim3(kThreads), args, smem, s);
  if (e) return cuda_error(e, "engine launch");
  return GCMC_OK;
}

size_t engine_buffer_bytes(int nslots, size_t* dec, size_t* res, size_t* ext) {
  *dec = (size_t)kMaxCtas * kDecStride * sizeof(uint64_t);
  *res = 2 * (size_t)nslots * kResWords * sizeof(uint64_t);
  *ext = 2 * (size_t)nslots * sizeof(SlotExt);
  return *dec + *res + *ext;
}

int engine_max_slots() { return kMaxSlots; }

}  // namespace gcmcb
