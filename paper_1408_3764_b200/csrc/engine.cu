// Persistent on-device Metropolis loop: Simulation::step() x n
// (engine.hpp:293-308, 350-426) with exact speculative evaluation.
//
// Why this is exact: every move's random draws are fixed before its ΔE is
// known (engine.hpp:207-213, 352-354), so the proposals are precomputed
// (gen.cu). One thread-block cluster per chain evaluates K = C*M consecutive
// proposals at once — M groups of 512/M threads per CTA, one proposal per
// group (cta_window.cuh) — all against the SAME state S. Moves before the
// first accepted one were each evaluated against exactly the state the
// serial chain would have seen (nothing changed in between), so their
// rejections are the serial chain's rejections. The first accepted move is
// committed by the CTA that evaluated it; later evaluations are discarded
// and redone next round against the new state. The chain is therefore
// move-for-move the reference chain (the paper's "run multiple moves
// concurrently ... keep the first one that is accepted"),
// while the serial latency is paid once per ACCEPTED move instead of once
// per move.
//
// Round protocol (one kernel launch for the whole batch; no host trips):
//   evaluate  group G (= rank*M + g) owns the one move m == G (mod K) in the
//             window [base, base+K): its proposal was prefetched rounds ago,
//             so only pos[pid] and the window cells are loaded; the group's
//             last warp prefetches the commit plan (commit.cuh) meanwhile.
//             accept + kind bits -> the CTA's flag word
//   barrier.cluster (release/acquire)
//   decide    every warp reads the C flag words over DSMEM, rotates the
//             K-bit masks to move order -> first accept j, kind counts
//   commit    group j's leader replays the prefetched plan (stores only);
//             CTA 0 warp 1 applies SystemState / RunStatistics bookkeeping
//             with the reference's sequential double adds; trace records;
//             consumed groups advance m += K and prefetch m + 2K
//   barrier.cluster
#include <cooperative_groups.h>

#include "commit.cuh"
#include "cta_window.cuh"
#include "internal.h"

namespace cg = cooperative_groups;

namespace gcmcb {

namespace {

struct EngineArgs {
  Grid g;
  Box b;
  double4* pos;
  ChainState* st;
  const Proposal* props;
  gcmc_trace_rec* trace;
  uint64_t nmoves;
  double beta, mu, lambda3, vol, temp, max_disp;
  uint64_t equil, interval;
  int tail, pad;
  double tail_cu, tail_cp, tail_s3, tail_bu, tail_bp;  // see engine_run()
  unsigned long long* prof;  // optional phase timers [C][16] (GCMC_ENGINE_PROFILE)
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
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

struct Eval {
  int kind;
  int flag;
  int empty;
  int pad;
  uint64_t pid;
  double du, dw, p, acc;
  double4 old;
  double nx, ny, nz;
};

// One move, one group of T threads. Warp 0 of the group builds the move
// context from the prefetched proposal (pid, old position, target, window
// runs); the group's last warp prefetches the commit plan; every thread scans
// its window rows; the leader finishes the acceptance test.
template <int T>
__device__ __forceinline__ void evaluate(const EngineArgs& a, const Proposal& pr, uint64_t n,
                                         MoveCtx& ctx, GroupReduce<T>& red, CommitPlan& cp,
                                         Eval& ev, int bar_id, unsigned long long* ep) {
  const int gt = threadIdx.x % T, lane = threadIdx.x & 31, gw = gt >> 5;
  unsigned long long t0 = 0;
  if (ep && threadIdx.x == 0) t0 = gtimer();
  if (gw == 0) {
    if (lane == 0) {
      ev.kind = pr.kind;
      ev.flag = 0;
      ev.pid = 0;
      ev.du = ev.dw = ev.p = 0.0;
      ev.old = make_double4(0, 0, 0, 0);
      ev.nx = pr.x;
      ev.ny = pr.y;
      ev.nz = pr.z;
      ev.acc = pr.acc;
      ctx.np = 1;
      ctx.exclude = (long long)n;
      ctx.x[0] = pr.x;
      ctx.y[0] = pr.y;
      ctx.z[0] = pr.z;
      ev.empty = (pr.kind != 1 && n == 0);  // counted rejection (engine.hpp:355,399)
      if (!ev.empty && pr.kind != 1) {
        ev.pid = index_from(pr.pick, n);
        ev.old = ld_cg(a.pos + ev.pid);
        ctx.exclude = (long long)ev.pid;
        if (pr.kind == 0) {
          if (a.max_disp > 0.0) {  // engine.hpp:359-365
            const double c = a.max_disp;
            ev.nx = wrap_axis(__dadd_rn(ev.old.x, __dmul_rn(__dsub_rn(__dmul_rn(2.0, pr.x), 1.0), c)), a.b.l);
            ev.ny = wrap_axis(__dadd_rn(ev.old.y, __dmul_rn(__dsub_rn(__dmul_rn(2.0, pr.y), 1.0), c)), a.b.l);
            ev.nz = wrap_axis(__dadd_rn(ev.old.z, __dmul_rn(__dsub_rn(__dmul_rn(2.0, pr.z), 1.0), c)), a.b.l);
          }
          ctx.np = 2;
          ctx.x[0] = ev.nx;
          ctx.y[0] = ev.ny;
          ctx.z[0] = ev.nz;
          ctx.x[1] = ev.old.x;
          ctx.y[1] = ev.old.y;
          ctx.z[1] = ev.old.z;
        } else {
          ctx.x[0] = ev.old.x;
          ctx.y[0] = ev.old.y;
          ctx.z[0] = ev.old.z;
        }
      }
    }
    __syncwarp();
    setup_runs(a.g, a.b, ctx);
  }
  if (ep && threadIdx.x == 0) { const unsigned long long t = gtimer(); ep[0] += t - t0; t0 = t; }
  group_sync(bar_id, T);
  if (ep && threadIdx.x == 0) { const unsigned long long t = gtimer(); ep[1] += t - t0; t0 = t; }
  if (ev.empty) return;  // uniform across the group
  if (gw == T / 32 - 1)
    commit_prefetch(a.g, a.pos, n, ev.kind, ev.pid, ev.old, ev.nx, ev.ny, ev.nz, cp);
  double du, dw;
  {
    const int gt2 = threadIdx.x % T;
    du = 0.0;
    dw = 0.0;
    if (a.g.kind == GCMC_MICROCELL)
      sums_microcell<T>(a.g, a.b, ctx, gt2, du, dw);
    else if (a.g.kind == GCMC_CELL_LIST)
      sums_cell_list<T>(a.g, a.b, ctx, gt2, du, dw);
    else
      sums_all_pairs<T>(a.b, a.pos, n, ctx, gt2, du, dw);
    if (ep && threadIdx.x == 0) { const unsigned long long t = gtimer(); ep[2] += t - t0; t0 = t; }
    group_reduce2<T>(du, dw, red, bar_id);
    if (ep && threadIdx.x == 0) { const unsigned long long t = gtimer(); ep[3] += t - t0; t0 = t; }
  }
  if (gt == 0) {
    if (ev.kind == 0) {
      ev.du = du;
      ev.dw = dw;
      ev.p = displacement_acceptance(du, a.beta);
    } else if (ev.kind == 1) {
      ev.du = du;
      ev.dw = dw;
      ev.p = insertion_acceptance(du, n, a.vol, a.beta, a.mu, a.lambda3);
    } else {
      ev.du = -du;
      ev.dw = -dw;
      ev.p = deletion_acceptance(ev.du, n, a.vol, a.beta, a.mu, a.lambda3);
    }
    ev.flag = ev.acc < ev.p;
  }
}

__device__ __forceinline__ bool sampled(const EngineArgs& a, uint64_t step) {
  return step > a.equil && (a.interval == 1 || (step - a.equil) % a.interval == 0);
}

__device__ __forceinline__ void cluster_arrive() {
  asm volatile("barrier.cluster.arrive.release;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
  asm volatile("barrier.cluster.wait.acquire;" ::: "memory");
}

// K-bit rotate right (move order from group order).
__device__ __forceinline__ uint64_t rotr(uint64_t v, int s, int K) {
  const uint64_t mask = K == 64 ? ~0ull : ((1ull << K) - 1);
  if (s == 0) return v & mask;
  return ((v >> s) | (v << (K - s))) & mask;
}

template <int M>
__global__ void __launch_bounds__(512, 1) k_engine(EngineArgs a) {
  constexpr int T = 512 / M;
  cg::cluster_group cluster = cg::this_cluster();
  const int tid = threadIdx.x, lane = tid & 31;
  const int g = tid / T, gt = tid % T, gw = gt >> 5;
  const int rank = (int)cluster.block_rank();
  const int C = (int)cluster.num_blocks();
  const int K = C * M;  // <= 64
  const int G = rank * M + g;
  const int bar_id = 1 + g;
  __shared__ uint32_t flagw[2];  // group g: bit 4g accept, bits 4g+1..2 kind; bit 31 stop
  __shared__ Eval ev[M];
  __shared__ MoveCtx ctx[M];
  __shared__ GroupReduce<T> red[M];
  __shared__ CommitPlan cp[M];
  __shared__ ChainState ks;  // bookkeeper's copy (CTA 0)

  uint64_t n = __ldcg(&a.st->n);
  const bool keeper = rank == 0 && tid >= 32 && tid < 64;
  if (keeper && lane == 0) ks = *a.st;
  if (tid == 0) flagw[0] = flagw[1] = 0;
  // group-owned move and its proposals (leader registers)
  uint64_t mg = (uint64_t)G;
  Proposal cur, nxt;
  if (gt == 0) {
    if (mg < a.nmoves) cur = a.props[mg];
    if (mg + K < a.nmoves) nxt = a.props[mg + K];
  }
  cluster.sync();

  uint64_t base = 0, rounds = 0;
  unsigned long long tp[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  unsigned long long ep[4] = {0, 0, 0, 0};
  unsigned long long tl = a.prof ? gtimer() : 0;
  auto mark = [&](int ph) {
    if (a.prof && tid == 0) {
      const unsigned long long t = gtimer();
      tp[ph] += t - tl;
      tl = t;
    }
  };
  while (base < a.nmoves) {
    const int par = (int)(rounds & 1);
    if (tid == 0) flagw[par ^ 1] = 0;
    const bool active = mg < a.nmoves;
    if (active) {
      evaluate<T>(a, cur, n, ctx[g], red[g], cp[g], ev[g], bar_id, a.prof ? ep : nullptr);
      mark(0);
      if (gt == 0)
        atomicOr(&flagw[par], ((uint32_t)ev[g].flag | ((uint32_t)ev[g].kind << 1)) << (4 * g));
    }
    cluster_arrive();  // B1
    mark(1);
    cluster_wait();
    mark(2);
    // ---- decide: move-order masks from the C flag words
    uint32_t fw = 0;
    if (lane < C) fw = *cluster.map_shared_rank(&flagw[par], lane);
    if (__any_sync(0xffffffffu, (fw >> 31) & 1u)) break;  // a commit failed last round
    uint64_t acc = 0, k0 = 0, k1 = 0;
#pragma unroll
    for (int q = 0; q < M; ++q) {
      const uint64_t bit = 1ull << (lane * M + q);
      if (lane < C) {
        if ((fw >> (4 * q)) & 1u) acc |= bit;
        if ((fw >> (4 * q + 1)) & 1u) k0 |= bit;
        if ((fw >> (4 * q + 2)) & 1u) k1 |= bit;
      }
    }
    auto or64 = [](uint64_t v) {
      const uint32_t lo = __reduce_or_sync(0xffffffffu, (uint32_t)v);
      const uint32_t hi = __reduce_or_sync(0xffffffffu, (uint32_t)(v >> 32));
      return ((uint64_t)hi << 32) | lo;
    };
    acc = or64(acc);
    k0 = or64(k0);
    k1 = or64(k1);
    const int off = (int)(base % (uint64_t)K);
    const uint64_t valid = min((uint64_t)K, a.nmoves - base);
    const uint64_t vmask = valid >= 64 ? ~0ull : ((1ull << valid) - 1);
    const uint64_t racc = rotr(acc, off, K) & vmask;
    uint64_t len = valid;
    int j = -1, jG = -1, dn = 0, jkind = 0;
    if (racc) {
      j = __ffsll((long long)racc) - 1;
      len = (uint64_t)j + 1;
      jG = (off + j) % K;
      jkind = (int)(((k0 >> jG) & 1ull) | (((k1 >> jG) & 1ull) << 1));
      dn = jkind == 1 ? 1 : (jkind == 2 ? -1 : 0);
    }
    const int my_off = (G - off + K) % K;
    mark(3);
    // ---- commit (group jG's leader; plan prefetched during evaluation)
    if (jG == G && gt == 0) {
      const Eval& e = ev[g];
      const int s = commit_apply(a.g, a.pos, a.st, n, e.kind, e.pid, e.nx, e.ny, e.nz, cp[g]);
      if (s != GCMC_OK) {
        a.st->error = s;
        a.st->err_a = cp[g].e1;
        a.st->err_b = cp[g].e2;
        a.st->err_c = (long long)(base + j);
        atomicOr(&flagw[par ^ 1], 0x80000000u);
      }
    }
    // ---- trace + advance of consumed groups
    const bool consumed = active && (uint64_t)my_off < len;
    if (gt == 0 && consumed) {
      if (a.trace) {
        gcmc_trace_rec t;
        t.kind = ev[g].kind;
        t.accepted = jG == G;
        t.delta_u = ev[g].du;
        t.delta_w = ev[g].dw;
        t.acceptance_prob = ev[g].p;
        t.n_after = n + (jG == G ? (int64_t)dn : 0);
        a.trace[mg] = t;
      }
      cur = nxt;
      if (mg + 2 * K < a.nmoves) nxt = a.props[mg + 2 * K];
    }
    if (consumed) mg += K;  // every thread of the group tracks its move
    if (keeper) {  // engine.hpp:293-308, 413-426
      double jdu = 0.0, jdw = 0.0;
      if (jG >= 0 && lane == 0) {
        const Eval* re = cluster.map_shared_rank(&ev[jG % M], jG / M);
        jdu = re->du;
        jdw = re->dw;
      }
      if (lane == 0) {
        const uint64_t lm = len >= 64 ? ~0ull : ((1ull << len) - 1);
        const int c1 = __popcll(rotr(k0, off, K) & lm), c2 = __popcll(rotr(k1, off, K) & lm);
        ks.attempted[0] += len - c1 - c2;
        ks.attempted[1] += c1;
        ks.attempted[2] += c2;
        const uint64_t pre = j >= 0 ? len - 1 : len;  // steps sampled in the pre-move state
        uint64_t step = ks.step, samples = ks.samples;
        double sum_n = ks.sum_n, sum_n2 = ks.sum_n2, sum_u = ks.sum_u, sum_p = ks.sum_p;
        if (pre) {
          const Observables ob = observables(a, n, ks.energy, ks.virial);
          const double nd = (double)n, nd2 = __dmul_rn(nd, nd);
          for (uint64_t t = 0; t < pre; ++t) {
            if (sampled(a, step + t + 1)) {
              ++samples;
              sum_n = __dadd_rn(sum_n, nd);
              sum_n2 = __dadd_rn(sum_n2, nd2);
              sum_u = __dadd_rn(sum_u, ob.rep_u);
              sum_p = __dadd_rn(sum_p, ob.pres);
            }
          }
        }
        step += pre;
        if (j >= 0) {
          ks.energy = __dadd_rn(ks.energy, jdu);
          ks.virial = __dadd_rn(ks.virial, jdw);
          ++ks.accepted[jkind];
          const uint64_t n2 = n + dn;
          ++step;
          if (sampled(a, step)) {
            const Observables ob = observables(a, n2, ks.energy, ks.virial);
            const double m1 = (double)n2;
            ++samples;
            sum_n = __dadd_rn(sum_n, m1);
            sum_n2 = __dadd_rn(sum_n2, __dmul_rn(m1, m1));
            sum_u = __dadd_rn(sum_u, ob.rep_u);
            sum_p = __dadd_rn(sum_p, ob.pres);
          }
        }
        ks.step = step;
        ks.samples = samples;
        ks.sum_n = sum_n;
        ks.sum_n2 = sum_n2;
        ks.sum_u = sum_u;
        ks.sum_p = sum_p;
      }
    }
    mark(4);
    cluster_arrive();  // B2
    mark(5);
    cluster_wait();
    mark(6);
    base += len;
    n += dn;
    ++rounds;
  }
  if (a.prof && tid == 0)
    for (int k = 0; k < 8; ++k) a.prof[rank * 16 + k] = tp[k];
  if (a.prof && tid == 0)
    for (int k = 0; k < 4; ++k) a.prof[rank * 16 + 9 + k] = ep[k];
  if (a.prof && tid == 0) a.prof[rank * 16 + 8] = rounds;
  if (keeper && lane == 0) {
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
  }
  (void)gw;
}

}  // namespace

gcmc_status engine_run(Chain& c, uint64_t nmoves, gcmc_trace_rec* trace_d, cudaStream_t s) {
  if (nmoves == 0) return GCMC_OK;
  const gcmc_params& P = c.params;
  EngineArgs a{};
  a.g = c.grid;
  a.b = c.box;
  a.pos = c.pos;
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
  const int C = c.engine_ctas;
  const int M = c.engine_warps;  // moves per CTA (1, 2, 4)
  void (*kern)(EngineArgs) = M == 1 ? k_engine<1> : M == 2 ? k_engine<2> : k_engine<4>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C, 1, 1);
  cfg.blockDim = dim3(512, 1, 1);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, a);
  if (e) return cuda_error(e, "engine launch");
  return GCMC_OK;
}

}  // namespace gcmcb
