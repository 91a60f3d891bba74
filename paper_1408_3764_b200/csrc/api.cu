// C ABI of libgcmc_b200.so (declared in include/gcmc_b200.h). Host-side
// plumbing only: argument checks with the reference's error wording, device
// allocation, staging copies, and dispatch to the kernels in grid.cu,
// delta.cu, energy.cu, gen.cu and engine.cu.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "internal.h"

using namespace gcmcb;

namespace gcmcb {

thread_local std::string g_last_error;

gcmc_status set_error(gcmc_status s, const std::string& msg) {
  g_last_error = msg;
  return s;
}

gcmc_status cuda_error(cudaError_t e, const char* where) {
  std::string m = std::string("CUDA error in ") + where + ": " + cudaGetErrorString(e);
  return set_error(GCMC_CUDA, m);
}

}  // namespace gcmcb

namespace {

#define CK(expr, where)                          \
  do {                                           \
    cudaError_t e_ = (expr);                     \
    if (e_ != cudaSuccess) return cuda_error(e_, where); \
  } while (0)

Chain* H(gcmc_dev* h) { return reinterpret_cast<Chain*>(h); }

gcmc_status invalid_pid(const Chain& c) {
  return set_error(GCMC_INVALID_PID, strategy_name(c.grid.kind) + ": invalid particle id");
}

std::string g17(double v) {
  char buf[64];
  std::snprintf(buf, sizeof buf, "%.17g", v);
  return buf;
}

// RunConfig::validate subset (config.hpp:69-87).
gcmc_status validate(const gcmc_params& p) {
  auto fail = [](const std::string& why) { return set_error(GCMC_ARG, "config: " + why); };
  if (!(p.temperature > 0.0)) return fail("temperature must be > 0");
  if (!(p.lambda > 0.0)) return fail("lambda must be > 0");
  if (!(p.sigma > 0.0)) return fail("sigma must be > 0");
  if (p.epsilon < 0.0) return fail("epsilon must be >= 0");
  if (!(p.r_cut > 0.0)) return fail("r_cut must be > 0");
  if (!(p.box_length > 0.0) || !std::isfinite(p.box_length)) return fail("box length must be > 0");
  if (p.r_cut > p.box_length / 2.0)
    return fail("r_cut must be <= box_length/2 for the minimum image convention (r_cut=" +
                g17(p.r_cut) + ", L=" + g17(p.box_length) + ")");
  if (p.displace_percent < 0.0 || p.displace_percent > 1.0)
    return fail("displace_percent must lie in [0, 1]");
  if (p.sampling_interval == 0) return fail("sampling_interval must be >= 1");
  if (p.cell_capacity < 0) return fail("cell_capacity must be >= 1 (or 0 for automatic)");
  if (p.microcell_capacity < 0) return fail("microcell_capacity must be >= 1");
  if (p.max_displacement < 0.0) return fail("max_displacement must be >= 0");
  if (p.strategy < GCMC_ALL_PAIRS || p.strategy > GCMC_MICROCELL) return fail("unknown strategy");
  return GCMC_OK;
}

void sync_state_to_device(Chain& c) {
  cudaMemcpyAsync(c.st, c.st_host, sizeof(ChainState), cudaMemcpyHostToDevice, c.stream);
}

gcmc_status pull_state(Chain& c) {
  CK(cudaMemcpyAsync(c.st_host, c.st, sizeof(ChainState), cudaMemcpyDeviceToHost, c.stream),
     "state");
  CK(cudaStreamSynchronize(c.stream), "state");
  return GCMC_OK;
}

// Mark the hot arena persisting in L2 for kernels on the chain's stream
// (best effort: devices without persisting L2 keep the default policy).
void set_l2_policy(Chain& c) {
  if (std::getenv("GCMC_NO_L2_POLICY")) return;
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, c.device) != cudaSuccess) return;
  if (prop.persistingL2CacheMaxSize <= 0 || prop.accessPolicyMaxWindowSize <= 0) return;
  const size_t setaside = (size_t)prop.persistingL2CacheMaxSize;
  if (cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, setaside) != cudaSuccess) {
    cudaGetLastError();
    return;
  }
  cudaStreamAttrValue v{};
  v.accessPolicyWindow.base_ptr = c.arena;
  v.accessPolicyWindow.num_bytes = std::min(c.arena_bytes, (size_t)prop.accessPolicyMaxWindowSize);
  v.accessPolicyWindow.hitRatio = 1.0f;
  v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
  v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
  if (cudaStreamSetAttribute(c.stream, cudaStreamAttributeAccessPolicyWindow, &v) != cudaSuccess)
    cudaGetLastError();
}

// Largest particle count the spatial structures admit: every particle has a
// reference-grid slot and a mirror record, and each overflows before the
// store could.
uint64_t store_bound(const Chain& c) {
  uint64_t b = (uint64_t)c.mirror.nb * (uint64_t)c.mirror.cap;
  if (c.grid.kind != GCMC_ALL_PAIRS) b = std::min<uint64_t>(b, (uint64_t)c.grid.cap * c.grid.ncells);
  return b;
}

// (Re)allocates the hot arena (mirror record planes, brick occupancy, store),
// the mirror ids, reference back-pointers and maintained energies for `mcap`
// records per brick and `capn` particles. With `keep`, the live store, its
// back-pointers and energies move over and the mirror is rebuilt from it.
gcmc_status arena_alloc(Chain& c, int mcap, uint64_t capn, bool keep) {
  Mirror& m = c.mirror;
  const uint64_t n = keep ? c.st_host->n : 0;
  const size_t nrec = (size_t)m.nb * mcap;
  const size_t plane = (nrec * sizeof(double) + 255) & ~size_t(255);
  const size_t occb = ((size_t)m.nb * sizeof(int32_t) + 255) & ~size_t(255);
  const size_t posb = capn * sizeof(double4);
  void* arena = nullptr;
  int32_t *rid = nullptr, *rslot = nullptr;
  double2* ep = nullptr;
  CK(cudaMalloc(&arena, 3 * plane + occb + posb), "alloc arena");
  CK(cudaMalloc(&rid, nrec * sizeof(int32_t)), "alloc mirror");
  CK(cudaMalloc(&rslot, capn * sizeof(int32_t)), "alloc rslot");
  CK(cudaMalloc(&ep, capn * sizeof(double2)), "alloc energies");
  char* p = static_cast<char*>(arena);
  double4* pos = reinterpret_cast<double4*>(p + 3 * plane + occb);
  CK(cudaMemsetAsync(pos, 0, posb, c.stream), "memset");
  CK(cudaMemsetAsync(p + 3 * plane, 0, occb, c.stream), "memset");
  if (n) {
    CK(cudaMemcpyAsync(pos, c.pos, n * sizeof(double4), cudaMemcpyDeviceToDevice, c.stream), "grow");
    CK(cudaMemcpyAsync(rslot, c.rslot, n * sizeof(int32_t), cudaMemcpyDeviceToDevice, c.stream), "grow");
    CK(cudaMemcpyAsync(ep, c.ep, n * sizeof(double2), cudaMemcpyDeviceToDevice, c.stream), "grow");
  }
  CK(cudaStreamSynchronize(c.stream), "grow");
  cudaFree(c.arena);
  cudaFree(m.rid);
  cudaFree(c.rslot);
  cudaFree(c.ep);
  c.arena = arena;
  c.arena_bytes = 3 * plane + occb + posb;
  m.rx = reinterpret_cast<double*>(p);
  m.ry = reinterpret_cast<double*>(p + plane);
  m.rz = reinterpret_cast<double*>(p + 2 * plane);
  m.occ = reinterpret_cast<int32_t*>(p + 3 * plane);
  m.rid = rid;
  m.cap = mcap;
  c.pos = pos;
  c.rslot = rslot;
  c.ep = ep;
  c.capn = capn;
  set_l2_policy(c);
  return keep ? mirror_build(c) : GCMC_OK;
}

// Before a batch of m moves: the store must hold every particle the batch can
// reach (min(N + m, store_bound)), growing like a vector.
gcmc_status ensure_store(Chain& c, uint64_t m) {
  const uint64_t need = std::min<uint64_t>(c.st_host->n + m, store_bound(c));
  if (need <= c.capn) return GCMC_OK;
  uint64_t cap = std::max<uint64_t>(need, c.capn + c.capn / 2);
  cap = std::min<uint64_t>(cap, store_bound(c));
  if (cap >= (1ull << 31)) return set_error(GCMC_ARG, "store capacity must be < 2^31 particles");
  return arena_alloc(c, c.mirror.cap, cap, true);
}

// grid_build, doubling the mirror's records per brick while the mirror (not
// the reference grid) is what overflows.
gcmc_status build_growing(Chain& c) {
  gcmc_status s = grid_build(c);
  while (s == GCMC_CELL_OVERFLOW && c.mirror_full && c.mirror.cap < kMaxCap) {
    if ((s = arena_alloc(c, std::min(kMaxCap, 2 * c.mirror.cap), std::max(c.capn, store_bound(c)), true)) &&
        !(s == GCMC_CELL_OVERFLOW && c.mirror_full))
      return s;
    if (!s) c.built = true;
  }
  return s;
}

gcmc_status ensure_batch(Chain& c, uint64_t n) {
  if (n <= c.batch_cap) return GCMC_OK;
  if (c.dscratch) cudaFree(c.dscratch);
  if (c.iscratch) cudaFree(c.iscratch);
  uint64_t cap = n < 1024 ? 1024 : n;
  // doubles: du, dw, xyz(3) ; ints: kinds ; u64 pids -> stored in the double block
  CK(cudaMalloc(&c.dscratch, cap * 7 * sizeof(double)), "alloc");
  CK(cudaMalloc(&c.iscratch, cap * sizeof(int32_t) + 64), "alloc");
  c.batch_cap = cap;
  return GCMC_OK;
}


#ifdef GCMC_PHASE_TIMERS
// Phase-timer build only (python tools/build_variant.py prof -DGCMC_PHASE_TIMERS,
// then GCMC_LIB=...prof.so GCMC_ENGINE_PROFILE=1): per-round phase cycles and
// latency stamps of the engine, printed to stderr after every chunk.
#define CKV(expr, where) \
  do {                   \
    if ((expr) != cudaSuccess) return; \
  } while (0)
void profile_arm(Chain& c) {
  if (std::getenv("GCMC_ENGINE_PROFILE") && !c.prof) {
    CKV(cudaMalloc(&c.prof, 4096 * sizeof(unsigned long long)), "prof");
  }
  if (c.prof) CKV(cudaMemsetAsync(c.prof, 0, 4096 * sizeof(unsigned long long), c.stream), "prof");
  const bool lat = std::getenv("GCMC_ENGINE_LATENCY") != nullptr;
  if (lat && !c.stamp) CKV(cudaMalloc(&c.stamp, 8 * 8192 * sizeof(unsigned long long)), "stamp");
  if (lat) {
    std::vector<unsigned long long> init(8 * 8192, 0);
    for (int k = 0; k < 8192; ++k) init[8 * k + 1] = init[8 * k + 5] = ~0ull;
    CKV(cudaMemcpyAsync(c.stamp, init.data(), init.size() * 8, cudaMemcpyHostToDevice, c.stream), "stamp");
  }
}

void profile_report(Chain& c) {
  if (!c.prof) return;
  unsigned long long hp[64];
  cudaMemcpy(hp, c.prof, sizeof hp, cudaMemcpyDeviceToHost);
  const double R = (double)(hp[15] ? hp[15] : 1);
  const char* sn[] = {"-", "poll", "walk_tail", "verify", "helpers_wait", "next_shape", "walk_masks", "walk_iter", "close_to_publish"};
  std::fprintf(stderr, "[engine prof] rounds %llu sequencer:", hp[15]);
  for (int k = 1; k < 9; ++k) std::fprintf(stderr, " %s=%.0f", sn[k], hp[k] / R);
  const char* en[] = {"idle", "poll_D", "assign", "setup_sync", "sums", "publish", "tail",
                      "s_prop", "s_neww", "s_load", "s_oldw", "s_finish"};
  std::fprintf(stderr, "\n[engine prof] evaluator(cta1,g0):");
  for (int k = 0; k < 12; ++k) std::fprintf(stderr, " %s=%.0f", en[k], hp[16 + k] / R);
  std::fprintf(stderr, "\n[engine prof] helpers: work=%.0f idle=%.0f (cycles/round)\n", hp[32] / R,
               hp[33] / R);
  std::fprintf(stderr, "[engine prof] round ends: end=%llu variant=%llu prev=%llu verify=%llu full=%llu overflow=%llu\n",
               hp[40], hp[41], hp[42], hp[43], hp[44], hp[45]);
  {
    unsigned long long xp[80];
    cudaMemcpy(xp, c.prof, sizeof xp, cudaMemcpyDeviceToHost);
    std::fprintf(stderr, "[engine prof] raw seq:");
    for (int k = 0; k < 12; ++k) std::fprintf(stderr, " %d=%.0f", k, xp[k] / R);
    std::fprintf(stderr, "\n[engine prof] raw eval:");
    for (int k = 0; k < 12; ++k) std::fprintf(stderr, " %d=%.0f", k, xp[16 + k] / R);
    const double ne = (double)(xp[68] ? xp[68] : 1);
    {
      unsigned long long cp[12];
      cudaMemcpy(cp, c.prof + 80, sizeof cp, cudaMemcpyDeviceToHost);
      const double nr = (double)(cp[7] ? cp[7] : 1);
      std::fprintf(stderr, "\n[engine prof] committer (per round, %llu rounds, %.2f commits, %.2f ordered): atab=%.0f move+ext=%.0f commit_load=%.0f deps=%.0f stores=%.0f ordered=%.0f fence=%.0f go_wait=%.0f forwarded=%.2f",
                   cp[7], cp[9] / nr, cp[8] / nr, cp[0] / nr, cp[1] / nr, cp[2] / nr, cp[3] / nr, cp[4] / nr, cp[5] / nr, cp[6] / nr, cp[10] / nr, cp[11] / nr);
    }
    {
      unsigned long long d2[5];
      cudaMemcpy(d2, c.prof + 3100, sizeof d2, cudaMemcpyDeviceToHost);
      if (d2[0]) std::fprintf(stderr, "\n[dbg] post-commit sightings=%llu last round=%llu go=%llu etrav=%llu k=%llu", d2[0], d2[1], d2[2], d2[3], d2[4]);
      unsigned long long d5[4];
      cudaMemcpy(d5, c.prof + 3500, sizeof d5, cudaMemcpyDeviceToHost);
      std::fprintf(stderr, "\n[dbg] verify per warp: max=%.0f mean=%.0f iters/round=%.1f xyz calls/round=%.2f", d5[0] / R, d5[1] / R, d5[2] / R, d5[3] / R);
      unsigned long long lt[18];
      cudaMemcpy(lt, c.prof + 3600, sizeof lt, cudaMemcpyDeviceToHost);
      if (lt[12] && lt[14] && lt[17])
        std::fprintf(stderr, "\n[dbg] latency ns: publish->CTA sees D mean=%.0f max=%.0f; publish->slot result mean=%.0f; publish->last result (per round) mean=%.0f; publish->sequencer has all mean=%.0f",
                     (double)lt[10] / lt[12], (double)lt[11], (double)lt[13] / lt[14], (double)lt[16] / lt[17], (double)lt[15] / lt[17]);
      unsigned long long pd[4];
      cudaMemcpy(pd, c.prof + 3680, sizeof pd, cudaMemcpyDeviceToHost);
      if (pd[2])
        std::fprintf(stderr, "\n[dbg] decision poll (per CTA-round): header words seen %.0f ns after publish, then %.0f ns until the state flags allowed it; flags held it > 300 ns in %.1f %% of polls",
                     (double)pd[0] / pd[2], (double)pd[1] / pd[2], 100.0 * pd[3] / pd[2]);
      unsigned long long gq[17];
      cudaMemcpy(gq, c.prof + 3640, sizeof gq, cudaMemcpyDeviceToHost);
      if (gq[7])
        std::fprintf(stderr, "\n[dbg] after go (ns): close wait starts=%.0f e updates done=%.0f commits done=%.0f decision published=%.0f",
                     (double)gq[4] / gq[7], (double)gq[5] / gq[7], (double)gq[6] / gq[7], (double)gq[8] / gq[7]);
      if (gq[10]) std::fprintf(stderr, "; committer released sflag=%.0f", (double)gq[9] / gq[10]);
      if (gq[12] && gq[14] && gq[16])
        std::fprintf(stderr, "; e-update group done (mean)=%.0f committer sees go=%.0f sees e done=%.0f",
                     (double)gq[11] / gq[12], (double)gq[15] / gq[16], (double)gq[13] / gq[14]);
      unsigned long long tq[80];
      cudaMemcpy(tq, c.prof + 3660, sizeof tq, cudaMemcpyDeviceToHost);
      std::fprintf(stderr, "\n[dbg] commit order causes:");
      for (int q = 0; q < 64; ++q)
        if (tq[q]) std::fprintf(stderr, " %s%d.%d=%llu", q < 9 ? "cell" : (q < 18 ? "brick" : (q < 43 ? "part" : "?")),
                                q < 18 ? (q % 9) / 3 : (q - 18) / 5, q < 18 ? q % 3 : (q - 18) % 5, tq[q]);
      std::fprintf(stderr, " | kinds(later,earlier):");
      for (int q = 0; q < 9; ++q) if (tq[70 + q]) std::fprintf(stderr, " %d,%d=%llu", q / 3, q % 3, tq[70 + q]);
      unsigned long long d4[4];
      cudaMemcpy(d4, c.prof + 3400, sizeof d4, cudaMemcpyDeviceToHost);
      std::fprintf(stderr, "\n[dbg] barrier: tid0 wait=%.0f last-arrival-after-tid0=%.0f", d4[3] / R, d4[2] / R);
      unsigned long long d3[4];
      cudaMemcpy(d3, c.prof + 3110, sizeof d3, cudaMemcpyDeviceToHost);
      if (d3[0]) std::fprintf(stderr, "\n[dbg] eval sightings=%llu round=%llu go=%llu sflag=%llu", d3[0], d3[1], d3[2], d3[3]);
    }
    if (std::getenv("GCMC_ROUND_LOG")) {
      { unsigned long long el[604]; cudaMemcpy(el, c.prof + 3300, sizeof el, cudaMemcpyDeviceToHost);
        for (unsigned long long q = 0; q < el[0] && q < 150; ++q) std::fprintf(stderr, "\n[eupd] r=%llu k=%llu kind=%llu nb=%llu cand=%llu", el[4 + 4 * q], el[5 + 4 * q] & 255, el[5 + 4 * q] >> 8, el[6 + 4 * q], el[7 + 4 * q]); }
      unsigned long long dbg[8];
      cudaMemcpy(dbg, c.prof + 3000, sizeof dbg, cudaMemcpyDeviceToHost);
      std::fprintf(stderr, "\n[dbg] near=%llu flag=%llu nacc=%llu pn=%llx pt1=%llx reach=%llu pt0=%llx base=%llu",
                   dbg[0], dbg[1], dbg[2], dbg[3], dbg[4], dbg[5], dbg[6], dbg[7]);
      std::vector<unsigned long long> rl(800);
      cudaMemcpy(rl.data(), c.prof + 256, 800 * 8, cudaMemcpyDeviceToHost);
      for (int q = 1; q < 40; ++q)
        std::fprintf(stderr, "\n[round %d] base=%llu len=%llu nacc=%llu cmin=%llu why=%llu", q, rl[4 * q],
                     rl[4 * q + 1], rl[4 * q + 2] & 0xffff, rl[4 * q + 2] >> 16, rl[4 * q + 3]);
    }
    std::fprintf(stderr, "\n[engine prof] commit task (per move, %llu): atab=%.0f commit=%.0f setup+waits=%.0f traverse=%.0f\n",
                 xp[68], xp[64] / ne, xp[65] / ne, xp[66] / ne, xp[67] / ne);
  }
  if (c.stamp) {
    std::vector<unsigned long long> st(8 * 8192);
    cudaMemcpy(st.data(), c.stamp, st.size() * 8, cudaMemcpyDeviceToHost);
    double a0 = 0, a1 = 0, a2 = 0, a3 = 0, a4 = 0, a5 = 0;
    int cnt = 0;
    for (int k = 2; k < 8192 && k < (int)hp[15]; ++k) {
      const unsigned long long* e = &st[8 * k];
      if (!e[0] || e[1] == ~0ull || !e[3] || !e[4] || !e[7]) continue;
      a0 += (double)(long long)(e[1] - e[0]);
      a1 += (double)(long long)(e[2] - e[0]);
      a2 += (double)(long long)(e[3] - e[0]);
      a3 += (double)(long long)(e[4] - e[3]);
      a4 += (double)(long long)(e[5] - e[0]);
      a5 += (double)e[6] / (double)e[7];
      ++cnt;
    }
    if (cnt)
      std::fprintf(stderr, "[engine prof] latency ns (%d rounds): publish->first CTA sees D=%.0f ->last CTA sees D=%.0f ->first result=%.0f ->mean result=%.0f ->last result=%.0f; last result->sequencer has all=%.0f\n",
                   cnt, a0 / cnt, a1 / cnt, a4 / cnt, a5 / cnt, a2 / cnt, a3 / cnt);
  }
}
#undef CKV
#else
void profile_arm(Chain&) {}
void profile_report(Chain&) {}
#endif

}  // namespace

extern "C" {

const char* gcmc_last_error(void) { return g_last_error.c_str(); }
const char* gcmc_version(void) { return "gcmc_b200 0.1 (sm_100a)"; }

gcmc_status gcmc_create(const gcmc_params* params, int device, gcmc_dev** out) {
  if (!params || !out) return set_error(GCMC_ARG, "null argument");
  *out = nullptr;
  gcmc_status s = validate(*params);
  if (s) return s;
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev), "device count");
  if (device < 0 || device >= ndev) return set_error(GCMC_ARG, "invalid device ordinal");
  CK(cudaSetDevice(device), "set device");
  auto* c = new Chain();
  c->device = device;
  c->params = *params;
  const gcmc_params& P = c->params;
  // Box / LJ constants (potential.hpp:17-27, box.hpp:47)
  c->box.l = P.box_length;
  c->box.inv_l = 1.0 / P.box_length;
  c->box.eps = P.epsilon;
  c->box.sigma = P.sigma;
  c->box.sigma2 = P.sigma * P.sigma;
  c->box.rc = P.r_cut;
  c->box.rc2 = P.r_cut * P.r_cut;
  c->box.four_eps = 4.0 * P.epsilon;
  c->box.tf_eps = 24.0 * P.epsilon;
  c->box.pad = 1e-9 * P.sigma;
  c->box.inv_sigma = 1.0 / P.sigma;
  // Grid geometry
  Grid& g = c->grid;
  g.kind = P.strategy;
  if (g.kind == GCMC_MICROCELL) {  // microcell_grid.hpp:29-35, 149
    const double cells = P.box_length / P.sigma;
    const double whole = std::floor(cells);
    const double frac = cells - whole;
    if (frac < 1e-9) {
      g.dims = (int)std::llround(whole);
      g.last_w = 1.0;
    } else {
      g.dims = (int)whole + 1;
      g.last_w = frac;
    }
    g.inv_cell = 1.0 / P.sigma;
    g.cap = P.microcell_capacity > 0 ? P.microcell_capacity : 5;
  } else if (g.kind == GCMC_CELL_LIST) {  // cell_grid.hpp:27-38
    int t = (int)(P.box_length / P.r_cut);
    while ((double)(t + 1) * P.r_cut <= P.box_length) ++t;
    while (t > 1 && (double)t * P.r_cut > P.box_length) --t;
    if (t < 3) t = 3;
    g.dims = t;
    g.inv_cell = 1.0 / (P.box_length / t);
    g.cap = P.cell_capacity > 0 ? P.cell_capacity : (P.r_cut <= 4.0 * P.sigma ? 48 : 96);
    g.last_w = 1.0;
  }
  if (g.cap > kMaxCap) {
    delete c;
    return set_error(GCMC_ARG, "cell capacity above the device limit of 128");
  }
  g.ncells = g.kind == GCMC_ALL_PAIRS ? 0 : (uint64_t)g.dims * g.dims * g.dims;
  if ((uint64_t)g.cap * g.ncells >= (1ull << 31)) {
    delete c;
    return set_error(GCMC_ARG, "grid too large (cap * cells must be < 2^31)");
  }
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, device), "props");
  c->sm_count = prop.multiProcessorCount;
  // Engine shape (engine.cu): one persistent CTA per SM, 1 sequencer + evaluators.
  c->engine_group = P.engine_group == 128 || P.engine_group == 512 ? P.engine_group : 256;
  c->engine2_group = P.engine_group == 256 || P.engine_group == 512 ? P.engine_group : 128;
  if (const char* eg = knob("GCMC_ENGINE_GROUP")) {  // experiments
    const int v = std::atoi(eg);
    if (v == 128 || v == 256 || v == 512) c->engine_group = c->engine2_group = v;
  }
  // one SM is left to generate the next batch of proposals concurrently
  c->engine_ctas = P.engine_ctas > 1 && P.engine_ctas <= c->sm_count ? P.engine_ctas : c->sm_count - 1;
  if (P.engine_ctas <= 1 && P.engine_share > 1) {  // K chains on one device: 1/K of the SMs each
    c->engine_ctas = (c->sm_count - P.engine_share) / P.engine_share;
    if (c->engine_ctas < 2 && (P.engine_mode == 2 || (P.engine_mode == 0 && P.engine_share >= 12)))
      c->engine_ctas = 2;  // (the chain-per-SM engine runs instead: one CTA per chain)
    if (c->engine_ctas < 2) {
      delete c;
      return set_error(GCMC_ARG, "engine_share: too many chains for this device");
    }
  }
  {
    const int mg = 512 / c->engine_group;
    const int max_ctas = 1 + engine_max_slots() / mg;
    if (c->engine_ctas > max_ctas) c->engine_ctas = max_ctas;
  }
  // engine2: in a small box the moves of a round conflict early (positions
  // within r_c, accepted moves within 2 r_c), so most evaluations of a full
  // round are discarded and only lengthen it. About one slot per 3 r_c^3 of
  // box, at least 64: 2k (L = 14.5) gets 18 CTAs, 2.5x the moves/s of the whole
  // GPU at mu = -2 and the same at mu = +1; from 32k up all CTAs.
  c->engine2_ctas = c->engine_ctas;
  if (P.engine_ctas <= 1) {
    const double rc3 = P.r_cut * P.r_cut * P.r_cut;
    const double want = std::max(64.0, P.box_length * P.box_length * P.box_length / (3.0 * rc3));
    const int mg2 = 512 / c->engine2_group;
    const double ctas = 1.0 + std::ceil(want / mg2);
    if (ctas < (double)c->engine2_ctas) c->engine2_ctas = (int)ctas;
  }
  c->engine_variants = P.engine_variants > 0 ? (P.engine_variants > 15 ? 15 : P.engine_variants) : 11;
  c->engine_bias = P.engine_bias > 0 ? 1 : -1;
  // Evaluation mirror: bricks of side L/dims >= r_cut (1e-9 relative margin).
  {
    Mirror& m = c->mirror;
    int d = (int)std::floor(P.box_length / (P.r_cut * (1.0 + 1e-9)));
    if (d < 1) d = 1;
    if (d > 255) d = 255;  // packed 8-bit brick coordinates (mirror.cuh)
    m.dims = d;
    m.nb = (uint32_t)d * d * d;
    m.side = P.box_length / d;
    m.inv = (double)d / P.box_length;
    // records per brick: generous over the densest LJ states (rho <= ~1.2)
    const double vb = m.side * m.side * m.side / (P.sigma * P.sigma * P.sigma);
    // (~2.4x the mean occupancy at rho = 1: 32 at the r_cut = 2.5 sigma bricks)
    int cap = (int)std::ceil(vb * 1.6);
    if (cap < 32) cap = 32;
    if (cap > 128) cap = 128;
    m.cap = cap;
    // conflict reach: the window (1 brick) and any reference cell
    double ref_side = 0.0;
    if (g.kind == GCMC_MICROCELL) ref_side = P.sigma;
    if (g.kind == GCMC_CELL_LIST) ref_side = P.box_length / g.dims;
    int reach = (int)std::ceil(ref_side / m.side);
    m.reach = reach < 1 ? 1 : reach;
  }
  // Store capacity: the store can never outgrow the reference grid or the
  // mirror (either overflows first), so by default it holds exactly that many
  // particles; gcmc_run_moves grows it (with the mirror) if they grow.
  c->capn = std::max<uint64_t>(P.max_particles, store_bound(*c));
  if (c->capn >= (1ull << 31)) {  // particle ids are int32 in the grids and the engine's words
    delete c;
    return set_error(GCMC_ARG, "store capacity must be < 2^31 particles");
  }
  CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking), "stream");
  CK(cudaStreamCreateWithFlags(&c->gen_stream, cudaStreamNonBlocking), "stream");
  for (auto& ev : c->ev) CK(cudaEventCreate(&ev), "event");
  for (auto& ev : c->ev_e) CK(cudaEventCreate(&ev), "event");
  CK(cudaEventCreateWithFlags(&c->ev_mt, cudaEventDisableTiming), "event");
  CK(cudaEventCreateWithFlags(&c->ev_ahead, cudaEventDisableTiming), "event");
  if ((s = arena_alloc(*c, c->mirror.cap, c->capn, false))) return s;
  if (g.ncells) {
    CK(cudaMalloc(&g.occ, g.ncells * sizeof(int32_t)), "alloc occ");
    CK(cudaMalloc(&g.slots, g.ncells * g.cap * sizeof(int32_t)), "alloc slots");
    CK(cudaMemset(g.occ, 0, g.ncells * sizeof(int32_t)), "memset");
    CK(cudaMemset(g.slots, 0xff, g.ncells * g.cap * sizeof(int32_t)), "memset");  // -1
  }
  {
    size_t bd, br, be;
    engine_buffer_bytes(engine_max_slots(), &bd, &br, &be);
    CK(cudaMalloc(&c->eng_dec, bd), "alloc engine");
    CK(cudaMalloc(&c->eng_res, br), "alloc engine");
    CK(cudaMalloc(&c->eng_ext, be), "alloc engine");
  }
  CK(cudaMalloc(&c->st, sizeof(ChainState)), "alloc state");
  CK(cudaMallocHost(&c->st_host, sizeof(ChainState)), "alloc state");
  std::memset(c->st_host, 0, sizeof(ChainState));
  CK(cudaMalloc(&c->mt, 314 * sizeof(uint64_t)), "alloc rng");
  CK(cudaMalloc(&c->mt_next, 314 * sizeof(uint64_t)), "alloc rng");
  if ((s = ensure_batch(*c, 1024))) return s;
  sync_state_to_device(*c);
  *out = reinterpret_cast<gcmc_dev*>(c);
  return gcmc_seed_rng(*out, 1);  // RunConfig::seed default (config.hpp:56)
}

gcmc_status gcmc_destroy(gcmc_dev* h) {
  if (!h) return GCMC_OK;
  Chain* c = H(h);
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  cudaStreamSynchronize(c->gen_stream);
  cudaFree(c->arena);
  cudaFree(c->props_next);
  cudaFree(c->mt_next);
  cudaEventDestroy(c->ev_mt);
  cudaEventDestroy(c->ev_ahead);
  cudaFree(c->grid.occ);
  cudaFree(c->grid.slots);
  cudaFree(c->rslot);
  cudaFree(c->ep);
  cudaFree(c->eng2_buf);
  cudaFree(c->mirror.rid);
  cudaFree(c->eng_dec);
  cudaFree(c->eng_res);
  cudaFree(c->eng_ext);
  cudaFree(c->st);
  cudaFreeHost(c->st_host);
  cudaFree(c->mt);
  cudaFree(c->props);
  cudaFree(c->trace);
  cudaFree(c->dscratch);
  cudaFree(c->iscratch);
  cudaFree(c->egrid);
  for (auto& ev : c->ev) cudaEventDestroy(ev);
  for (auto& ev : c->ev_e) cudaEventDestroy(ev);
  cudaStreamDestroy(c->stream);
  cudaStreamDestroy(c->gen_stream);
  delete c;
  return GCMC_OK;
}

gcmc_status gcmc_upload_positions(gcmc_dev* h, const double* xyz, uint64_t n) {
  Chain& c = *H(h);
  cudaSetDevice(c.device);
  if (n && !xyz) return set_error(GCMC_ARG, "null positions");
  if (n >= (1ull << 31)) return set_error(GCMC_ARG, "store capacity must be < 2^31 particles");
  gcmc_status s = pull_state(c);
  if (s) return s;
  if (n > c.capn && (s = arena_alloc(c, c.mirror.cap, n, false))) return s;
  std::vector<double4> tmp(n);
  for (uint64_t i = 0; i < n; ++i) tmp[i] = make_double4(xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2], 0.0);
  if (n) CK(cudaMemcpyAsync(c.pos, tmp.data(), n * sizeof(double4), cudaMemcpyHostToDevice, c.stream), "upload");
  // a new store under a new strategy: every slot reads -1 before the binning
  // (the reference's grid ctors; build() itself only resets the occupancy,
  // microcell_grid.hpp:194-198, cell_grid.hpp:88-92)
  if (c.grid.ncells)
    CK(cudaMemsetAsync(c.grid.slots, 0xff, c.grid.ncells * c.grid.cap * sizeof(int32_t), c.stream),
       "upload");
  c.st_host->n = n;
  c.st_host->peak = 0;
  c.st_host->error = 0;
  sync_state_to_device(c);
  return build_growing(c);
}

gcmc_status gcmc_download_positions(gcmc_dev* h, double* xyz, uint64_t capacity, uint64_t* n) {
  Chain& c = *H(h);
  cudaSetDevice(c.device);
  gcmc_status s = pull_state(c);
  if (s) return s;
  const uint64_t cnt = c.st_host->n;
  if (n) *n = cnt;
  if (!xyz) return GCMC_OK;
  if (capacity < cnt) return set_error(GCMC_ARG, "position buffer too small");
  std::vector<double4> tmp(cnt);
  if (cnt) CK(cudaMemcpy(tmp.data(), c.pos, cnt * sizeof(double4), cudaMemcpyDeviceToHost), "download");
  for (uint64_t i = 0; i < cnt; ++i) {
    xyz[3 * i] = tmp[i].x;
    xyz[3 * i + 1] = tmp[i].y;
    xyz[3 * i + 2] = tmp[i].z;
  }
  return GCMC_OK;
}

gcmc_status gcmc_store_set(gcmc_dev* h, uint64_t pid, const double pos[3]) {
  Chain& c = *H(h);
  cudaSetDevice(c.device);
  if (!pos) return set_error(GCMC_ARG, "null position");
  gcmc_status s = pull_state(c);
  if (s) return s;
  if (pid >= c.st_host->n) return set_error(GCMC_INVALID_PID, "store: invalid particle id");
  // x, y, z only: the grid, the mirror and its back-pointer word stay as they are
  CK(cudaMemcpyAsync(reinterpret_cast<double*>(c.pos + pid), pos, 3 * sizeof(double),
                     cudaMemcpyHostToDevice, c.stream), "store set");
  CK(cudaStreamSynchronize(c.stream), "store set");
  return GCMC_OK;
}

gcmc_status gcmc_build(gcmc_dev* h) {
  Chain& c = *H(h);
  cudaSetDevice(c.device);
  gcmc_status s = pull_state(c);
  if (s) return s;
  return build_growing(c);
}

gcmc_status gcmc_grid_info(gcmc_dev* h, int32_t* dims, int32_t* capacity, uint64_t* ncells) {
  Chain& c = *H(h);
  if (dims) *dims = c.grid.dims;
  if (capacity) *capacity = c.grid.cap;
  if (ncells) *ncells = c.grid.ncells;
  return GCMC_OK;
}

gcmc_status gcmc_download_grid(gcmc_dev* h, int32_t* occ, int32_t* slots) {
  Chain& c = *H(h);
  cudaSetDevice(c.device);
  if (!c.grid.ncells) return GCMC_OK;
  CK(cudaStreamSynchronize(c.stream), "download grid");
  if (occ) CK(cudaMemcpy(occ, c.grid.occ, c.grid.ncells * 4, cudaMemcpyDeviceToHost), "download grid");
  if (slots)
    CK(cudaMemcpy(slots, c.grid.slots, c.grid.ncells * c.grid.cap * 4, cudaMemcpyDeviceToHost),
       "download grid");
  return GCMC_OK;
}

gcmc_status gcmc_rebuild_check(gcmc_dev* h, char* msg, size_t msg_cap, int32_t* clean) {
  Chain& c = *H(h);
  cudaSetDevice(c.device);
  gcmc_status s = pull_state(c);
  if (s) return s;
  std::string issue;
  s = grid_check(c, &issue);
  if (s) return s;
  if (clean) *clean = issue.empty() ? 1 : 0;
  if (msg && msg_cap) {
    std::strncpy(msg, issue.c_str(), msg_cap - 1);
    msg[msg_cap - 1] = 0;
  }
  return GCMC_OK;
}

gcmc_status gcmc_peak_occupancy(gcmc_dev* h, int32_t* peak) {
  Chain& c = *H(h);
  cudaSetDevice(c.device);
  gcmc_status s = pull_state(c);
  if (s) return s;
  *peak = c.st_host->peak;
  return GCMC_OK;
}

gcmc_status gcmc_delta_batch(gcmc_dev* h, uint64_t n, const int32_t* kinds, const uint64_t* pids,
                             const double* xyz, double* du, double* dw) {
  Chain& c = *H(h);
  cudaSetDevice(c.device);
  if (n == 0) return GCMC_OK;
  gcmc_status s = pull_state(c);
  if (s) return s;
  for (uint64_t i = 0; i < n; ++i) {
    if (kinds[i] < 0 || kinds[i] > 2) return set_error(GCMC_ARG, "bad move kind");
    if (kinds[i] != 1 && pids[i] >= c.st_host->n) return invalid_pid(c);
  }
  if ((s = ensure_batch(c, n))) return s;
  double* d_du = c.dscratch;
  double* d_dw = d_du + c.batch_cap;
  double* d_xyz = d_dw + c.batch_cap;
  uint64_t* d_pid = reinterpret_cast<uint64_t*>(d_xyz + 3 * c.batch_cap);
  int32_t* d_kind = c.iscratch;
  std::vector<double> xyz_buf(3 * n, 0.0);
  std::vector<uint64_t> pid_buf(n, 0);
  for (uint64_t i = 0; i < n; ++i) {
    if (xyz) for (int k = 0; k < 3; ++k) xyz_buf[3 * i + k] = xyz[3 * i + k];
    if (pids) pid_buf[i] = pids[i];
  }
  CK(cudaMemcpyAsync(d_kind, kinds, n * 4, cudaMemcpyHostToDevice, c.stream), "delta");
  CK(cudaMemcpyAsync(d_pid, pid_buf.data(), n * 8, cudaMemcpyHostToDevice, c.stream), "delta");
  CK(cudaMemcpyAsync(d_xyz, xyz_buf.data(), n * 24, cudaMemcpyHostToDevice, c.stream), "delta");
  if ((s = delta_batch(c, n, d_kind, d_pid, d_xyz, d_du, d_dw))) return s;
  CK(cudaMemcpyAsync(du, d_du, n * 8, cudaMemcpyDeviceToHost, c.stream), "delta");
  CK(cudaMemcpyAsync(dw, d_dw, n * 8, cudaMemcpyDeviceToHost, c.stream), "delta");
  CK(cudaStreamSynchronize(c.stream), "delta");
  return GCMC_OK;
}

gcmc_status gcmc_delta_displace(gcmc_dev* h, uint64_t pid, const double pos[3], double* du,
                                double* dw) {
  const int32_t k = 0;
  return gcmc_delta_batch(h, 1, &k, &pid, pos, du, dw);
}

gcmc_status gcmc_delta_insert(gcmc_dev* h, const double pos[3], double* du, double* dw) {
  const int32_t k = 1;
  const uint64_t pid = 0;
  return gcmc_delta_batch(h, 1, &k, &pid, pos, du, dw);
}

gcmc_status gcmc_delta_delete(gcmc_dev* h, uint64_t pid, double* du, double* dw) {
  const int32_t k = 2;
  const double z[3] = {0, 0, 0};
  return gcmc_delta_batch(h, 1, &k, &pid, z, du, dw);
}

gcmc_status gcmc_commit_displace(gcmc_dev* h, uint64_t pid, const double pos[3]) {
  Chain& c = *H(h);
  cudaSetDevice(c.device);
  gcmc_status s = pull_state(c);
  if (s) return s;
  if (pid >= c.st_host->n) return invalid_pid(c);
  return commit_one(c, 0, pid, pos, nullptr);
}

gcmc_status gcmc_commit_insert(gcmc_dev* h, const double pos[3], uint64_t* pid) {
  Chain& c = *H(h);
  cudaSetDevice(c.device);
  gcmc_status s = pull_state(c);
  if (s) return s;
  if (c.st_host->n + 1 > c.capn) return set_error(GCMC_ARG, "store capacity exhausted");
  return commit_one(c, 1, 0, pos, pid);
}

gcmc_status gcmc_commit_delete(gcmc_dev* h, uint64_t pid) {
  Chain& c = *H(h);
  cudaSetDevice(c.device);
  gcmc_status s = pull_state(c);
  if (s) return s;
  if (pid >= c.st_host->n) return invalid_pid(c);
  return commit_one(c, 2, pid, nullptr, nullptr);
}

gcmc_status gcmc_total_energy(gcmc_dev* h, double* u, double* w) {
  Chain& c = *H(h);
  cudaSetDevice(c.device);
  gcmc_status s = pull_state(c);
  if (s) return s;
  return total_energy(c, u, w);
}

extern "C" gcmc_status gcmc_debug_energies(gcmc_dev* h, double* maint, double* fresh) {
  Chain& c = *H(h);
  cudaSetDevice(c.device);
  gcmc_status s = pull_state(c);
  if (s) return s;
  return epart_dump(c, maint, fresh);
}

gcmc_status gcmc_total_energy_bruteforce(gcmc_dev* h, double* u, double* w) {
  Chain& c = *H(h);
  cudaSetDevice(c.device);
  gcmc_status s = pull_state(c);
  if (s) return s;
  return total_energy_bruteforce(c, u, w);
}

gcmc_status gcmc_energy_timing(gcmc_dev* h, double* pass_ms, double* kernel_ms) {
  Chain& c = *H(h);
  if (pass_ms) *pass_ms = c.energy_ms[0];
  if (kernel_ms) *kernel_ms = c.energy_ms[1];
  return GCMC_OK;
}

gcmc_status gcmc_energy_drift(gcmc_dev* h, double* max_du, double* max_dw) {
  Chain& c = *H(h);
  cudaSetDevice(c.device);
  gcmc_status s = pull_state(c);
  if (s) return s;
  return epart_drift(c, max_du, max_dw);
}

gcmc_status gcmc_seed_rng(gcmc_dev* h, uint64_t seed) {
  std::mt19937_64 eng(seed);  // RngStream(seed) (rng.hpp:23)
  std::ostringstream os;
  os << eng;
  std::istringstream is(os.str());
  uint64_t words[313];
  for (auto& w : words) is >> w;
  return gcmc_set_rng_state(h, words, words[312], 0);
}

gcmc_status gcmc_set_rng_state(gcmc_dev* h, const uint64_t words[312], uint64_t index,
                               uint64_t draws) {
  Chain& c = *H(h);
  cudaSetDevice(c.device);
  if (index > 312) return set_error(GCMC_ARG, "rng state: bad position");
  uint64_t buf[314];
  std::memcpy(buf, words, 312 * 8);
  buf[312] = index;
  buf[313] = draws;
  c.ahead_n = 0;  // proposals generated ahead belong to the old stream
  CK(cudaStreamSynchronize(c.gen_stream), "rng");
  CK(cudaMemcpyAsync(c.mt, buf, sizeof buf, cudaMemcpyHostToDevice, c.stream), "rng");
  CK(cudaStreamSynchronize(c.stream), "rng");
  return GCMC_OK;
}

gcmc_status gcmc_get_rng_state(gcmc_dev* h, uint64_t words[312], uint64_t* index,
                               uint64_t* draws) {
  Chain& c = *H(h);
  cudaSetDevice(c.device);
  uint64_t buf[314];
  CK(cudaMemcpyAsync(buf, c.mt, sizeof buf, cudaMemcpyDeviceToHost, c.stream), "rng");
  CK(cudaStreamSynchronize(c.stream), "rng");
  if (words) std::memcpy(words, buf, 312 * 8);
  if (index) *index = buf[312];
  if (draws) *draws = buf[313];
  return GCMC_OK;
}

gcmc_status gcmc_set_state(gcmc_dev* h, const gcmc_state* s_in) {
  Chain& c = *H(h);
  cudaSetDevice(c.device);
  gcmc_status s = pull_state(c);
  if (s) return s;
  ChainState& st = *c.st_host;
  st.step = s_in->step;
  st.energy = s_in->energy;
  st.virial = s_in->virial;
  for (int k = 0; k < 3; ++k) {
    st.attempted[k] = s_in->attempted[k];
    st.accepted[k] = s_in->accepted[k];
  }
  st.samples = s_in->samples;
  st.sum_u = s_in->sum_u;
  st.sum_p = s_in->sum_p;
  st.sum_n = s_in->sum_n;
  st.sum_n2 = s_in->sum_n2;
  sync_state_to_device(c);
  CK(cudaStreamSynchronize(c.stream), "state");
  return GCMC_OK;
}

gcmc_status gcmc_get_state(gcmc_dev* h, gcmc_state* out) {
  Chain& c = *H(h);
  cudaSetDevice(c.device);
  gcmc_status s = pull_state(c);
  if (s) return s;
  const ChainState& st = *c.st_host;
  out->step = st.step;
  out->n = st.n;
  out->energy = st.energy;
  out->virial = st.virial;
  for (int k = 0; k < 3; ++k) {
    out->attempted[k] = st.attempted[k];
    out->accepted[k] = st.accepted[k];
  }
  out->samples = st.samples;
  out->sum_u = st.sum_u;
  out->sum_p = st.sum_p;
  out->sum_n = st.sum_n;
  out->sum_n2 = st.sum_n2;
  out->peak_occupancy = st.peak;
  out->pad = 0;
  return GCMC_OK;
}

// Proposal buffers for chunks of up to chunk_cap moves.
gcmc_status props_reserve(Chain& c, uint64_t chunk_cap, bool trace) {
  if (chunk_cap > c.props_cap) {
    CK(cudaStreamSynchronize(c.gen_stream), "proposals");
    cudaFree(c.props);
    cudaFree(c.props_next);
    c.props = c.props_next = nullptr;
    CK(cudaMalloc(&c.props, chunk_cap * sizeof(Proposal)), "alloc proposals");
    CK(cudaMalloc(&c.props_next, chunk_cap * sizeof(Proposal)), "alloc proposals");
    c.props_cap = chunk_cap;
    c.ahead_n = 0;
  }
  if (trace && chunk_cap > c.trace_cap) {
    cudaFree(c.trace);
    c.trace = nullptr;
    CK(cudaMalloc(&c.trace, chunk_cap * sizeof(gcmc_trace_rec)), "alloc trace");
    c.trace_cap = chunk_cap;
  }
  return GCMC_OK;
}

// The proposals of the next m moves into c.props (generated during the
// previous chunk when it had the same size), then the chunk after it (mn
// moves) on the SM the engine leaves free.
gcmc_status props_next_chunk(Chain& c, uint64_t m, uint64_t mn) {
  gcmc_status s = GCMC_OK;
  CK(cudaEventRecord(c.ev[0], c.stream), "event");
  if (c.ahead_n == m) {  // generated during the previous batch
    CK(cudaStreamWaitEvent(c.stream, c.ev_ahead, 0), "ahead");
    std::swap(c.props, c.props_next);
    std::swap(c.mt, c.mt_next);
  } else {
    // a look-ahead copy of c.mt may still be in flight on gen_stream
    CK(cudaStreamWaitEvent(c.stream, c.ev_ahead, 0), "ahead");
    if ((s = gen_proposals(c, m, c.stream))) return s;
  }
  c.ahead_n = 0;
  CK(cudaEventRecord(c.ev_mt, c.stream), "ahead");
  CK(cudaStreamWaitEvent(c.gen_stream, c.ev_mt, 0), "ahead");
  CK(cudaMemcpyAsync(c.mt_next, c.mt, 314 * sizeof(uint64_t), cudaMemcpyDeviceToDevice, c.gen_stream),
     "ahead");
  if ((s = gen_proposals_into(c, c.mt_next, c.props_next, mn, c.gen_stream))) return s;
  CK(cudaEventRecord(c.ev_ahead, c.gen_stream), "ahead");
  c.ahead_n = mn;
  return GCMC_OK;
}

// Moves [off, m) of the chunk in c.props on the chain's own engine. When the
// evaluation mirror (not the reference grid) runs out of records in a brick,
// the engine stops before the move that overflowed with everything before it
// committed: the mirror's records per brick double and the chunk continues
// there, so the mirror never fails a state the reference accepts (up to
// kMaxCap).
gcmc_status run_chunk_from(Chain& c, uint64_t m, uint64_t off, gcmc_trace_rec* trace_d, float& eng_ms,
                           uint64_t& rounds) {
  gcmc_status s = GCMC_OK;
  for (;;) {
    if ((s = ensure_store(c, m - off))) return s;
    profile_arm(c);
    Proposal* const p0 = c.props;
    c.props += off;
    CK(cudaEventRecord(c.ev[1], c.stream), "event");
    s = engine_run(c, m - off, trace_d ? trace_d + off : nullptr, c.stream);
    c.props = p0;
    if (s) return s;
    CK(cudaEventRecord(c.ev[2], c.stream), "event");
    if ((s = pull_state(c))) return s;
    float b = 0;
    cudaEventElapsedTime(&b, c.ev[1], c.ev[2]);
    eng_ms += b;
    rounds += c.st_host->rounds;
    profile_report(c);
    ChainState& st = *c.st_host;
    if (st.error == GCMC_CELL_OVERFLOW && st.err_c == 1 && c.mirror.cap < kMaxCap) {
      off += st.moves_done;
      st.error = 0;
      sync_state_to_device(c);
      if ((s = arena_alloc(c, std::min(kMaxCap, 2 * c.mirror.cap), c.capn, true))) return s;
      continue;
    }
    return GCMC_OK;
  }
}

// A failed chain's error in the reference's wording (clears the device flag).
gcmc_status chain_error(Chain& c) {
  const ChainState& st = *c.st_host;
  const int err = st.error;
  const int64_t ea = st.err_a, eb = st.err_b, ec = st.err_c;
  c.st_host->error = 0;
  sync_state_to_device(c);
  if (err == GCMC_CELL_OVERFLOW && ec == 1) {
    std::ostringstream os;
    os << "mirror: brick " << ea << " exceeds capacity " << c.mirror.cap
       << " (the evaluation mirror's limit; density too high)";
    return set_error(GCMC_CELL_OVERFLOW, os.str());
  }
  if (err == GCMC_CELL_OVERFLOW) return set_error(GCMC_CELL_OVERFLOW, overflow_message(c, ea, eb));
  std::ostringstream os;
  os << strategy_name(c.grid.kind) << ": particle " << ea << " not found in cell " << eb;
  return set_error((gcmc_status)err, os.str());
}

gcmc_status gcmc_run_moves(gcmc_dev* h, uint64_t n, gcmc_trace_rec* trace, gcmc_run_result* out) {
  Chain& c = *H(h);
  cudaSetDevice(c.device);
  if (!c.built) return set_error(GCMC_STATE, "grid not built (upload positions first)");
  const uint64_t kChunk = 1ull << 21;
  const uint64_t chunk_cap = n < kChunk ? (n ? n : 1) : kChunk;
  gcmc_status s = props_reserve(c, chunk_cap, trace != nullptr);
  if (s) return s;
  float gen_ms = 0.f, eng_ms = 0.f;
  uint64_t done = 0, rounds = 0;
  if (out) {  // the device counter before the call
    gcmc_status ps = pull_state(c);
    if (ps) return ps;
  }
  const unsigned long long pairs0 = c.st_host->pair_evals;
  while (done < n) {
    const uint64_t m = std::min(chunk_cap, n - done);
    const uint64_t left = n - done - m;
    if ((s = props_next_chunk(c, m, left ? std::min(chunk_cap, left) : m))) return s;
    CK(cudaEventRecord(c.ev[3], c.stream), "event");
    if ((s = run_chunk_from(c, m, 0, trace ? c.trace : nullptr, eng_ms, rounds))) return s;
    float a = 0;
    cudaEventElapsedTime(&a, c.ev[0], c.ev[3]);
    gen_ms += a;
    if (trace)
      CK(cudaMemcpyAsync(trace + done, c.trace, m * sizeof(gcmc_trace_rec), cudaMemcpyDeviceToHost,
                         c.stream),
         "trace");
    CK(cudaStreamSynchronize(c.stream), "trace");
    if (c.st_host->error) {
      c.ahead_n = 0;  // the look-ahead batch continues a stream the chain did not reach
      break;
    }
    done += m;
  }
  if (c.st_host->error) return chain_error(c);
  if (out) {
    gcmc_get_state(h, &out->state);
    out->moves = done;
    out->rounds = rounds;
    out->device_ms = eng_ms;
    out->gen_ms = gen_ms;
    out->pair_evals = c.st_host->pair_evals - pairs0;
    out->engine = c.last_engine;
    out->pad = 0;
  }
  return GCMC_OK;
}

// K chain-per-SM chains on one device in ONE launch per chunk (one CTA per
// chain): separate launches from separate streams serialise once the streams
// outnumber the device's hardware queues. The chunk's proposals of every
// chain are generated in one launch too (one CTA per chain) before it; a
// chain whose mirror overflows mid-chunk finishes that chunk on its own
// launches.
gcmc_status run_chains_sm(const std::vector<Chain*>& cs, const uint64_t* n, gcmc_run_result* out) {
  const int k = (int)cs.size();
  const uint64_t kChunk = 1ull << 21;
  gcmc_status s = GCMC_OK;
  std::vector<uint64_t> cap(k), done(k, 0), rounds(k, 0), m(k, 0);
  std::vector<float> eng_ms(k, 0.f), gen_ms(k, 0.f);
  std::vector<unsigned long long> pairs0(k);
  for (int i = 0; i < k; ++i) {
    Chain& c = *cs[i];
    if (!c.built) return set_error(GCMC_STATE, "grid not built (upload positions first)");
    cap[i] = n[i] < kChunk ? (n[i] ? n[i] : 1) : kChunk;
    if ((s = props_reserve(c, cap[i], false))) return s;
    if ((s = pull_state(c))) return s;
    pairs0[i] = c.st_host->pair_evals;
  }
  Chain& c0 = *cs[0];
  for (;;) {
    std::vector<Chain*> run;
    std::vector<uint64_t> rm;
    std::vector<int> idx;
    for (int i = 0; i < k; ++i) {
      if (done[i] >= n[i]) continue;
      m[i] = std::min(cap[i], n[i] - done[i]);
      run.push_back(cs[i]);
      rm.push_back(m[i]);
      idx.push_back(i);
    }
    if (run.empty()) break;
    // this chunk's proposals: every chain's in one launch (a look-ahead batch
    // left by gcmc_run_moves is used when it has the right size)
    CK(cudaEventRecord(c0.ev[0], c0.stream), "event");
    std::vector<Chain*> gen;
    std::vector<uint64_t> gm;
    for (size_t q = 0; q < run.size(); ++q) {
      Chain& c = *run[q];
      CK(cudaStreamWaitEvent(c0.stream, c.ev_ahead, 0), "ahead");
      if (c.ahead_n == rm[q]) {
        std::swap(c.props, c.props_next);
        std::swap(c.mt, c.mt_next);
      } else {
        gen.push_back(&c);
        gm.push_back(rm[q]);
      }
      c.ahead_n = 0;
    }
    if ((s = gen_proposals_many(gen.data(), (int)gen.size(), gm.data(), c0.stream))) return s;
    for (size_t q = 0; q < run.size(); ++q) {
      Chain& c = *run[q];
      if ((s = ensure_store(c, rm[q]))) return s;
      if (!c.e_valid) {
        if ((s = epart_build(c, c.ep))) return s;
        c.e_valid = true;
      }
      CK(cudaEventRecord(c.ev[1], c.stream), "event");
      CK(cudaStreamWaitEvent(c0.stream, c.ev[1], 0), "event");
    }
    CK(cudaEventRecord(c0.ev[3], c0.stream), "event");
    if ((s = engine_sm_run_many(run.data(), (int)run.size(), rm.data(), c0.stream))) return s;
    CK(cudaEventRecord(c0.ev[2], c0.stream), "event");
    float ems = 0.f;
    CK(cudaEventSynchronize(c0.ev[2]), "engine");
    cudaEventElapsedTime(&ems, c0.ev[3], c0.ev[2]);
    for (size_t q = 0; q < run.size(); ++q) {
      const int i = idx[q];
      Chain& c = *run[q];
      CK(cudaStreamWaitEvent(c.stream, c0.ev[2], 0), "event");
      float a = 0.f;
      cudaEventElapsedTime(&a, c0.ev[0], c0.ev[3]);
      gen_ms[i] += a;
      eng_ms[i] += ems;
      if ((s = pull_state(c))) return s;
      rounds[i] += c.st_host->rounds;
      c.last_engine = 3;
      ChainState& st = *c.st_host;
      if (st.error == GCMC_CELL_OVERFLOW && st.err_c == 1 && c.mirror.cap < kMaxCap) {
        const uint64_t off = st.moves_done;  // finish this chunk on the chain's own launches
        st.error = 0;
        sync_state_to_device(c);
        if ((s = arena_alloc(c, std::min(kMaxCap, 2 * c.mirror.cap), c.capn, true))) return s;
        if ((s = run_chunk_from(c, m[i], off, nullptr, eng_ms[i], rounds[i]))) return s;
      }
      if (c.st_host->error) {
        c.ahead_n = 0;
        const gcmc_status e = chain_error(c);
        return set_error(e, "chain " + std::to_string(i) + ": " + g_last_error);
      }
      done[i] += m[i];
    }
  }
  if (out)
    for (int i = 0; i < k; ++i) {
      Chain& c = *cs[i];
      gcmc_get_state(reinterpret_cast<gcmc_dev*>(cs[i]), &out[i].state);
      out[i].moves = done[i];
      out[i].rounds = rounds[i];
      out[i].device_ms = eng_ms[i];
      out[i].gen_ms = gen_ms[i];
      out[i].pair_evals = c.st_host->pair_evals - pairs0[i];
      out[i].engine = 3;
      out[i].pad = 0;
    }
  return GCMC_OK;
}

// K independent chains advanced concurrently ("multiple
// large-scale simulations on a single GPU simultaneously"). Each chain owns
// its streams and its engine's CTAs (gcmc_params.engine_ctas), so K engines
// share the SMs of one device; one host thread per chain drives its
// gcmc_run_moves (the host waits on a chain's stream between its batches, not
// on the other chains). Every chain follows exactly the trajectory it would
// follow alone.
gcmc_status gcmc_run_chains(gcmc_dev* const* hs, int32_t k, const uint64_t* n, gcmc_run_result* out) {
  if (k < 0 || (k > 0 && (!hs || !n))) return set_error(GCMC_ARG, "null argument");
  for (int32_t i = 0; i < k; ++i) {
    if (!hs[i]) return set_error(GCMC_ARG, "null chain handle");
    for (int32_t j = 0; j < i; ++j)
      if (hs[j] == hs[i]) return set_error(GCMC_ARG, "a chain appears twice");
  }
  if (k == 1) return gcmc_run_moves(hs[0], n[0], nullptr, out);
  {  // chain-per-SM chains on one device: one launch for all of them
    std::vector<Chain*> cs;
    bool batch = true;
    for (int32_t i = 0; i < k; ++i) {
      Chain* c = H(hs[i]);
      batch = batch && c->device == H(hs[0])->device && engine_sm_supported(*c);
      cs.push_back(c);
    }
    if (batch) {
      cudaSetDevice(cs[0]->device);
      return run_chains_sm(cs, n, out);
    }
  }
  std::vector<gcmc_status> st(k, GCMC_OK);
  std::vector<std::string> msg(k);
  std::vector<std::thread> th;
  th.reserve(k);
  for (int32_t i = 0; i < k; ++i)
    th.emplace_back([&, i]() {
      st[i] = gcmc_run_moves(hs[i], n[i], nullptr, out ? out + i : nullptr);
      if (st[i]) msg[i] = g_last_error;  // thread-local: carried to the caller's thread
    });
  for (auto& t : th) t.join();
  for (int32_t i = 0; i < k; ++i)
    if (st[i]) return set_error(st[i], "chain " + std::to_string(i) + ": " + msg[i]);
  return GCMC_OK;
}

gcmc_status gcmc_device_initial_configuration(int device, uint64_t n, double box_length, double min_sep,
                                              uint64_t seed, double* out_xyz, uint64_t words[312],
                                              uint64_t* index, uint64_t* draws) {
  if (n && !out_xyz) return set_error(GCMC_ARG, "null positions");
  if (!words || !index) return set_error(GCMC_ARG, "null argument");
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev), "device count");
  if (device < 0 || device >= ndev) return set_error(GCMC_ARG, "invalid device ordinal");
  return device_initial_configuration(device, n, box_length, min_sep, seed, out_xyz, words, index, draws);
}

gcmc_status gcmc_random_initial_configuration(uint64_t n, double l, double min_sep, uint64_t seed,
                                              double* out_xyz, uint64_t words[312],
                                              uint64_t* index, uint64_t* draws) {
  // init_config.hpp:19-64, same draw sequence (3 per candidate incl. rejects).
  if (!(l > 0.0) || !(min_sep > 0.0)) return set_error(GCMC_ARG, "bad box or separation");
  std::mt19937_64 eng(seed);
  uint64_t ndraws = 0;
  auto uniform = [&]() {
    ++ndraws;
    return static_cast<double>(eng() >> 11) * 0x1.0p-53;
  };
  auto wrap = [l](double v) {
    double r = std::fmod(v, l);
    if (r < 0.0) r += l;
    if (r >= l) r = 0.0;
    return r;
  };
  int dims = static_cast<int>(l / min_sep);
  if (dims < 1) dims = 1;
  const double inv_width = dims / l;
  const uint64_t ncells = (uint64_t)dims * dims * dims;
  std::vector<int64_t> head(ncells, -1), next(n ? n : 1, -1);
  auto coord = [&](double v) {
    const int c = static_cast<int>(v * inv_width);
    return c < dims ? c : dims - 1;
  };
  const double min_sep2 = min_sep * min_sep;
  const double inv_l = 1.0 / l;
  uint64_t count = 0, rejects = 0;
  while (count < n) {
    const double x = wrap(uniform() * l), y = wrap(uniform() * l), z = wrap(uniform() * l);
    const int cx = coord(x), cy = coord(y), cz = coord(z);
    const int span = std::min(3, dims);
    bool clash = false;
    for (int a = 0; a < span && !clash; ++a)
      for (int b = 0; b < span && !clash; ++b)
        for (int q = 0; q < span && !clash; ++q) {
          int ix = (cx - 1) % dims, iy = (cy - 1) % dims, iz = (cz - 1) % dims;
          if (ix < 0) ix += dims;
          if (iy < 0) iy += dims;
          if (iz < 0) iz += dims;
          ix = (ix + q) % dims;
          iy = (iy + b) % dims;
          iz = (iz + a) % dims;
          for (int64_t j = head[ix + (uint64_t)dims * (iy + (uint64_t)dims * iz)]; j >= 0; j = next[j]) {
            double dx = x - out_xyz[3 * j], dy = y - out_xyz[3 * j + 1], dz = z - out_xyz[3 * j + 2];
            // box.hpp:45-55 (host build has no -march, hence no FMA contraction)
            dx -= l * std::nearbyint(dx * inv_l);
            dy -= l * std::nearbyint(dy * inv_l);
            dz -= l * std::nearbyint(dz * inv_l);
            const double r2 = dx * dx + dy * dy + dz * dz;
            if (r2 < min_sep2) {
              clash = true;
              break;
            }
          }
        }
    if (clash) {
      if (++rejects >= 1000000)
        return set_error(GCMC_ARG, "initial configuration: 1000000 consecutive rejections; "
                                   "density too high for the minimum separation");
      continue;
    }
    rejects = 0;
    out_xyz[3 * count] = x;
    out_xyz[3 * count + 1] = y;
    out_xyz[3 * count + 2] = z;
    const uint64_t cell = cx + (uint64_t)dims * (cy + (uint64_t)dims * cz);
    next[count] = head[cell];
    head[cell] = (int64_t)count;
    ++count;
  }
  std::ostringstream os;
  os << eng;
  std::istringstream is(os.str());
  uint64_t w[313];
  for (auto& v : w) is >> v;
  if (words) std::memcpy(words, w, 312 * 8);
  if (index) *index = w[312];
  if (draws) *draws = ndraws;
  return GCMC_OK;
}

}  // extern "C"
