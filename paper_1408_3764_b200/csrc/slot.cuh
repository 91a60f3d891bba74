// Group-cooperative trial-move energy over the brick mirror: one group of T
// threads evaluates one or two windows of one proposal — the paper's "one
// block of threads per move" retargeted at sm_100a, and
// the B200 form of the reference's sum_around / delta_* traversals
// (cell_grid.hpp:97-138, 208-235; microcell_grid.hpp:200-241, 458-470;
// strategy.hpp:64-116).
//
//   setup   warp 0: the pruned 3x3x3 brick window of each endpoint
//           (mirror.cuh), occupancies (shared-memory replica or global),
//           warp scan, then expansion of (brick, slot) pairs into a per-group
//           candidate list in shared memory;          one group barrier
//   gather  every thread loads the x/y/z record planes of its candidates
//           (one dependent L2 hop for the whole window);
//   math    FP64 minimum-image r^2 with the reference's exact rounding
//           (common.cuh) and the LJ pair for those within r_cut (latency
//           form: two candidates per thread, no compaction);
//   reduce  warp tree + fixed-order cross-warp sum (deterministic).
//
// The mover's own record is excluded by record index (the reference skips
// it by id), so records carry no id in the hot planes.
#pragma once
#include "mirror.cuh"

namespace gcmcb {

constexpr int kMaxEnt = 54;     // 2 windows x 27 bricks
constexpr int kCandMax = 1536;  // expanded candidates per group per pass

template <int T>
struct WinWs {
  double cx[2], cy[2], cz[2];  // window centres (0: + sign, 1: - sign)
  int nwin;                    // windows in use (1 or 2); window 1 has sign -1 when sign1 < 0
  int sign1;                   // +1 / -1 sign of window 1
  int nent0, nent;             // bricks of window 0, of both windows
  int total;                   // candidates
  int excl;                    // excluded record index (-1: none)
  uint32_t brick[kMaxEnt];
  int pre[kMaxEnt + 1];
  uint16_t cand[kCandMax];     // entry << 7 | slot
  double red[T / 32][2];
};

// Named barrier over a group of warps. The non-.aligned form: the warps of a
// group reach it from lane-divergent code (one lane polling a flag, lanes
// leaving a loop at different trip counts), where the .aligned bar.sync is
// undefined behaviour (in practice it counts a warp as arrived when its first
// lanes do, releasing the barrier early). The __syncwarp reconverges first.
__device__ __forceinline__ void group_sync(int id, int nthreads) {
  __syncwarp();
  asm volatile("barrier.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// Warp 0 of the group, step 1 (per window): the pruned brick window of a
// centre appended to ws.brick[nent..]; returns the new entry count.
template <int T>
__device__ __forceinline__ int win_add(const Mirror& m, const Box& b, WinWs<T>& ws, int nent,
                                       double x, double y, double z, int lane) {
  return nent + window_bricks_warp(m, b, x, y, z, ws.brick + nent, lane);
}

// Warp 0 of the group, step 2: occupancies (shared-memory replica or global),
// exclusive prefix over nent <= 54 entries, candidate expansion.
template <int T>
__device__ __forceinline__ void win_finish(const Mirror& m, WinWs<T>& ws, const uint8_t* occ_s,
                                           int nent, int nent0, int lane) {
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
  // one scan of both halves packed in 16 bits each (counts <= 27 * cap < 2^16)
  int s = o0 | (o1 << 16);
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, s, o);
    if (lane >= o) s += t;
  }
  const int last = __shfl_sync(0xffffffffu, s, 31);
  const int tot0 = last & 0xffff;
  const int e0 = (s & 0xffff) - o0, e1 = tot0 + (s >> 16) - o1;  // exclusive
  if (lane < nent) ws.pre[lane] = e0;
  if (lane + 32 < nent) ws.pre[lane + 32] = e1;
  const int total = tot0 + (last >> 16);
  if (lane == 0) {
    ws.nent0 = nent0;
    ws.nent = nent;
    ws.pre[nent] = total;
    ws.total = total;
  }
  // expansion (first kCandMax candidates; the rest are found by search)
#pragma unroll 1
  for (int k = 0; k < o0; ++k)
    if (e0 + k < kCandMax) ws.cand[e0 + k] = (uint16_t)((lane << 7) | k);
#pragma unroll 1
  for (int k = 0; k < o1; ++k)
    if (e1 + k < kCandMax) ws.cand[e1 + k] = (uint16_t)(((lane + 32) << 7) | k);
}

// Both steps for the windows already described in ws (cx/cy/cz, nwin).
template <int T>
__device__ __forceinline__ void win_setup_warp(const Mirror& m, const Box& b, WinWs<T>& ws,
                                               const uint8_t* occ_s, int lane) {
  int nent = 0, nent0 = 0;
  for (int w = 0; w < ws.nwin; ++w) {
    nent = win_add<T>(m, b, ws, nent, ws.cx[w], ws.cy[w], ws.cz[w], lane);
    if (w == 0) nent0 = nent;
  }
  win_finish<T>(m, ws, occ_s, nent, nent0, lane);
}

__device__ __forceinline__ void lj_accum(const Box& b, double r2, double sign, double& du,
                                         double& dw) {
  double u, w;
  lj_pair_clamped(r2, b, u, w);
  du = __dadd_rn(du, __dmul_rn(sign, u));
  dw = __dadd_rn(dw, __dmul_rn(sign, w));
}

// All T threads (after the group barrier that publishes ws): Σ_w sign_w Σ
// pair(centre_w, record) over the candidates, excluding record ws.excl.
// Returns per-thread partial sums (reduce with group_reduce). Latency form:
// a thread takes candidates gt and gt + T (both gathers in flight at once),
// then runs the pair math on each; no compaction (one window is < 2T).
template <int T>
__device__ __forceinline__ void win_sums(const Mirror& m, const Box& b, WinWs<T>& ws, int gt,
                                         double& du, double& dw) {
  const int total = ws.total;
  du = 0.0;
  dw = 0.0;
#pragma unroll 1
  for (int base = 0; base < total; base += 2 * T) {
    double rx[2], ry[2], rz[2];
    int win[2];
    bool ok[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int f = base + u * T + gt;
      ok[u] = f < total;
      win[u] = 0;
      rx[u] = ry[u] = rz[u] = 0.0;
      if (ok[u]) {
        int e, k;
        if (f < kCandMax) {
          const int c = ws.cand[f];
          e = c >> 7;
          k = c & 127;
        } else {  // rare: binary search of the prefix
          int lo = 0, hi = ws.nent - 1;
          while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (ws.pre[mid] <= f) lo = mid; else hi = mid - 1;
          }
          e = lo;
          k = f - ws.pre[lo];
        }
        win[u] = e >= ws.nent0;
        const int idx = (int)ws.brick[e] * m.cap + k;
        if (idx == ws.excl) {
          ok[u] = false;
        } else {
          rx[u] = __ldcg(m.rx + idx);
          ry[u] = __ldcg(m.ry + idx);
          rz[u] = __ldcg(m.rz + idx);
        }
      }
    }
#pragma unroll 1
    for (int u = 0; u < 2; ++u) {
      const bool o = u ? ok[1] : ok[0];
      if (o) {
        const int w = u ? win[1] : win[0];
        const double r2 = min_image_dist2(ws.cx[w], ws.cy[w], ws.cz[w], u ? rx[1] : rx[0],
                                          u ? ry[1] : ry[0], u ? rz[1] : rz[0], b);
        if (r2 <= b.rc2) lj_accum(b, r2, w ? (double)ws.sign1 : 1.0, du, dw);
      }
    }
  }
}

// Group-wide deterministic reduction; result valid in thread gt == leader_gt
// after the call (all T threads call).
template <int T>
__device__ __forceinline__ void group_reduce(WinWs<T>& ws, double& du, double& dw, int bar_id,
                                             int gt, int leader_gt = 0) {
  const int lane = threadIdx.x & 31, w = gt >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    du = __dadd_rn(du, __shfl_xor_sync(0xffffffffu, du, o));
    dw = __dadd_rn(dw, __shfl_xor_sync(0xffffffffu, dw, o));
  }
  if constexpr (T > 32) {
    if (lane == 0) {
      ws.red[w][0] = du;
      ws.red[w][1] = dw;
    }
    group_sync(bar_id, T);
    if (gt == leader_gt) {
      double a = 0.0, c = 0.0;
#pragma unroll
      for (int i = 0; i < T / 32; ++i) {
        a = __dadd_rn(a, ws.red[i][0]);
        c = __dadd_rn(c, ws.red[i][1]);
      }
      du = a;
      dw = c;
    }
  }
}

// All-pairs strategy (strategy.hpp:64-116): the window is the whole store.
template <int T>
__device__ __forceinline__ void allpairs_sums(const Box& b, const double4* pos, uint64_t n,
                                              WinWs<T>& ws, long long exclude, int gt, double& du,
                                              double& dw) {
  du = 0.0;
  dw = 0.0;
  for (uint64_t j = gt; j < n; j += T) {
    if ((long long)j == exclude) continue;
    const double4 r = ld_cg(pos + j);
    for (int w = 0; w < ws.nwin; ++w) {
      const double r2 = min_image_dist2(ws.cx[w], ws.cy[w], ws.cz[w], r.x, r.y, r.z, b);
      if (r2 <= b.rc2) lj_accum(b, r2, w ? (double)ws.sign1 : 1.0, du, dw);
    }
  }
}

}  // namespace gcmcb
