// Warp-cooperative trial-move energy sums over one or two search windows.
//
// This is the B200 form of the reference's sum_around / delta_* traversals
// (microcell_grid.hpp:200-241, 392-470; cell_grid.hpp:97-138, 208-235;
// strategy.hpp:64-116). One warp evaluates a whole move:
//
//   hop 1  lanes stride over the window cells (x-fastest, 216-512 cells for
//          a microcell arc, 27 for the cell list) and load occupancies;
//          a warp scan compacts the occupied slots into a per-warp list in
//          shared memory (slot index | endpoint tag);
//   hop 2  lanes stride over the list and load the coordinate-mirror records
//          (double4 x, y, z, pid) — one 32-byte sector each, no pid->pos
//          gather;
//   math   r^2 and the LJ pair with the reference's exact rounding, Kahan
//          per lane, then a compensated (TwoSum) warp tree.
//
// Any window that covers the cutoff sphere yields the same mathematical sum;
// these are the reference's own windows, so the visited neighbour sets are
// identical (tests/test_gpu_parity.py checks them).
#pragma once
#include "common.cuh"

namespace gcmcb {

struct Kahan {
  double s, c;
  __device__ __forceinline__ void add(double v) {
    const double y = __dsub_rn(v, c);
    const double t = __dadd_rn(s, y);
    c = __dsub_rn(__dsub_rn(t, s), y);
    s = t;
  }
};

// Compensated warp reduction of a Kahan accumulator (TwoSum per level).
__device__ __forceinline__ double warp_sum_comp(Kahan k) {
  double s = k.s, e = -k.c;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double s2 = __shfl_xor_sync(0xffffffffu, s, o);
    const double e2 = __shfl_xor_sync(0xffffffffu, e, o);
    const double t = __dadd_rn(s, s2);
    const double bp = __dsub_rn(t, s);
    const double err = __dadd_rn(__dsub_rn(s, __dsub_rn(t, bp)), __dsub_rn(s2, bp));
    s = t;
    e = __dadd_rn(__dadd_rn(e, e2), err);
  }
  return __dadd_rn(s, e);
}

struct Endpoints {
  int np;              // 1 or 2
  double x[2], y[2], z[2];
  long long exclude;   // pid skipped in every sum (n for an insertion)
};

struct Sums {
  double u[2], w[2];
};

// Per-lane accumulators for up to two endpoints (kept in registers: no
// dynamic indexing).
struct Acc {
  Kahan u0, w0, u1, w1;
};

__device__ __forceinline__ void accumulate(const Box& b, const Endpoints& ep, int e, double qx,
                                           double qy, double qz, Acc& acc) {
  const double px = e ? ep.x[1] : ep.x[0];
  const double py = e ? ep.y[1] : ep.y[0];
  const double pz = e ? ep.z[1] : ep.z[0];
  const double r2 = min_image_dist2(px, py, pz, qx, qy, qz, b);
  if (r2 <= b.rc2) {
    double u, w;
    lj_pair_clamped(r2, b, u, w);
    if (e) {
      acc.u1.add(u);
      acc.w1.add(w);
    } else {
      acc.u0.add(u);
      acc.w0.add(w);
    }
  }
}

__device__ __forceinline__ Sums finish(const Acc& acc, int np) {
  Sums s;
  s.u[0] = warp_sum_comp(acc.u0);
  s.w[0] = warp_sum_comp(acc.w0);
  s.u[1] = s.w[1] = 0.0;
  if (np > 1) {
    s.u[1] = warp_sum_comp(acc.u1);
    s.w[1] = warp_sum_comp(acc.w1);
  }
  return s;
}

// Records of the compacted list [0, count): slot index in bits 0..30,
// endpoint in bit 31.
template <int R>
__device__ __forceinline__ void drain_list(const Grid& g, const Box& b, const Endpoints& ep,
                                           const uint32_t* list, int count, Acc& acc) {
  const int lane = threadIdx.x & 31;
  for (int base = 0; base < count; base += 32 * R) {
    double4 r[R];
    uint32_t tag[R];
#pragma unroll
    for (int t = 0; t < R; ++t) {
      const int i = base + lane + 32 * t;
      tag[t] = i < count ? list[i] : 0xffffffffu;
      if (tag[t] != 0xffffffffu) r[t] = ld_cg(g.cellpos + (tag[t] & 0x7fffffffu));
    }
#pragma unroll
    for (int t = 0; t < R; ++t) {
      if (tag[t] == 0xffffffffu) continue;
      if (bits_pid(r[t].w) == ep.exclude) continue;
      accumulate(b, ep, (int)(tag[t] >> 31), r[t].x, r[t].y, r[t].z, acc);
    }
  }
}

// Grid strategies. `list` is per-warp shared scratch of `list_cap` entries
// (>= 32 * cap). Result sums are valid in every lane.
template <int CH>
__device__ Sums window_sums_grid(const Grid& g, const Box& b, const Endpoints& ep,
                                 uint32_t* list, int list_cap) {
  const int lane = threadIdx.x & 31;
  AxisRun ax0, ay0, az0, ax1 = {0, 1}, ay1 = {0, 1}, az1 = {0, 1};
  window_of(g, b, ep.x[0], ep.y[0], ep.z[0], ax0, ay0, az0);
  const int tot0 = ax0.count * ay0.count * az0.count;
  int tot1 = 0;
  if (ep.np > 1) {
    window_of(g, b, ep.x[1], ep.y[1], ep.z[1], ax1, ay1, az1);
    tot1 = ax1.count * ay1.count * az1.count;
  }
  const int total = tot0 + tot1;
  Acc acc = {};
  int count = 0;
  for (int base = 0; base < total; base += 32 * CH) {
    int cell[CH], occv[CH];
#pragma unroll
    for (int t = 0; t < CH; ++t) {
      const int idx = base + lane + 32 * t;
      cell[t] = -1;
      occv[t] = 0;
      if (idx < total) {
        const int e = idx >= tot0;
        cell[t] = e ? (window_cell(g, ax1, ay1, az1, idx - tot0) | (int)0x80000000)
                    : window_cell(g, ax0, ay0, az0, idx);
      }
    }
#pragma unroll
    for (int t = 0; t < CH; ++t)
      if (cell[t] != -1) occv[t] = ld_cg(g.occ + (cell[t] & 0x7fffffff));
    int mine = 0;
#pragma unroll
    for (int t = 0; t < CH; ++t) mine += occv[t];
    int incl = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    const int chunk = __shfl_sync(0xffffffffu, incl, 31);
    if (count + chunk > list_cap) {
      __syncwarp();
      drain_list<8>(g, b, ep, list, count, acc);
      __syncwarp();
      count = 0;
    }
    if (chunk > list_cap) {
      // Pathological density: visit this chunk's cells directly.
#pragma unroll
      for (int t = 0; t < CH; ++t) {
        if (occv[t] == 0) continue;
        const int c = cell[t] & 0x7fffffff;
        const int e = (unsigned)cell[t] >> 31;
        for (int k = 0; k < occv[t]; ++k) {
          const double4 r = ld_cg(g.cellpos + slot_index(g, c, k));
          if (bits_pid(r.w) == ep.exclude) continue;
          accumulate(b, ep, e, r.x, r.y, r.z, acc);
        }
      }
      continue;
    }
    int off = count + incl - mine;
#pragma unroll
    for (int t = 0; t < CH; ++t) {
      const int c = cell[t] & 0x7fffffff;
      const uint32_t etag = (uint32_t)cell[t] & 0x80000000u;
      for (int k = 0; k < occv[t]; ++k) list[off++] = (uint32_t)slot_index(g, c, k) | etag;
    }
    count += chunk;
  }
  __syncwarp();
  drain_list<8>(g, b, ep, list, count, acc);
  __syncwarp();
  return finish(acc, ep.np);
}

// all_pairs: every live particle, ascending j (strategy.hpp:64-116).
static __device__ __forceinline__ Sums window_sums_all_pairs(const Box& b, const double4* pos, uint64_t n,
                                      const Endpoints& ep) {
  const int lane = threadIdx.x & 31;
  Acc acc = {};
  constexpr int R = 4;
  for (uint64_t base = 0; base < n; base += 32 * R) {
    double4 r[R];
#pragma unroll
    for (int t = 0; t < R; ++t) {
      const uint64_t j = base + lane + 32 * t;
      if (j < n) r[t] = ld_cg(pos + j);
    }
#pragma unroll
    for (int t = 0; t < R; ++t) {
      const uint64_t j = base + lane + 32 * t;
      if (j >= n || (long long)j == ep.exclude) continue;
      accumulate(b, ep, 0, r[t].x, r[t].y, r[t].z, acc);
      if (ep.np > 1) accumulate(b, ep, 1, r[t].x, r[t].y, r[t].z, acc);
    }
  }
  return finish(acc, ep.np);
}

__device__ __forceinline__ Sums window_sums(const Grid& g, const Box& b, const double4* pos,
                                            uint64_t n, const Endpoints& ep, uint32_t* list,
                                            int list_cap) {
  if (g.kind == GCMC_ALL_PAIRS) return window_sums_all_pairs(b, pos, n, ep);
  return window_sums_grid<8>(g, b, ep, list, list_cap);
}

}  // namespace gcmcb
