// Group-cooperative trial-move energy: a group of T threads (T = 512/M for
// M moves per CTA) evaluates one move — the paper's "one block of threads per
// move, one thread per microcell" re-targeted at sm_100a:
// several moves share an SM, each on its own named barrier.
//
// setup      lanes 0..5 of the group's first warp compute the six axis runs
//            of the move's windows (microcell arcs, microcell_grid.hpp:85-103;
//            cell-list 3-cubes, cell_grid.hpp:59-65) once and publish them in
//            shared memory with the endpoints;
// microcell  thread t <-> cube cells t, t+T, ... of an 8x8x8 cube over each
//            window: occupancies first, then the coordinate-mirror records
//            of the occupied cells — two overlapped L2 hops per move;
// cell list  thread t <-> (window, cell, slot lane) of the 27-cell windows;
// all pairs  threads stride over the store (strategy.hpp:64-116).
//
// Pair terms are bit-identical to the reference (common.cuh). Each thread
// accumulates the signed move delta (+new window, -old window), then a warp
// tree and a cross-warp tree. The reference's Kahan chains are
// summation-order variants of the same sum: agreement ~1e-15 relative
// (tests bound it at 1e-10).
#pragma once
#include "window.cuh"

namespace gcmcb {

// Per-move scalars shared by the group.
struct MoveCtx {
  double x[2], y[2], z[2];  // endpoints (0: new / only, 1: old)
  long long exclude;
  int np;
  int run[2][3][2];         // [endpoint][axis][first, count]
  int rows0, rows;          // x-rows of window 0, total rows
};

template <int T>
struct GroupReduce {
  double v[T / 32][2];
  double out[2];
};

__device__ __forceinline__ void group_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// Lanes 0..5 of the calling warp fill ctx.run (and row counts). Caller syncs.
__device__ __forceinline__ void setup_runs(const Grid& g, const Box& b, MoveCtx& ctx) {
  const int lane = threadIdx.x & 31;
  if (lane < 6) {
    const int e = lane / 3, axis = lane % 3;
    int first = 0, count = 0;
    if (e < ctx.np) {
      const double v = axis == 0 ? ctx.x[e] : (axis == 1 ? ctx.y[e] : ctx.z[e]);
      if (g.kind == GCMC_MICROCELL) {
        microcell_axis_arc(v, b, g.dims, first, count);
      } else {
        const int d = g.dims;
        int f = coord(g, v) - 1;
        f += f < 0 ? d : 0;
        first = f;
        count = d < 3 ? d : 3;
      }
    }
    ctx.run[e][axis][0] = first;
    ctx.run[e][axis][1] = count;
  }
  __syncwarp();
  if (lane == 0) {
    ctx.rows0 = ctx.run[0][1][1] * ctx.run[0][2][1];
    ctx.rows = ctx.rows0 + ctx.run[1][1][1] * ctx.run[1][2][1];
  }
}

__device__ __forceinline__ void pair_term(const Box& b, double px, double py, double pz,
                                          const double4& r, long long exclude, double sign,
                                          double& du, double& dw) {
  if (bits_pid(r.w) == exclude) return;
  const double r2 = min_image_dist2(px, py, pz, r.x, r.y, r.z, b);
  if (r2 <= b.rc2) {
    double u, w;
    lj_pair_clamped(r2, b, u, w);
    du = __dadd_rn(du, __dmul_rn(sign, u));
    dw = __dadd_rn(dw, __dmul_rn(sign, w));
  }
}

// Group-wide reduction of (du, dw); all T threads call; result returned in
// every thread (after the trailing group barrier).
template <int T>
__device__ __forceinline__ void group_reduce2(double& du, double& dw, GroupReduce<T>& red,
                                              int bar_id) {
  const int gt = threadIdx.x % T, w = gt >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    du = __dadd_rn(du, __shfl_xor_sync(0xffffffffu, du, o));
    dw = __dadd_rn(dw, __shfl_xor_sync(0xffffffffu, dw, o));
  }
  if constexpr (T > 32) {
    if (lane == 0) {
      red.v[w][0] = du;
      red.v[w][1] = dw;
    }
    group_sync(bar_id, T);
    double a = 0.0, c = 0.0;
#pragma unroll
    for (int i = 0; i < T / 32; ++i) {
      a = __dadd_rn(a, red.v[i][0]);
      c = __dadd_rn(c, red.v[i][1]);
    }
    du = a;
    dw = c;
  }
}

__device__ __forceinline__ int run_cell(int first, int i, int d) {
  const int v = first + i;
  return v >= d ? v - d : v;
}

// Microcell: an 8x8x8 cube laid over each window (tiled when an axis has more
// than 8 cells); thread t owns cube cells t, t+T, ... of both windows. All
// occupancy loads are issued first, then the slot-0/slot-1 records of the
// occupied cells, so a thread's cells cost two overlapped L2 hops.
template <int T>
__device__ __forceinline__ void sums_microcell(const Grid& g, const Box& b, const MoveCtx& ctx,
                                               int gt, double& du, double& dw) {
  constexpr int P = 512 / T;  // cube cells per thread per window
  const int d = g.dims;
  const int mx = max(ctx.run[0][0][1], ctx.run[1][0][1]);
  const int my = max(ctx.run[0][1][1], ctx.run[1][1][1]);
  const int mz = max(ctx.run[0][2][1], ctx.run[1][2][1]);
  for (int oz = 0; oz < mz; oz += 8)
    for (int oy = 0; oy < my; oy += 8)
      for (int ox = 0; ox < mx; ox += 8) {
        int cell[2 * P], o[2 * P];
#pragma unroll
        for (int q = 0; q < 2 * P; ++q) {
          const int e = q / P;
          const int ci = gt + (q % P) * T;
          const int ix = ox + (ci & 7), iy = oy + ((ci >> 3) & 7), iz = oz + (ci >> 6);
          cell[q] = -1;
          if (ix < ctx.run[e][0][1] && iy < ctx.run[e][1][1] && iz < ctx.run[e][2][1])
            cell[q] = run_cell(ctx.run[e][0][0], ix, d) +
                      d * (run_cell(ctx.run[e][1][0], iy, d) + d * run_cell(ctx.run[e][2][0], iz, d));
          o[q] = cell[q] >= 0 ? ld_cg(g.occ + cell[q]) : 0;
        }
        double4 r0[2 * P], r1[2 * P];
#pragma unroll
        for (int q = 0; q < 2 * P; ++q) {
          if (o[q] > 0) r0[q] = ld_cg(g.cellpos + cell[q]);  // slot 0 of cell c sits at index c
          if (o[q] > 1) r1[q] = ld_cg(g.cellpos + g.ncells + cell[q]);
        }
#pragma unroll
        for (int q = 0; q < 2 * P; ++q) {
          const int e = q / P;
          const double sign = e ? -1.0 : 1.0;
          if (o[q] > 0) pair_term(b, ctx.x[e], ctx.y[e], ctx.z[e], r0[q], ctx.exclude, sign, du, dw);
          if (o[q] > 1) pair_term(b, ctx.x[e], ctx.y[e], ctx.z[e], r1[q], ctx.exclude, sign, du, dw);
          for (int k = 2; k < o[q]; ++k)
            pair_term(b, ctx.x[e], ctx.y[e], ctx.z[e],
                      ld_cg(g.cellpos + (uint64_t)k * g.ncells + cell[q]), ctx.exclude, sign, du,
                      dw);
        }
      }
}

// Cell list: 27 cells per window; threads = (window, cell, slot lane).
template <int T>
__device__ __forceinline__ void sums_cell_list(const Grid& g, const Box& b, const MoveCtx& ctx,
                                               int gt, double& du, double& dw) {
  constexpr int kCellsPad = 32;
  const int per_window = ctx.np > 1 ? T / 2 : T;
  const int lanes = per_window / kCellsPad > 0 ? per_window / kCellsPad : 1;
  const int e = ctx.np > 1 ? gt / per_window : 0;
  const int local = gt - e * per_window;
  const int k0 = local % lanes;
  const int d = g.dims;
  const double sign = e ? -1.0 : 1.0;
  for (int ci = local / lanes; ci < 27; ci += per_window / lanes) {
    const int c = run_cell(ctx.run[e][0][0], ci % 3, d) +
                  d * (run_cell(ctx.run[e][1][0], (ci / 3) % 3, d) +
                       d * run_cell(ctx.run[e][2][0], ci / 9, d));
    const int o = ld_cg(g.occ + c);
    const double4* base = g.cellpos + (uint64_t)c * g.cap;
    for (int k = k0; k < o; k += lanes)
      pair_term(b, ctx.x[e], ctx.y[e], ctx.z[e], ld_cg(base + k), ctx.exclude, sign, du, dw);
  }
}

template <int T>
__device__ __forceinline__ void sums_all_pairs(const Box& b, const double4* pos, uint64_t n,
                                               const MoveCtx& ctx, int gt, double& du,
                                               double& dw) {
  for (uint64_t j = gt; j < n; j += T) {
    if ((long long)j == ctx.exclude) continue;
    const double4 r = ld_cg(pos + j);
    const double4 q = make_double4(r.x, r.y, r.z, pid_bits(j));
    pair_term(b, ctx.x[0], ctx.y[0], ctx.z[0], q, -1, 1.0, du, dw);
    if (ctx.np > 1) pair_term(b, ctx.x[1], ctx.y[1], ctx.z[1], q, -1, -1.0, du, dw);
  }
}

// All T threads of the group call with ctx published (group-synced).
// Returns Σ_new - Σ_old (or Σ for one endpoint) in every thread.
template <int T>
__device__ __forceinline__ void group_delta(const Grid& g, const Box& b, const double4* pos,
                                            uint64_t n, const MoveCtx& ctx, GroupReduce<T>& red,
                                            int bar_id, double& du, double& dw) {
  const int gt = threadIdx.x % T;
  du = 0.0;
  dw = 0.0;
  if (g.kind == GCMC_MICROCELL)
    sums_microcell<T>(g, b, ctx, gt, du, dw);
  else if (g.kind == GCMC_CELL_LIST)
    sums_cell_list<T>(g, b, ctx, gt, du, dw);
  else
    sums_all_pairs<T>(b, pos, n, ctx, gt, du, dw);
  group_reduce2<T>(du, dw, red, bar_id);
}

}  // namespace gcmcb
