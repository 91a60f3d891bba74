// Brick-mirror geometry shared by the trial-move kernels (slot.cuh), the
// engine's conflict tests (engine.cu) and the mirror maintenance (grid.cu,
// commit.cuh).
//
// A point is summarised by its packed brick coordinates
//   bx | by << 8 | bz << 16             (24 bits, kNoPoint = none; dims <= 255)
// so that speculative evaluations can be checked against the positions an
// accepted move changed: two points are "near" when their cyclic brick
// distance is <= reach on every axis (reach >= 1 covers the 3x3x3 window and
// the reference cell of either point; host sets it in api.cu).
#pragma once
#include "common.cuh"

namespace gcmcb {

constexpr uint64_t kNoPoint = 0xffffffull;

__device__ __forceinline__ int mcoord(const Mirror& m, double v) {
  const int c = (int)__dmul_rn(v, m.inv);
  return c < m.dims ? (c < 0 ? 0 : c) : m.dims - 1;
}
__device__ __forceinline__ uint64_t mpoint(const Mirror& m, double x, double y, double z) {
  return (uint64_t)mcoord(m, x) | ((uint64_t)mcoord(m, y) << 8) |
         ((uint64_t)mcoord(m, z) << 16);
}
__device__ __forceinline__ int pt_x(uint64_t p) { return (int)(p & 0xff); }
__device__ __forceinline__ int pt_y(uint64_t p) { return (int)((p >> 8) & 0xff); }
__device__ __forceinline__ int pt_z(uint64_t p) { return (int)((p >> 16) & 0xff); }
__device__ __forceinline__ uint32_t mbrick(const Mirror& m, uint64_t p) {
  return (uint32_t)pt_x(p) + (uint32_t)m.dims * ((uint32_t)pt_y(p) + (uint32_t)m.dims * (uint32_t)pt_z(p));
}

__device__ __forceinline__ bool axis_near(int a, int b, int d, int reach) {
  int t = a - b;
  t = t < 0 ? -t : t;
  t = t < d - t ? t : d - t;
  return t <= reach;
}
__device__ __forceinline__ bool mnear(const Mirror& m, uint64_t a, uint64_t b) {
  if (a == kNoPoint || b == kNoPoint) return false;
  return axis_near(pt_x(a), pt_x(b), m.dims, m.reach) &&
         axis_near(pt_y(a), pt_y(b), m.dims, m.reach) &&
         axis_near(pt_z(a), pt_z(b), m.dims, m.reach);
}

// Brick (ox, oy, oz) offsets of the 3x3x3 window that can hold a particle
// within r_cut of p: bricks whose box lies farther than r_cut from p are
// pruned (spherical window; ~20 of 27 bricks at side ~ r_cut). Returns the
// brick count and writes ids to out[0..26]. Lanes 0..26 of a warp call it
// cooperatively (one offset each); result compacted by ballot.
__device__ __forceinline__ int window_bricks_warp(const Mirror& m, const Box& b, double x,
                                                  double y, double z, uint32_t* out, int lane) {
  const int d = m.dims;
  const int cnt = d < 3 ? d : 3;
  const int bx = mcoord(m, x), by = mcoord(m, y), bz = mcoord(m, z);
  bool keep = false;
  uint32_t id = 0;
  if (lane < cnt * cnt * cnt) {
    const int ix = lane % cnt, iy = (lane / cnt) % cnt, iz = lane / (cnt * cnt);
    // offsets -1, 0, +1 (or 0..cnt-1 from -1 for tiny grids)
    const int ox = ix - 1, oy = iy - 1, oz = iz - 1;
    int cx = bx + ox, cy = by + oy, cz = bz + oz;
    cx += cx < 0 ? d : 0;
    cx -= cx >= d ? d : 0;
    cy += cy < 0 ? d : 0;
    cy -= cy >= d ? d : 0;
    cz += cz < 0 ? d : 0;
    cz -= cz >= d ? d : 0;
    id = (uint32_t)cx + (uint32_t)d * ((uint32_t)cy + (uint32_t)d * (uint32_t)cz);
    keep = true;
    if (d >= 3) {
      // distance from p to the brick's box along each axis
      auto ax = [&](double v, int bc, int o) {
        const double f = __dsub_rn(v, __dmul_rn((double)bc, m.side));  // offset in own brick
        double t = o == 0 ? 0.0 : (o > 0 ? __dsub_rn(m.side, f) : f);
        return t > 0.0 ? t : 0.0;
      };
      const double dx = ax(x, bx, ox), dy = ax(y, by, oy), dz = ax(z, bz, oz);
      const double d2 = dx * dx + dy * dy + dz * dz;
      keep = d2 <= b.rc2 * (1.0 + 1e-9) + 1e-12;
    }
  }
  const unsigned mask = __ballot_sync(0xffffffffu, keep);
  if (keep) out[__popc(mask & ((1u << lane) - 1u))] = id;
  return __popc(mask);
}

}  // namespace gcmcb
