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

// Tiny grids (dims < 3): every brick of the box is in the window.
static __device__ __noinline__ int window_bricks_small(const Mirror& m, uint32_t* out, int lane) {
  const int nb = m.dims * m.dims * m.dims;
  if (lane < nb) out[lane] = (uint32_t)lane;
  return nb;
}

// Window offset `lane` (0..26: ox = lane % 3 - 1, oy = lane / 3 % 3 - 1,
// oz = lane / 9 - 1) of a point in brick (bx, by, bz), dims >= 3: its brick
// id, and whether the brick's box lies within r_cut of the point (spherical
// pruning; ~20 of 27 bricks at side ~ r_cut).
__device__ __forceinline__ bool window_keep(const Mirror& m, const Box& b, double x, double y,
                                            double z, int bx, int by, int bz, int lane,
                                            uint32_t& id) {
  const int d = m.dims;
  const int ox = lane % 3 - 1, oy = (lane / 3) % 3 - 1, oz = lane / 9 - 1;
  int cx = bx + ox, cy = by + oy, cz = bz + oz;
  cx += cx < 0 ? d : 0;
  cx -= cx >= d ? d : 0;
  cy += cy < 0 ? d : 0;
  cy -= cy >= d ? d : 0;
  cz += cz < 0 ? d : 0;
  cz -= cz >= d ? d : 0;
  id = (uint32_t)cx + (uint32_t)d * ((uint32_t)cy + (uint32_t)d * (uint32_t)cz);
  // distance from p to the brick's box along each axis
  auto ax = [&](double v, int bc, int o) {
    const double f = __dsub_rn(v, __dmul_rn((double)bc, m.side));  // offset in own brick
    const double t = o == 0 ? 0.0 : (o > 0 ? __dsub_rn(m.side, f) : f);
    return t > 0.0 ? t : 0.0;
  };
  const double dx = ax(x, bx, ox), dy = ax(y, by, oy), dz = ax(z, bz, oz);
  const double d2 = dx * dx + dy * dy + dz * dz;
  return d2 <= b.rc2 * (1.0 + 1e-9) + 1e-12;
}

// The window of a point as brick ids in out[0..], lanes 0..26 of a warp
// cooperatively (one offset each), compacted by ballot in offset order.
__device__ __forceinline__ int window_bricks_warp(const Mirror& m, const Box& b, double x,
                                                  double y, double z, uint32_t* out, int lane) {
  if (m.dims < 3) return window_bricks_small(m, out, lane);
  const int bx = mcoord(m, x), by = mcoord(m, y), bz = mcoord(m, z);
  uint32_t id = 0;
  const bool keep = lane < 27 && window_keep(m, b, x, y, z, bx, by, bz, lane, id);
  const unsigned mask = __ballot_sync(0xffffffffu, keep);
  if (keep) out[__popc(mask & ((1u << lane) - 1u))] = id;
  return __popc(mask);
}

// The same window from a precomputed offset mask (Proposal::wmask) and
// packed brick point: integer work only.
__device__ __forceinline__ int window_bricks_mask(const Mirror& m, uint32_t wmask, uint32_t bpt,
                                                  uint32_t* out, int lane) {
  const bool keep = lane < 27 && ((wmask >> lane) & 1u);
  if (keep) {
    const int d = m.dims;
    int cx = pt_x(bpt) + lane % 3 - 1, cy = pt_y(bpt) + (lane / 3) % 3 - 1, cz = pt_z(bpt) + lane / 9 - 1;
    cx += cx < 0 ? d : 0;
    cx -= cx >= d ? d : 0;
    cy += cy < 0 ? d : 0;
    cy -= cy >= d ? d : 0;
    cz += cz < 0 ? d : 0;
    cz -= cz >= d ? d : 0;
    out[__popc(wmask & ((1u << lane) - 1u))] =
        (uint32_t)cx + (uint32_t)d * ((uint32_t)cy + (uint32_t)d * (uint32_t)cz);
  }
  return __popc(wmask);
}

}  // namespace gcmcb
