// Full-system energy and virial: total_energy() (engine.hpp:74-94) for
// initialisation and audits.
//
// The reference sums N(N-1)/2 pairs in one O(N^2) loop (~1.7 h at 1 M on a
// host core). Here: a counting sort of the particles into a coarse cell grid
// (cells >= r_cut, compute_cell_dims, cell_grid.hpp:27-33) giving a
// cell-ordered double4 coordinate array (x, y, z, id), then one warp per
// cell scans its 27-cell neighbourhood; a pair (i, j) is evaluated once,
// from the cell of i, when id_j > id_i. Within a cell the ids are sorted, so
// the result is deterministic. FP64 pair math is bit-identical to the
// reference; sums are Kahan per lane + compensated trees (not the
// reference's single ascending chain: agreement ~1e-14 relative).
#include <cub/device/device_scan.cuh>

#include <cmath>
#include <cstdlib>
#include <sstream>

#include "internal.h"
#include "common.cuh"

namespace gcmcb {

namespace {

struct EGrid {
  int dims;
  double inv;
  uint64_t ncells;
};

__device__ __forceinline__ int ecoord(const EGrid& e, double v) {
  const int c = (int)__dmul_rn(v, e.inv);
  return c < e.dims ? c : e.dims - 1;
}

__global__ void k_ecount(EGrid eg, const double4* __restrict__ pos, uint64_t n, int* cid,
                         int* count) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double4 p = pos[i];
  const int c = ecoord(eg, p.x) + eg.dims * (ecoord(eg, p.y) + eg.dims * ecoord(eg, p.z));
  cid[i] = c;
  atomicAdd(count + c, 1);
}

__global__ void k_escatter(uint64_t n, const int* cid, const int* start, int* fill, int* ids) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int c = cid[i];
  ids[start[c] + atomicAdd(fill + c, 1)] = (int)i;
}

// One warp per cell: ids ascending (deterministic pair order), then the
// double and float records.
__global__ void k_esort(uint64_t ncells, const int* start, const int* count, int* ids,
                        const double4* __restrict__ pos, double4* rec, float4* recf) {
  const uint64_t c = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (c >= ncells) return;
  int* a = ids + start[c];
  const int m = count[c];
  warp_rank_sort(a, m, lane);
  for (int i = lane; i < m; i += 32) {
    const double4 p = pos[a[i]];
    rec[start[c] + i] = make_double4(p.x, p.y, p.z, pid_bits((uint64_t)a[i]));
    recf[start[c] + i] = make_float4((float)p.x, (float)p.y, (float)p.z, 0.0f);
  }
}

constexpr int kEWarps = 4;
constexpr int kOwnMax = 64;
constexpr int kECand = 512;

struct Prefilter {
  float l, inv_l, cut2;  // float box, 1/L and the conservative r^2 bound
  int on;
};

// One warp per cell c: pairs (i in c, j in the half shell of c) — c itself
// (i < j by id) and its 13 forward neighbours — so every pair is visited
// once. An FP32 minimum image with a conservative bound rejects the ~85% of
// candidates beyond r_cut; survivors get the reference's exact FP64
// minimum image and LJ pair (common.cuh), Kahan per lane and a compensated
// warp tree. Overlap (r^2 < 1e-12 sigma^2) is reported like total_energy's
// runtime_error (engine.hpp:74-94).
template <bool kShift>
__global__ void __launch_bounds__(kEWarps * 32)
    k_energy(EGrid eg, Box b, Prefilter pf, const int* __restrict__ start,
             const int* __restrict__ count, const double4* __restrict__ rec,
             const float4* __restrict__ recf, double* part_u, double* part_w,
             unsigned long long* overlap) {
  __shared__ double4 own_s[kEWarps][kOwnMax];
  __shared__ float4 ownf_s[kEWarps][kOwnMax];
  __shared__ int cand_s[kEWarps][kECand];
  __shared__ int queue_s[kEWarps][64];  // (record << 6 | own index) of pairs that passed the prefilter
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t c = blockIdx.x * (uint64_t)kEWarps + warp;
  if (c >= eg.ncells) return;
  const int d = eg.dims;
  const int cx = (int)(c % d), cy = (int)((c / d) % d), cz = (int)(c / ((uint64_t)d * d));
  // half shell: offsets 0..13 of the 27-cube in x-fastest order starting at
  // (0,0,0): {self} + the 13 cells after it in lexicographic (z, y, x) order
  // kShift: each neighbour's periodic image shift (-L, 0, +L per axis, the
  // image adjacent to this cell) rides in the low 6 bits of its candidate
  // entries, so the FP32 prefilter needs no minimum-image rounding (valid
  // for cells >= r_cut: a pair within r_cut has no other close image)
  int ncnt = 0, nstart = 0, scode = 21;  // 21: no shift on any axis
  if (lane < 14) {
    const int t = 13 + lane;  // cube index: (ox, oy, oz) = (t % 3, t / 3 % 3, t / 9) - 1
    const int ox = t % 3 - 1, oy = (t / 3) % 3 - 1, oz = t / 9 - 1;
    const int rx = cx + ox, ry = cy + oy, rz = cz + oz;
    const int nx = (rx + d) % d, ny = (ry + d) % d, nz = (rz + d) % d;
    const int nc = nx + d * (ny + d * nz);
    scode = (rx < 0 ? 0 : (rx >= d ? 2 : 1)) | (ry < 0 ? 0 : (ry >= d ? 2 : 1)) << 2 |
            (rz < 0 ? 0 : (rz >= d ? 2 : 1)) << 4;
    ncnt = count[nc];
    nstart = start[nc];
  }
  int incl = ncnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  const int total = __shfl_sync(0xffffffffu, incl, 13);
  const int own_start = __shfl_sync(0xffffffffu, nstart, 0);
  const int own_n = __shfl_sync(0xffffffffu, ncnt, 0);
  Kahan ku = {0, 0}, kw = {0, 0};
  for (int ob = 0; ob < own_n; ob += kOwnMax) {
    const int on = min(kOwnMax, own_n - ob);
    for (int i = lane; i < on; i += 32) {
      own_s[warp][i] = rec[own_start + ob + i];
      ownf_s[warp][i] = recf[own_start + ob + i];
    }
    for (int cb = 0; cb < total; cb += kECand) {
      // expansion of the candidate list (record indices), chunked
      __syncwarp();
      {
        const int e0 = incl - ncnt;
        for (int k = 0; k < ncnt; ++k) {
          const int f = e0 + k - cb;
          if (f >= 0 && f < kECand) cand_s[warp][f] = kShift ? ((nstart + k) << 6) | scode : nstart + k;
        }
      }
      __syncwarp();
      const int ctot = min(kECand, total - cb);
      // prefilter every (own i, candidate t) pair; pairs that may lie inside
      // r_cut are queued and evaluated exactly 32 at a time (full warps)
      int qn = 0;
      auto drain = [&](int m) {
        if (lane < m) {
          const int pk = queue_s[warp][lane];
          const double4 p = own_s[warp][pk & 63];
          const double4 q = rec[(unsigned)pk >> 6];
          const double r2 = min_image_dist2(p.x, p.y, p.z, q.x, q.y, q.z, b);
          if (r2 <= b.rc2) {
            if (r2 < __dmul_rn(1e-12, b.sigma2)) {
              long long iid = bits_pid(p.w), jid = bits_pid(q.w);
              if (iid > jid) {
                const long long t2 = iid;
                iid = jid;
                jid = t2;
              }
              atomicMin(overlap, ((unsigned long long)iid << 32) | (unsigned long long)jid);
            } else {
              double u, w;
              lj_pair_clamped(r2, b, u, w);
              ku.add(u);
              kw.add(w);
            }
          }
        }
      };
      for (int t0 = 0; t0 < ctot; t0 += 32) {
        const int t = t0 + lane;
        const bool have = t < ctot;
        const int ce = have ? cand_s[warp][t] : 0;
        const int qi = kShift ? ce >> 6 : ce;
        float4 qf = have ? recf[qi] : make_float4(0, 0, 0, 0);
        if (kShift) {
          qf.x += (float)((ce & 3) - 1) * pf.l;
          qf.y += (float)(((ce >> 2) & 3) - 1) * pf.l;
          qf.z += (float)(((ce >> 4) & 3) - 1) * pf.l;
        }
        // own i < lim passes the i < j rule (self cell) / all own i (others)
        const int lim = !have ? 0 : (cb + t < own_n ? cb + t - ob : on);
        const float cut2 = pf.on ? pf.cut2 : __int_as_float(0x7f800000);
        for (int i = 0; i < on; ++i) {
          bool pass;
          if (kShift) {
            const float4 pff = ownf_s[warp][i];
            const float dx = pff.x - qf.x, dy = pff.y - qf.y, dz = pff.z - qf.z;
            pass = i < lim && __fmaf_rn(dz, dz, __fmaf_rn(dy, dy, __fmul_rn(dx, dx))) <= cut2;
          } else {
            pass = i < lim;
            if (pass && pf.on) {
              const float4 pff = ownf_s[warp][i];
              float dx = pff.x - qf.x, dy = pff.y - qf.y, dz = pff.z - qf.z;
              dx -= pf.l * rintf(dx * pf.inv_l);
              dy -= pf.l * rintf(dy * pf.inv_l);
              dz -= pf.l * rintf(dz * pf.inv_l);
              pass = dx * dx + dy * dy + dz * dz <= pf.cut2;
            }
          }
          const unsigned m = __ballot_sync(0xffffffffu, pass);
          if (m) {
            const int pos = qn + __popc(m & ((1u << lane) - 1u));
            if (pass) queue_s[warp][pos] = (qi << 6) | i;
            qn += __popc(m);
            __syncwarp();
            if (qn >= 32) {
              drain(32);
              qn -= 32;
              const int carry = queue_s[warp][32 + lane];
              __syncwarp();
              if (lane < qn) queue_s[warp][lane] = carry;
              __syncwarp();
            }
          }
        }
      }
      __syncwarp();
      drain(qn);
    }
    __syncwarp();
  }
  const double su = warp_sum_comp(ku), sw = warp_sum_comp(kw);
  if (lane == 0) {
    part_u[c] = su;
    part_w[c] = sw;
  }
}

// The image-shift pass with the FP32 prefilter on paired lanes of Blackwell's
// packed FP32 pipe (FADD2 / FMUL2 / FFMA2): each lane tests two candidates
// against an own particle per instruction stream, 64 candidates per chunk and
// one vote pair per own particle. Same pair set and the same rounding of the
// prefilter r^2 as k_energy<true>; survivors are queued and evaluated exactly
// 32 at a time in (own, chunk half, lane) order.
__global__ void __launch_bounds__(kEWarps * 32)
    k_energy_pk(EGrid eg, Box b, Prefilter pf, const int* __restrict__ start,
                const int* __restrict__ count, const double4* __restrict__ rec,
                const float4* __restrict__ recf, double* part_u, double* part_w,
                unsigned long long* overlap) {
  __shared__ double4 own_s[kEWarps][kOwnMax];
  __shared__ float4 ownf_s[kEWarps][kOwnMax];
  __shared__ int cand_s[kEWarps][kECand];
  __shared__ int queue_s[kEWarps][128];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t c = blockIdx.x * (uint64_t)kEWarps + warp;
  if (c >= eg.ncells) return;
  const int d = eg.dims;
  const int cx = (int)(c % d), cy = (int)((c / d) % d), cz = (int)(c / ((uint64_t)d * d));
  int ncnt = 0, nstart = 0, scode = 21;
  if (lane < 14) {
    const int t = 13 + lane;
    const int ox = t % 3 - 1, oy = (t / 3) % 3 - 1, oz = t / 9 - 1;
    const int rx = cx + ox, ry = cy + oy, rz = cz + oz;
    const int nx = (rx + d) % d, ny = (ry + d) % d, nz = (rz + d) % d;
    const int nc = nx + d * (ny + d * nz);
    scode = (rx < 0 ? 0 : (rx >= d ? 2 : 1)) | (ry < 0 ? 0 : (ry >= d ? 2 : 1)) << 2 |
            (rz < 0 ? 0 : (rz >= d ? 2 : 1)) << 4;
    ncnt = count[nc];
    nstart = start[nc];
  }
  int incl = ncnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  const int total = __shfl_sync(0xffffffffu, incl, 13);
  const int own_start = __shfl_sync(0xffffffffu, nstart, 0);
  const int own_n = __shfl_sync(0xffffffffu, ncnt, 0);
  Kahan ku = {0, 0}, kw = {0, 0};
  auto exact = [&](int pk) {
    const double4 p = own_s[warp][pk & 63];
    const double4 q = rec[(unsigned)pk >> 6];
    const double r2 = min_image_dist2(p.x, p.y, p.z, q.x, q.y, q.z, b);
    if (r2 <= b.rc2) {
      if (r2 < __dmul_rn(1e-12, b.sigma2)) {
        long long iid = bits_pid(p.w), jid = bits_pid(q.w);
        if (iid > jid) {
          const long long t2 = iid;
          iid = jid;
          jid = t2;
        }
        atomicMin(overlap, ((unsigned long long)iid << 32) | (unsigned long long)jid);
      } else {
        double u, w;
        lj_pair_clamped(r2, b, u, w);
        ku.add(u);
        kw.add(w);
      }
    }
  };
  const float cut2 = pf.on ? pf.cut2 : __int_as_float(0x7f800000);
  for (int ob = 0; ob < own_n; ob += kOwnMax) {
    const int on = min(kOwnMax, own_n - ob);
    for (int i = lane; i < on; i += 32) {
      own_s[warp][i] = rec[own_start + ob + i];
      ownf_s[warp][i] = recf[own_start + ob + i];
    }
    for (int cb = 0; cb < total; cb += kECand) {
      __syncwarp();
      {
        const int e0 = incl - ncnt;
        for (int k = 0; k < ncnt; ++k) {
          const int f = e0 + k - cb;
          if (f >= 0 && f < kECand) cand_s[warp][f] = ((nstart + k) << 6) | scode;
        }
      }
      __syncwarp();
      const int ctot = min(kECand, total - cb);
      int qn = 0;
      for (int t0 = 0; t0 < ctot; t0 += 64) {
        int qi[2], lim[2];
        float2 nqx, nqy, nqz;
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const int t = t0 + 32 * hh + lane;
          const bool have = t < ctot;
          const int ce = have ? cand_s[warp][t] : 0;
          qi[hh] = ce >> 6;
          float4 qf = have ? recf[qi[hh]] : make_float4(0, 0, 0, 0);
          qf.x += (float)((ce & 3) - 1) * pf.l;
          qf.y += (float)(((ce >> 2) & 3) - 1) * pf.l;
          qf.z += (float)(((ce >> 4) & 3) - 1) * pf.l;
          if (hh == 0) {
            nqx.x = -qf.x;
            nqy.x = -qf.y;
            nqz.x = -qf.z;
          } else {
            nqx.y = -qf.x;
            nqy.y = -qf.y;
            nqz.y = -qf.z;
          }
          lim[hh] = !have ? 0 : (cb + t < own_n ? cb + t - ob : on);
        }
        for (int i = 0; i < on; ++i) {
          const float4 pff = ownf_s[warp][i];
          const float2 dx = __fadd2_rn(make_float2(pff.x, pff.x), nqx);
          const float2 dy = __fadd2_rn(make_float2(pff.y, pff.y), nqy);
          const float2 dz = __fadd2_rn(make_float2(pff.z, pff.z), nqz);
          const float2 r2 = __ffma2_rn(dz, dz, __ffma2_rn(dy, dy, __fmul2_rn(dx, dx)));
          const bool pa = i < lim[0] && r2.x <= cut2, pb = i < lim[1] && r2.y <= cut2;
          const unsigned ma = __ballot_sync(0xffffffffu, pa), mb = __ballot_sync(0xffffffffu, pb);
          if (ma | mb) {
            const unsigned below = (1u << lane) - 1u;
            if (pa) queue_s[warp][qn + __popc(ma & below)] = (qi[0] << 6) | i;
            if (pb) queue_s[warp][qn + __popc(ma) + __popc(mb & below)] = (qi[1] << 6) | i;
            qn += __popc(ma) + __popc(mb);
            __syncwarp();
            while (qn >= 32) {
              exact(queue_s[warp][lane]);
              qn -= 32;
              const int c0 = queue_s[warp][32 + lane], c1 = queue_s[warp][64 + lane];
              __syncwarp();
              if (lane < qn) queue_s[warp][lane] = c0;
              if (32 + lane < qn) queue_s[warp][32 + lane] = c1;
              __syncwarp();
            }
          }
        }
      }
      __syncwarp();
      if (lane < qn) exact(queue_s[warp][lane]);
      __syncwarp();
    }
    __syncwarp();
  }
  const double su = warp_sum_comp(ku), sw = warp_sum_comp(kw);
  if (lane == 0) {
    part_u[c] = su;
    part_w[c] = sw;
  }
}

// Deterministic final reduction over the per-cell partials.
// Deterministic reduction of n partials (u, w): block b sums its contiguous
// chunk (Kahan per thread + compensated trees) into ou[b], ow[b]. Used twice:
// 1024-value chunks over the per-cell partials, then one block over those.
constexpr int kRedChunk = 4096;

__global__ void __launch_bounds__(1024) k_ereduce(uint64_t n, const double* pu, const double* pw,
                                                  double* ou, double* ow) {
  __shared__ double su[32], sw[32];
  Kahan ku = {0, 0}, kw = {0, 0};
  const uint64_t lo = (uint64_t)blockIdx.x * kRedChunk;
  const uint64_t hi = lo + kRedChunk < n ? lo + kRedChunk : n;
  for (uint64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    ku.add(pu[i]);
    kw.add(pw[i]);
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double a = warp_sum_comp(ku), bsum = warp_sum_comp(kw);
  if (lane == 0) {
    su[warp] = a;
    sw[warp] = bsum;
  }
  __syncthreads();
  if (warp == 0) {
    Kahan k1 = {lane < (int)(blockDim.x / 32) ? su[lane] : 0.0, 0.0};
    Kahan k2 = {lane < (int)(blockDim.x / 32) ? sw[lane] : 0.0, 0.0};
    const double tu = warp_sum_comp(k1), tw = warp_sum_comp(k2);
    if (lane == 0) {
      ou[blockIdx.x] = tu;
      ow[blockIdx.x] = tw;
    }
  }
}

// Deterministic compensated sum of one block's per-thread accumulators.
__device__ __forceinline__ void block_sum_comp(Kahan ku, Kahan kw, double* su, double* sw,
                                               double& ou, double& ow) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double a = warp_sum_comp(ku), c = warp_sum_comp(kw);
  if (lane == 0) {
    su[warp] = a;
    sw[warp] = c;
  }
  __syncthreads();
  ou = ow = 0.0;
  if (warp == 0) {
    const int nw = blockDim.x >> 5;
    Kahan k1 = {lane < nw ? su[lane] : 0.0, 0.0}, k2 = {lane < nw ? sw[lane] : 0.0, 0.0};
    ou = warp_sum_comp(k1);
    ow = warp_sum_comp(k2);
  }
}

// O(N^2) cross-check (gcmc_total_energy_bruteforce): every pair i < j with
// the FP32 minimum image as a prefilter and the reference's FP64 minimum
// image + LJ pair for the survivors; no cell structure at all. Test / audit
// infrastructure for the cell-based pass above (a 1M check takes ~1 s).
constexpr int kBfThreads = 256;
constexpr int kBfTile = 1024;

__global__ void __launch_bounds__(kBfThreads)
    k_energy_bf(Box b, Prefilter pf, uint64_t n, const double4* __restrict__ pos, double* part,
                unsigned* done, double* out, unsigned long long* overlap) {
  __shared__ float4 tile[kBfTile];
  __shared__ double su[kBfThreads / 32], sw[kBfThreads / 32];
  __shared__ bool last;
  const uint64_t i = blockIdx.x * (uint64_t)kBfThreads + threadIdx.x;
  const uint64_t j0 = blockIdx.x * (uint64_t)kBfThreads;  // first j any thread of the block needs
  Kahan ku = {0, 0}, kw = {0, 0};
  double4 p = i < n ? pos[i] : make_double4(0, 0, 0, 0);
  const float px = (float)p.x, py = (float)p.y, pz = (float)p.z;
  for (uint64_t tb = j0; tb < n; tb += kBfTile) {
    __syncthreads();
    for (int k = threadIdx.x; k < kBfTile; k += kBfThreads) {
      const uint64_t j = tb + k;
      const double4 q = j < n ? pos[j] : make_double4(0, 0, 0, 0);
      tile[k] = make_float4((float)q.x, (float)q.y, (float)q.z, 0.0f);
    }
    __syncthreads();
    if (i >= n) continue;
    const int kmax = n - tb < (uint64_t)kBfTile ? (int)(n - tb) : kBfTile;
    for (int k = 0; k < kmax; ++k) {
      const uint64_t j = tb + k;
      const float4 q = tile[k];
      float dx = px - q.x, dy = py - q.y, dz = pz - q.z;
      dx -= pf.l * rintf(dx * pf.inv_l);
      dy -= pf.l * rintf(dy * pf.inv_l);
      dz -= pf.l * rintf(dz * pf.inv_l);
      if (j > i && (!pf.on || dx * dx + dy * dy + dz * dz <= pf.cut2)) {
        const double4 qd = pos[j];
        const double r2 = min_image_dist2(p.x, p.y, p.z, qd.x, qd.y, qd.z, b);
        if (r2 <= b.rc2) {
          if (r2 < __dmul_rn(1e-12, b.sigma2)) {
            atomicMin(overlap, ((unsigned long long)i << 32) | (unsigned long long)j);
          } else {
            double u, w;
            lj_pair_clamped(r2, b, u, w);
            ku.add(u);
            kw.add(w);
          }
        }
      }
    }
  }
  double bu, bw;
  block_sum_comp(ku, kw, su, sw, bu, bw);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = bu;
    part[2 * blockIdx.x + 1] = bw;
    __threadfence();
    last = atomicAdd(done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  Kahan k1 = {0, 0}, k2 = {0, 0};
  for (unsigned q = threadIdx.x; q < gridDim.x; q += kBfThreads) {
    k1.add(__ldcg(part + 2 * q));
    k2.add(__ldcg(part + 2 * q + 1));
  }
  __syncthreads();
  block_sum_comp(k1, k2, su, sw, bu, bw);
  if (threadIdx.x == 0) {
    out[0] = bu;
    out[1] = bw;
  }
}


inline unsigned blocks(uint64_t n, int t) { return (unsigned)((n + t - 1) / t); }

}  // namespace

gcmc_status total_energy(Chain& c, double* u, double* w) {
  const uint64_t n = c.st_host->n;
  *u = 0.0;
  *w = 0.0;
  if (n < 2) return GCMC_OK;
  // coarse grid: compute_cell_dims (cell_grid.hpp:27-33)
  const double l = c.box.l, rc = c.box.rc;
  int t = (int)(l / rc);
  while ((double)(t + 1) * rc <= l) ++t;
  while (t > 1 && (double)t * rc > l) --t;
  if (t < 3) t = 3;
  EGrid eg{t, 1.0 / (l / t), (uint64_t)t * t * t};
  const uint64_t nc = eg.ncells;
  // scratch layout
  size_t scan_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, (int*)nullptr, (int*)nullptr, (int)nc);
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  const size_t need = al(n * 4) * 2 + al(nc * 4) * 3 + al(n * 32) + al(n * 16) + al(nc * 8) * 2 +
                      al(64 + 16 * ((nc + kRedChunk - 1) / kRedChunk)) + al(scan_bytes);
  cudaError_t e;
  if (need > c.egrid_bytes) {
    if (c.egrid) cudaFree(c.egrid);
    c.egrid = nullptr;
    if ((e = cudaMalloc(&c.egrid, need))) return cuda_error(e, "total_energy alloc");
    c.egrid_bytes = need;
  }
  char* p = static_cast<char*>(c.egrid);
  auto take = [&](size_t bytes) {
    char* r = p;
    p += al(bytes);
    return r;
  };
  int* cid = (int*)take(n * 4);
  int* ids = (int*)take(n * 4);
  int* count = (int*)take(nc * 4);
  int* start = (int*)take(nc * 4);
  int* fill = (int*)take(nc * 4);
  double4* rec = (double4*)take(n * 32);
  float4* recf = (float4*)take(n * 16);
  double* pu = (double*)take(nc * 8);
  double* pw = (double*)take(nc * 8);
  const size_t nred = (nc + kRedChunk - 1) / kRedChunk;
  char* small = take(64 + 16 * nred);  // overlap word, result, first-level partials
  void* scan_tmp = take(scan_bytes);
  unsigned long long* overlap = (unsigned long long*)small;
  double* out = (double*)(small + 16);
  cudaStream_t s = c.stream;
  cudaEventRecord(c.ev_e[0], s);
  cudaMemsetAsync(count, 0, nc * 4, s);
  cudaMemsetAsync(fill, 0, nc * 4, s);
  cudaMemsetAsync(overlap, 0xff, 8, s);
  k_ecount<<<blocks(n, 256), 256, 0, s>>>(eg, c.pos, n, cid, count);
  cub::DeviceScan::ExclusiveSum(scan_tmp, scan_bytes, count, start, (int)nc, s);
  k_escatter<<<blocks(n, 256), 256, 0, s>>>(n, cid, start, fill, ids);
  k_esort<<<blocks(nc * 32, 256), 256, 0, s>>>(nc, start, count, ids, c.pos, rec, recf);
  // FP32 prefilter: the bound adds 2 sqrt(3) r_cut delta + 3 delta^2 (plus
  // float rounding of the sum) to r_cut^2. Off when the minimum-image choice
  // itself could differ between FP32 and FP64 (L close to 2 r_cut).
  Prefilter pf;
  {
    // per-axis error of the FP32 minimum image: inputs, difference, and the
    // L * rint product each contribute at most L 2^-24 -> delta = 3 * (3 L 2^-24)
    const double delta = 9.0 * l * std::ldexp(1.0, -24);
    const double cut2 = c.box.rc2 + 2.0 * rc * std::sqrt(3.0) * delta + 3.0 * delta * delta;
    pf.l = (float)l;
    pf.inv_l = (float)(1.0 / l);
    pf.cut2 = (float)(cut2 * (1.0 + 1e-5) + 1e-6);
    pf.on = l > 2.0 * rc + 0.5 ? 1 : 0;
  }
  cudaEventRecord(c.ev_e[1], s);
  // the image-shift prefilter needs cells >= r_cut (t >= 3 forced otherwise)
  static const bool rint_form = knob("GCMC_ENERGY_RINT") != nullptr;  // A/B
  static const bool scalar_form = knob("GCMC_ENERGY_SCALAR") != nullptr;  // A/B
  if (l / t >= rc && !rint_form && !scalar_form)
    k_energy_pk<<<blocks(nc, kEWarps), kEWarps * 32, 0, s>>>(eg, c.box, pf, start, count, rec, recf,
                                                            pu, pw, overlap);
  else if (l / t >= rc && !rint_form)
    k_energy<true><<<blocks(nc, kEWarps), kEWarps * 32, 0, s>>>(eg, c.box, pf, start, count, rec, recf,
                                                               pu, pw, overlap);
  else
    k_energy<false><<<blocks(nc, kEWarps), kEWarps * 32, 0, s>>>(eg, c.box, pf, start, count, rec,
                                                                recf, pu, pw, overlap);
  cudaEventRecord(c.ev_e[2], s);
  {  // two deterministic levels: chunks of the per-cell partials, then the chunks
    const unsigned nb = (unsigned)((nc + kRedChunk - 1) / kRedChunk);
    double* r2 = out + 2;  // [2 * nb] after the result (small scratch)
    k_ereduce<<<nb, 1024, 0, s>>>(nc, pu, pw, r2, r2 + nb);
    k_ereduce<<<1, 1024, 0, s>>>(nb, r2, r2 + nb, out, out + 1);
  }
  cudaEventRecord(c.ev_e[3], s);
  double h[2];
  unsigned long long ov = 0;
  cudaMemcpyAsync(h, out, 16, cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(&ov, overlap, 8, cudaMemcpyDeviceToHost, s);
  if ((e = cudaStreamSynchronize(s))) return cuda_error(e, "total_energy");
  cudaEventElapsedTime(&c.energy_ms[0], c.ev_e[0], c.ev_e[3]);
  cudaEventElapsedTime(&c.energy_ms[1], c.ev_e[1], c.ev_e[2]);
  if (ov != ~0ull) {
    std::ostringstream os;
    os << "total_energy: particles " << (ov >> 32) << " and " << (ov & 0xffffffffu) << " overlap";
    return set_error(GCMC_OVERLAP, os.str());
  }
  *u = h[0];
  *w = h[1];
  return GCMC_OK;
}

gcmc_status total_energy_bruteforce(Chain& c, double* u, double* w) {
  const uint64_t n = c.st_host->n;
  *u = 0.0;
  *w = 0.0;
  if (n < 2) return GCMC_OK;
  const unsigned nblk = blocks(n, kBfThreads);
  char* buf = nullptr;
  cudaError_t e = cudaMalloc(&buf, (size_t)nblk * 16 + 64);
  if (e) return cuda_error(e, "total_energy_bruteforce alloc");
  unsigned long long* overlap = (unsigned long long*)(buf + (size_t)nblk * 16);
  double* out = (double*)(buf + (size_t)nblk * 16 + 16);
  unsigned* done = (unsigned*)(buf + (size_t)nblk * 16 + 32);
  cudaStream_t s = c.stream;
  cudaMemsetAsync(overlap, 0xff, 8, s);
  cudaMemsetAsync(done, 0, 4, s);
  const double l = c.box.l, rc = c.box.rc;
  Prefilter pf;
  const double delta = 9.0 * l * std::ldexp(1.0, -24);
  const double cut2 = c.box.rc2 + 2.0 * rc * std::sqrt(3.0) * delta + 3.0 * delta * delta;
  pf.l = (float)l;
  pf.inv_l = (float)(1.0 / l);
  pf.cut2 = (float)(cut2 * (1.0 + 1e-5) + 1e-6);
  pf.on = l > 2.0 * rc + 0.5 ? 1 : 0;
  k_energy_bf<<<nblk, kBfThreads, 0, s>>>(c.box, pf, n, c.pos, (double*)buf, done, out, overlap);
  double h[2];
  unsigned long long ov = 0;
  cudaMemcpyAsync(h, out, 16, cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(&ov, overlap, 8, cudaMemcpyDeviceToHost, s);
  e = cudaStreamSynchronize(s);
  if (!e) e = cudaGetLastError();
  cudaFree(buf);
  if (e) return cuda_error(e, "total_energy_bruteforce");
  if (ov != ~0ull) {
    std::ostringstream os;
    os << "total_energy: particles " << (ov >> 32) << " and " << (ov & 0xffffffffu) << " overlap";
    return set_error(GCMC_OVERLAP, os.str());
  }
  *u = h[0];
  *w = h[1];
  return GCMC_OK;
}

}  // namespace gcmcb
