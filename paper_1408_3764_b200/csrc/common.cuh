// Device primitives shared by every kernel of the GCMC engine.
//
// Bit-exactness contract: every expression that the reference evaluates
// with two roundings (a*b then +c) is written with explicit __dmul_rn /
// __dadd_rn / __dsub_rn so nvcc can never contract it into an FMA — the
// reference's x86-64 build has no FMA (no -march, proj/CMakeLists.txt:1-18).
// Pair terms and r^2 are therefore bit-identical to the reference; only the
// order of the final sums differs (tree reduction instead of one sequential
// Kahan chain), which keeps ΔE within ~1e-15 relative.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "gcmc_b200.h"

namespace gcmcb {

constexpr int kMaxCap = 128;  // largest slots-per-cell the device paths support

// ----------------------------------------------------------------- params
struct Box {
  double l, inv_l;          // side length, 1/L (box.hpp:47)
  double eps, sigma, sigma2, rc, rc2;
  double four_eps, tf_eps;  // 4*eps, 24*eps (potential.hpp:45)
  double pad, inv_sigma;    // 1e-9*sigma, 1/sigma (microcell_grid.hpp:87-88)
};

// Spatial index (reference layout + coordinate mirror).
struct Grid {
  int kind;                 // GCMC_ALL_PAIRS / GCMC_CELL_LIST / GCMC_MICROCELL
  int dims;                 // cells per axis
  int cap;                  // slots per cell
  int pad0;
  uint64_t ncells;
  double inv_cell;          // 1/S (cell list) or 1/sigma (microcell)
  double last_w;            // microcell boundary cell width (sigma units)
  int32_t* occ;             // [ncells]          occupancy_view()
  int32_t* slots;           // [cap*ncells]      slots_view(): micro k*nc+c, cell c*cap+k
};

// Evaluation mirror ("bricks"): cells of side L/dims >= r_cut, so the 3x3x3
// brick neighbourhood of a point holds every particle within r_cut (the
// reference's traditional cell-list geometry, cell_grid.hpp:27-33, with a
// 1e-9 relative margin). Records are SoA double planes indexed brick*cap+k,
// densely packed per brick (swap-last removal), so the resident footprint is
// ~N*28 bytes regardless of the strategy whose reference layout (Grid) is
// maintained for parity. Any window covering the cutoff sphere yields the
// same pair set, so the ΔE it produces is the reference's up to summation
// order.
struct Mirror {
  int dims;                 // bricks per axis
  int cap;                  // records per brick
  uint32_t nb;              // dims^3
  int reach;                // conflict reach in bricks (engine.cu)
  double inv;               // dims / L
  double side;              // L / dims
  double* rx;               // [nb*cap] record planes
  double* ry;
  double* rz;
  int32_t* rid;             // [nb*cap] particle id of each record
  int32_t* occ;             // [nb]
};

// Per-chain scalars on the device (one 256-byte block, L2 resident).
struct ChainState {
  uint64_t n;               // live particles
  uint64_t step;            // Simulation::step_ (engine.hpp:436)
  double energy, virial;    // SystemState (engine.hpp:112-117)
  uint64_t attempted[3], accepted[3];
  uint64_t samples;         // RunStatistics (engine.hpp:125-131)
  double sum_u, sum_p, sum_n, sum_n2;
  int32_t peak;             // peak_cell_occupancy()
  int32_t error;            // gcmc_status of the first failure
  int64_t err_a, err_b, err_c;  // failure detail (cell, occupancy, particle)
  uint64_t moves_done;      // moves completed by the last engine call
  uint64_t rounds;          // speculative rounds of the last engine call
  unsigned long long pair_evals;  // FP64 pair evaluations the engines performed (cumulative)
  uint64_t pad[10];
};
static_assert(sizeof(ChainState) == 256, "ChainState layout");

// Move proposal parsed from the MT stream (engine.hpp:207-213, 350-411).
// kind: 0 displace, 1 insert, 2 remove. For displacements with
// max_displacement > 0, (x, y, z) hold the raw uniforms u1..u3 (the target
// depends on the old position); otherwise the wrapped target point.
struct Proposal {
  double x, y, z;
  double pick;
  double acc;
  int32_t kind;
  // State-independent data of the new position, filled by k_annotate (gen.cu)
  // off the engine's critical path: the pruned 3x3x3 brick window as a 27-bit
  // mask (kNoMask: not precomputed), the packed brick point and the
  // reference-grid cell.
  uint32_t wmask;
  uint32_t bpt;
  int32_t cell;
};
static_assert(sizeof(Proposal) == 56, "Proposal layout");
constexpr uint32_t kNoMask = 0xffffffffu;

// ----------------------------------------------------------------- box.hpp
// box.hpp:24-31. fmod is exact in CUDA as in glibc.
__device__ __forceinline__ double wrap_axis(double v, double l) {
  double r = fmod(v, l);
  if (r < 0.0) r = __dadd_rn(r, l);
  if (r >= l) r = 0.0;
  return r;
}

// box.hpp:45-55 with the reference's exact rounding sequence.
__device__ __forceinline__ double min_image_dist2(double ax, double ay, double az, double bx,
                                                  double by, double bz, const Box& b) {
  double dx = __dsub_rn(ax, bx);
  double dy = __dsub_rn(ay, by);
  double dz = __dsub_rn(az, bz);
  dx = __dsub_rn(dx, __dmul_rn(b.l, rint(__dmul_rn(dx, b.inv_l))));
  dy = __dsub_rn(dy, __dmul_rn(b.l, rint(__dmul_rn(dy, b.inv_l))));
  dz = __dsub_rn(dz, __dmul_rn(b.l, rint(__dmul_rn(dz, b.inv_l))));
  return __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
}

// potential.hpp:39-54 for 0 < r2 <= rc2 (callers test the cutoff first).
__device__ __forceinline__ void lj_pair_clamped(double r2, const Box& b, double& u, double& w) {
  if (r2 < __dmul_rn(1e-12, b.sigma2)) {
    u = 1e30;
    w = 1e30;
    return;
  }
  const double s2 = __ddiv_rn(b.sigma2, r2);
  const double s6 = __dmul_rn(__dmul_rn(s2, s2), s2);
  const double s12 = __dmul_rn(s6, s6);
  u = __dmul_rn(b.four_eps, __dsub_rn(s12, s6));
  w = __dmul_rn(b.tf_eps, __dsub_rn(__dmul_rn(2.0, s12), s6));
}

// rng.hpp:38-41
__device__ __forceinline__ uint64_t index_from(double u, uint64_t n) {
  const uint64_t i = (uint64_t)__dmul_rn(u, (double)n);
  return i < n ? i : n - 1;
}

// engine.hpp:28-59 (operation order preserved).
__device__ __forceinline__ double metropolis(double r) { return r < 1.0 ? r : 1.0; }
__device__ __forceinline__ double displacement_acceptance(double du, double beta) {
  return metropolis(exp(__dmul_rn(-beta, du)));
}
__device__ __forceinline__ double insertion_acceptance(double du, uint64_t n, double vol,
                                                       double beta, double mu, double lambda3) {
  return metropolis(
      __dmul_rn(__ddiv_rn(vol, __dmul_rn(lambda3, (double)(n + 1))),
                exp(__dmul_rn(beta, __dsub_rn(mu, du)))));
}
__device__ __forceinline__ double deletion_acceptance(double du, uint64_t n, double vol,
                                                      double beta, double mu, double lambda3) {
  return metropolis(__dmul_rn(__ddiv_rn(__dmul_rn(lambda3, (double)n), vol),
                              exp(__dmul_rn(-beta, __dadd_rn(mu, du)))));
}

// ----------------------------------------------------------------- grids
__device__ __forceinline__ int coord(const Grid& g, double v) {
  const int c = (int)__dmul_rn(v, g.inv_cell);
  return c < g.dims ? c : g.dims - 1;
}
__device__ __forceinline__ int cell_of(const Grid& g, double x, double y, double z) {
  return coord(g, x) + g.dims * (coord(g, y) + g.dims * coord(g, z));
}
__device__ __forceinline__ uint64_t slot_index(const Grid& g, int cell, int k) {
  return g.kind == GCMC_MICROCELL ? (uint64_t)k * g.ncells + (uint64_t)cell
                                  : (uint64_t)cell * (uint64_t)g.cap + (uint64_t)k;
}

// microcell_grid.hpp:85-103: the cyclic run of cells intersecting
// [x - rc - pad, x + rc + pad].
//
// The reference computes the unwrapped cell as k*dims + cell(w) with
// w = wrap_axis(t) (fmod) and k = llround((t - w)/L). For stored
// coordinates x in [0, L) and rc + pad <= L/2 every t lies in (-L, 2L), where
// fmod is the identity or an exact subtraction and k is -1, 0 or 1; the
// branches below give the same w and k as the fmod/divide form, including
// the "t + L rounds to L -> w = 0, k = 0" corner.
__device__ __forceinline__ long long arc_global_cell(double t, double l, double inv_sigma,
                                                     int dims) {
  double w;
  long long k;
  if (t < 0.0) {
    w = __dadd_rn(t, l);
    if (w >= l) {
      w = 0.0;
      k = 0;
    } else {
      k = -1;
    }
  } else if (t >= l) {
    w = __dsub_rn(t, l);  // exact (Sterbenz), equals fmod(t, l)
    k = 1;
  } else {
    w = t;
    k = 0;
  }
  int c = (int)__dmul_rn(w, inv_sigma);
  if (c >= dims) c = dims - 1;
  return k * dims + c;
}
__device__ __forceinline__ void microcell_axis_arc(double x, const Box& b, int dims, int& first,
                                                   int& count) {
  const long long lo = arc_global_cell(__dsub_rn(__dsub_rn(x, b.rc), b.pad), b.l, b.inv_sigma, dims);
  const long long span =
      arc_global_cell(__dadd_rn(__dadd_rn(x, b.rc), b.pad), b.l, b.inv_sigma, dims) - lo + 1;
  // lo lies in [-dims, 2*dims): reduce without a 64-bit modulo
  int f = (int)lo;
  f += f < 0 ? dims : 0;
  f -= f >= dims ? dims : 0;
  first = f;
  count = span >= dims ? dims : (int)span;
}

// One axis of a search window: cells first, first+1, ... (mod dims).
struct AxisRun {
  int first, count;
};

// Window for a position (the set of cells the delta path scans).
//  microcell: product of the three axis arcs (microcell_grid.hpp:393-409);
//  cell list: the 27-cube around cell_of(p) (cell_grid.hpp:59-65, 208-221).
__device__ __forceinline__ void window_of(const Grid& g, const Box& b, double x, double y,
                                          double z, AxisRun& ax, AxisRun& ay, AxisRun& az) {
  if (g.kind == GCMC_MICROCELL) {
    microcell_axis_arc(x, b, g.dims, ax.first, ax.count);
    microcell_axis_arc(y, b, g.dims, ay.first, ay.count);
    microcell_axis_arc(z, b, g.dims, az.first, az.count);
  } else {
    const int d = g.dims;
    const int cnt = d < 3 ? d : 3;
    int fx = coord(g, x) - 1, fy = coord(g, y) - 1, fz = coord(g, z) - 1;
    fx = ((fx % d) + d) % d;
    fy = ((fy % d) + d) % d;
    fz = ((fz % d) + d) % d;
    ax = {fx, cnt};
    ay = {fy, cnt};
    az = {fz, cnt};
  }
}

__device__ __forceinline__ int window_cell(const Grid& g, const AxisRun& ax, const AxisRun& ay,
                                           const AxisRun& az, int idx) {
  const int ix = idx % ax.count;
  const int rest = idx / ax.count;
  const int iy = rest % ay.count;
  const int iz = rest / ay.count;
  int cx = ax.first + ix;
  if (cx >= g.dims) cx -= g.dims;
  int cy = ay.first + iy;
  if (cy >= g.dims) cy -= g.dims;
  int cz = az.first + iz;
  if (cz >= g.dims) cz -= g.dims;
  return cx + g.dims * (cy + g.dims * cz);
}

// Cache-global loads: the chain state is rewritten by other SMs between
// rounds, so never trust L1.
__device__ __forceinline__ int ld_cg(const int32_t* p) { return __ldcg(p); }
__device__ __forceinline__ double4 ld_cg(const double4* p) {
  const double2 a = __ldcg(reinterpret_cast<const double2*>(p));
  const double2 b = __ldcg(reinterpret_cast<const double2*>(p) + 1);
  return make_double4(a.x, a.y, b.x, b.y);
}
__device__ __forceinline__ void st_cg(double4* p, double4 v) {
  __stcg(reinterpret_cast<double2*>(p), make_double2(v.x, v.y));
  __stcg(reinterpret_cast<double2*>(p) + 1, make_double2(v.z, v.w));
}

// The mirror back-pointer of particle i (record index brick*cap+k, mirror.cuh)
// lives in the otherwise unused 4th word of its store record, so the mover's
// position and its record index arrive in one 32-byte sector.
__device__ __forceinline__ int32_t* bslot_of(double4* pos, uint64_t i) {
  return reinterpret_cast<int32_t*>(pos + i) + 6;
}
__device__ __forceinline__ const int32_t* bslot_of(const double4* pos, uint64_t i) {
  return reinterpret_cast<const int32_t*>(pos + i) + 6;
}
__device__ __forceinline__ int32_t bslot_in(const double4& r) {
  return (int32_t)(uint32_t)__double_as_longlong(r.w);
}
// Position only: keeps the back-pointer word.
__device__ __forceinline__ void st_xyz(double4* p, double x, double y, double z) {
  __stcg(reinterpret_cast<double2*>(p), make_double2(x, y));
  __stcg(reinterpret_cast<double*>(p) + 2, z);
}

__device__ __forceinline__ double pid_bits(uint64_t pid) {
  return __longlong_as_double((long long)pid);
}
__device__ __forceinline__ long long bits_pid(double w) { return __double_as_longlong(w); }

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Compensated accumulator (kahan.hpp:8-20) and a TwoSum warp tree; used by
// the full-system energy (energy.cu).
struct Kahan {
  double s, c;
  __device__ __forceinline__ void add(double v) {
    const double y = __dsub_rn(v, c);
    const double t = __dadd_rn(s, y);
    c = __dsub_rn(__dsub_rn(t, s), y);
    s = t;
  }
};

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


// Warp-cooperative ascending sort of a short list of distinct ids in place
// (the reference keeps each cell's ids ascending after build, grid_common.hpp
// :11-21): lanes hold up to 64 ids, each computes its rank by comparison and
// scatters; longer lists fall back to one lane's insertion sort. Returns the
// sorted id for slot `lane` and `lane + 32` via out0/out1 (unused if >= m).
__device__ __forceinline__ void warp_rank_sort(int32_t* a, int m, int lane) {
  if (m <= 1) return;
  if (m > 64) {
    if (lane == 0)
      for (int i = 1; i < m; ++i) {
        const int32_t v = a[i];
        int j = i - 1;
        while (j >= 0 && a[j] > v) {
          a[j + 1] = a[j];
          --j;
        }
        a[j + 1] = v;
      }
    __syncwarp();
    return;
  }
  const int32_t v0 = lane < m ? a[lane] : 0x7fffffff;
  const int32_t v1 = lane + 32 < m ? a[lane + 32] : 0x7fffffff;
  int r0 = 0, r1 = 0;
  if (m <= 32) {  // (the usual case: one value per lane, m rounds)
    for (int k = 0; k < m; ++k) r0 += __shfl_sync(0xffffffffu, v0, k) < v0;
  } else {
    for (int k = 0; k < 32; ++k) {
      const int32_t w0 = __shfl_sync(0xffffffffu, v0, k);
      const int32_t w1 = __shfl_sync(0xffffffffu, v1, k);
      r0 += (w0 < v0) + (w1 < v0);
      r1 += (w0 < v1) + (w1 < v1);
    }
  }
  __syncwarp();
  if (lane < m) a[r0] = v0;
  if (lane + 32 < m) a[r1] = v1;
  __syncwarp();
}

}  // namespace gcmcb
