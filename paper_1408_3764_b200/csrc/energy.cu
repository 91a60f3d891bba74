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

__global__ void k_esort(uint64_t ncells, const int* start, const int* count, int* ids,
                        const double4* __restrict__ pos, double4* rec) {
  const uint64_t c = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (c >= ncells) return;
  int* a = ids + start[c];
  const int m = count[c];
  for (int i = 1; i < m; ++i) {
    const int v = a[i];
    int j = i - 1;
    while (j >= 0 && a[j] > v) {
      a[j + 1] = a[j];
      --j;
    }
    a[j + 1] = v;
  }
  for (int i = 0; i < m; ++i) {
    const double4 p = pos[a[i]];
    rec[start[c] + i] = make_double4(p.x, p.y, p.z, pid_bits((uint64_t)a[i]));
  }
}

constexpr int kEWarps = 4;
constexpr int kOwnMax = 64;

__global__ void __launch_bounds__(kEWarps * 32)
    k_energy(EGrid eg, Box b, const int* __restrict__ start, const int* __restrict__ count,
             const double4* __restrict__ rec, double* part_u, double* part_w,
             unsigned long long* overlap) {
  __shared__ double4 own_s[kEWarps][kOwnMax];
  __shared__ int pre_s[kEWarps][28];
  __shared__ int cell_s[kEWarps][27];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t c = blockIdx.x * (uint64_t)kEWarps + warp;
  if (c >= eg.ncells) return;
  const int d = eg.dims;
  const int cx = (int)(c % d), cy = (int)((c / d) % d), cz = (int)(c / ((uint64_t)d * d));
  // 27-cube (distinct for d >= 3, compute_cell_dims guarantees it)
  int ncnt = 0;
  if (lane < 27) {
    const int ox = lane % 3 - 1, oy = (lane / 3) % 3 - 1, oz = lane / 9 - 1;
    const int nx = (cx + ox + d) % d, ny = (cy + oy + d) % d, nz = (cz + oz + d) % d;
    const int nc = nx + d * (ny + d * nz);
    cell_s[warp][lane] = nc;
    ncnt = count[nc];
  }
  int incl = ncnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane < 27) pre_s[warp][lane + 1] = incl;
  if (lane == 0) pre_s[warp][0] = 0;
  const int total = __shfl_sync(0xffffffffu, incl, 26);
  const int own_start = start[c], own_n = count[c];
  __syncwarp();
  Kahan ku = {0, 0}, kw = {0, 0};
  for (int ob = 0; ob < own_n; ob += kOwnMax) {
    const int on = min(kOwnMax, own_n - ob);
    for (int i = lane; i < on; i += 32) own_s[warp][i] = rec[own_start + ob + i];
    __syncwarp();
    for (int t = lane; t < total; t += 32) {
      int k = 0;
      while (pre_s[warp][k + 1] <= t) ++k;
      const int nc = cell_s[warp][k];
      const double4 q = rec[start[nc] + (t - pre_s[warp][k])];
      const long long jid = bits_pid(q.w);
      for (int i = 0; i < on; ++i) {
        const double4 p = own_s[warp][i];
        const long long iid = bits_pid(p.w);
        if (jid <= iid) continue;
        const double r2 = min_image_dist2(p.x, p.y, p.z, q.x, q.y, q.z, b);
        if (r2 > b.rc2) continue;
        if (r2 < __dmul_rn(1e-12, b.sigma2)) {
          atomicMin(overlap, ((unsigned long long)iid << 32) | (unsigned long long)jid);
          continue;
        }
        double u, w;
        lj_pair_clamped(r2, b, u, w);
        ku.add(u);
        kw.add(w);
      }
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
__global__ void k_ereduce(uint64_t ncells, const double* pu, const double* pw, double* out) {
  __shared__ double su[32], sw[32], cu[32], cw[32];
  Kahan ku = {0, 0}, kw = {0, 0};
  for (uint64_t i = threadIdx.x; i < ncells; i += blockDim.x) {
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
      out[0] = tu;
      out[1] = tw;
    }
    (void)cu;
    (void)cw;
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
  const size_t need = al(n * 4) * 2 + al(nc * 4) * 3 + al(n * 32) + al(nc * 8) * 2 + al(64) +
                      al(scan_bytes);
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
  double* pu = (double*)take(nc * 8);
  double* pw = (double*)take(nc * 8);
  char* small = take(64);
  void* scan_tmp = take(scan_bytes);
  unsigned long long* overlap = (unsigned long long*)small;
  double* out = (double*)(small + 16);
  cudaStream_t s = c.stream;
  cudaMemsetAsync(count, 0, nc * 4, s);
  cudaMemsetAsync(fill, 0, nc * 4, s);
  cudaMemsetAsync(overlap, 0xff, 8, s);
  k_ecount<<<blocks(n, 256), 256, 0, s>>>(eg, c.pos, n, cid, count);
  cub::DeviceScan::ExclusiveSum(scan_tmp, scan_bytes, count, start, (int)nc, s);
  k_escatter<<<blocks(n, 256), 256, 0, s>>>(n, cid, start, fill, ids);
  k_esort<<<blocks(nc, 128), 128, 0, s>>>(nc, start, count, ids, c.pos, rec);
  k_energy<<<blocks(nc, kEWarps), kEWarps * 32, 0, s>>>(eg, c.box, start, count, rec, pu, pw,
                                                         overlap);
  k_ereduce<<<1, 1024, 0, s>>>(nc, pu, pw, out);
  double h[2];
  unsigned long long ov = 0;
  cudaMemcpyAsync(h, out, 16, cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(&ov, overlap, 8, cudaMemcpyDeviceToHost, s);
  if ((e = cudaStreamSynchronize(s))) return cuda_error(e, "total_energy");
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
