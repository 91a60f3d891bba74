// Cell-list / microcell build, consistency check and single-move commits.
//
// Build = the reference's build() (microcell_grid.hpp:194-198,
// cell_grid.hpp:233-237): particles are binned in ascending id order, so
// each cell's slots hold ascending ids. On the device: one thread per
// particle bins with an atomic slot counter (order within a cell is then
// arbitrary), then one thread per cell sorts its <= cap ids ascending and
// writes the coordinate mirror — byte-identical occ/slots to the reference.
#include <cub/device/device_scan.cuh>

#include <sstream>

#include "commit.cuh"
#include "internal.h"

namespace gcmcb {

namespace {

__global__ void k_bin(Grid g, const double4* __restrict__ pos, uint64_t n, int* overflow) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double4 p = pos[i];
  const int c = cell_of(g, p.x, p.y, p.z);
  const int k = atomicAdd(g.occ + c, 1);
  if (k < g.cap)
    g.slots[slot_index(g, c, k)] = (int32_t)i;
  else
    atomicExch(overflow, 1);
}

// Per cell: ascending insertion sort of the ids (grid_common.hpp:11-21
// ordering), mirror records, peak occupancy.
__global__ void k_sort_cells(Grid g, int32_t* rslot, ChainState* st) {
  const uint64_t c = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  int occ = 0;
  if (c < g.ncells) {
    occ = g.occ[c];
    if (occ > g.cap) occ = g.cap;
    int32_t ids[kMaxCap];
    for (int k = 0; k < occ; ++k) ids[k] = g.slots[slot_index(g, (int)c, k)];
    for (int i = 1; i < occ; ++i) {
      const int32_t v = ids[i];
      int j = i - 1;
      while (j >= 0 && ids[j] > v) {
        ids[j + 1] = ids[j];
        --j;
      }
      ids[j + 1] = v;
    }
    for (int k = 0; k < occ; ++k) {
      g.slots[slot_index(g, (int)c, k)] = ids[k];
      rslot[ids[k]] = k;
    }
  }
  // block max -> peak
  for (int o = 16; o > 0; o >>= 1) occ = max(occ, __shfl_xor_sync(0xffffffffu, occ, o));
  if ((threadIdx.x & 31) == 0 && occ > 0) atomicMax(&st->peak, occ);
}


// Mirror build: bin by brick (atomic slot), then per brick sort the ids
// ascending (deterministic record order) and write the record planes and
// the back-pointers.
__global__ void k_mbin(Mirror m, const double4* __restrict__ pos, uint64_t n,
                       int* overflow) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double4 p = pos[i];
  const uint32_t b = mbrick(m, mpoint(m, p.x, p.y, p.z));
  const int k = atomicAdd(m.occ + b, 1);
  if (k < m.cap)
    m.rid[(size_t)b * m.cap + k] = (int32_t)i;
  else
    atomicMax(overflow, (int)b + 1);
}

__global__ void k_msort(Mirror m, double4* pos) {
  const uint32_t b = (uint32_t)((blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (b >= m.nb) return;
  int occ = m.occ[b];
  if (occ > m.cap) occ = m.cap;
  int32_t* ids = m.rid + (size_t)b * m.cap;
  warp_rank_sort(ids, occ, lane);
  for (int k = lane; k < occ; k += 32) {
    const size_t s = (size_t)b * m.cap + k;
    const double4 p = pos[ids[k]];
    m.rx[s] = p.x;
    m.ry[s] = p.y;
    m.rz[s] = p.z;
    *bslot_of(pos, ids[k]) = (int32_t)s;
  }
}

// Overflow diagnosis (error path only): for every overflowing cell, the
// (cap+1)-th smallest member id is the insertion at which the reference's
// build throws; the smallest such id names the cell in the message.
__global__ void k_overflow_members(Grid g, const double4* __restrict__ pos, uint64_t n,
                                   const int* off, int* fill, int32_t* members) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double4 p = pos[i];
  const int c = cell_of(g, p.x, p.y, p.z);
  if (g.occ[c] <= g.cap) return;
  members[off[c] + atomicAdd(fill + c, 1)] = (int32_t)i;
}

__global__ void k_overflow_pick(Grid g, const int* off, int32_t* members,
                                unsigned long long* best) {
  const uint64_t c = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (c >= g.ncells) return;
  const int occ = g.occ[c];
  if (occ <= g.cap) return;
  int32_t* m = members + off[c];
  // partial selection: the (cap+1)-th smallest
  for (int i = 0; i <= g.cap; ++i) {
    int mi = i;
    for (int j = i + 1; j < occ; ++j)
      if (m[j] < m[mi]) mi = j;
    const int32_t t = m[i];
    m[i] = m[mi];
    m[mi] = t;
  }
  atomicMin(best, ((unsigned long long)(uint32_t)m[g.cap] << 32) | (uint32_t)c);
}

__global__ void k_overflow_sizes(Grid g, int* sizes) {
  const uint64_t c = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (c >= g.ncells) return;
  const int occ = g.occ[c];
  sizes[c] = occ > g.cap ? occ : 0;
}

// rebuild_check (microcell_grid.hpp:270-292, cell_grid.hpp:168-191):
// fresh counts, then per cell: occupancy equal, every slot id lives in that
// cell, no duplicates, and the coordinate mirror matches the store.
__global__ void k_fresh_count(Grid g, const double4* __restrict__ pos, uint64_t n, int* fresh) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double4 p = pos[i];
  atomicAdd(fresh + cell_of(g, p.x, p.y, p.z), 1);
}

// code: 1 overflow, 2 occupancy mismatch, 3 set mismatch, 4 mirror stale.
__global__ void k_check_cells(Grid g, const double4* __restrict__ pos, uint64_t n,
                              const int* fresh, unsigned long long* first) {
  const uint64_t c = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (c >= g.ncells) return;
  const int f = fresh[c];
  const int occ = g.occ[c];
  int code = 0;
  if (f > g.cap)
    code = 1;
  else if (f != occ)
    code = 2;
  else {
    for (int k = 0; k < occ && !code; ++k) {
      const uint64_t s = slot_index(g, (int)c, k);
      const int32_t id = g.slots[s];
      if (id < 0 || (uint64_t)id >= n) {
        code = 3;
        break;
      }
      const double4 p = pos[id];
      if (cell_of(g, p.x, p.y, p.z) != (int)c) code = 3;
      for (int j = 0; j < k; ++j)
        if (g.slots[slot_index(g, (int)c, j)] == id) code = 3;
    }
  }
  if (code) atomicMin(first, ((unsigned long long)c << 8) | (unsigned long long)code);
}

// Mirror + back-pointers against the store (engine-internal consistency;
// reported by rebuild_check as a stale coordinate mirror).
__global__ void k_check_mirror(Grid g, Mirror m, const double4* __restrict__ pos,
                               const int32_t* rslot, uint64_t n,
                               unsigned long long* first) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double4 p = pos[i];
  bool bad = false;
  const int32_t bs = bslot_in(p);
  const uint32_t b = mbrick(m, mpoint(m, p.x, p.y, p.z));
  if (bs < 0 || (uint32_t)(bs / m.cap) != b || bs % m.cap >= m.occ[b] || m.rid[bs] != (int32_t)i ||
      m.rx[bs] != p.x || m.ry[bs] != p.y || m.rz[bs] != p.z)
    bad = true;
  if (g.kind != GCMC_ALL_PAIRS) {
    const int c = cell_of(g, p.x, p.y, p.z);
    const int k = rslot[i];
    if (k < 0 || k >= g.occ[c] || g.slots[slot_index(g, c, k)] != (int32_t)i) bad = true;
  }
  if (bad) atomicMin(first, (unsigned long long)i);
}

struct CommitArgs {
  int kind;
  uint64_t pid, n;
  double x, y, z;
};

__global__ void k_commit_one(Grid g, Mirror m, Store s, ChainState* st, CommitArgs a,
                             long long* out) {
  MoveData d;
  d.nx = a.x;
  d.ny = a.y;
  d.nz = a.z;
  load_move(s, a.kind, a.pid, d);
  long long e1, e2, e3;
  const int r = commit_move(g, m, s, &st->peak, a.kind, a.pid, a.n, d, e1, e2, e3);
  if (r == GCMC_OK) st->n = a.kind == 1 ? a.n + 1 : (a.kind == 2 ? a.n - 1 : a.n);
  out[0] = r;
  out[1] = e1;
  out[2] = e2;
  out[3] = e3;
}

inline unsigned blocks(uint64_t n, int t) { return (unsigned)((n + t - 1) / t); }

}  // namespace

std::string strategy_name(int kind) {
  return kind == GCMC_MICROCELL ? "microcell" : (kind == GCMC_CELL_LIST ? "cell_list" : "all_pairs");
}

std::string overflow_message(const Chain& c, int64_t cell, int64_t occ) {
  std::ostringstream os;
  const bool micro = c.grid.kind == GCMC_MICROCELL;
  os << (micro ? "microcell" : "cell_list") << ": cell " << cell << " exceeds capacity "
     << c.grid.cap << " (occupancy " << occ << "); rerun with a larger "
     << (micro ? "microcell_capacity" : "cell_capacity");
  return os.str();
}

gcmc_status mirror_build(Chain& c) {
  const uint64_t n = c.st_host->n;
  c.e_valid = false;
  cudaStream_t s = c.stream;
  int* flag = c.iscratch;
  cudaError_t e;
  Mirror& m = c.mirror;
  if ((e = cudaMemsetAsync(m.occ, 0, (size_t)m.nb * sizeof(int32_t), s))) return cuda_error(e, "mirror");
  if ((e = cudaMemsetAsync(flag, 0, sizeof(int), s))) return cuda_error(e, "mirror");
  if (n) k_mbin<<<blocks(n, 256), 256, 0, s>>>(m, c.pos, n, flag);
  k_msort<<<blocks((uint64_t)m.nb * 32, 256), 256, 0, s>>>(m, c.pos);
  int overflow = 0;
  if ((e = cudaMemcpyAsync(&overflow, flag, sizeof(int), cudaMemcpyDeviceToHost, s))) return cuda_error(e, "mirror");
  if ((e = cudaStreamSynchronize(s))) return cuda_error(e, "mirror");
  c.mirror_full = overflow != 0;
  if (overflow) {
    std::ostringstream os;
    os << "mirror: brick " << overflow - 1 << " exceeds capacity " << m.cap
       << " (density too high for the evaluation mirror)";
    return set_error(GCMC_CELL_OVERFLOW, os.str());
  }
  c.built = true;
  return GCMC_OK;
}

gcmc_status grid_build(Chain& c) {
  const uint64_t n = c.st_host->n;
  c.built = false;
  if (c.grid.kind == GCMC_ALL_PAIRS) return mirror_build(c);
  cudaStream_t s = c.stream;
  int* flag = c.iscratch;
  cudaError_t e;
  if ((e = cudaMemsetAsync(c.grid.occ, 0, c.grid.ncells * sizeof(int32_t), s))) return cuda_error(e, "build");
  if ((e = cudaMemsetAsync(flag, 0, sizeof(int), s))) return cuda_error(e, "build");
  if ((e = cudaMemsetAsync(&c.st->peak, 0, sizeof(int32_t), s))) return cuda_error(e, "build");
  if (n) k_bin<<<blocks(n, 256), 256, 0, s>>>(c.grid, c.pos, n, flag);
  int overflow = 0;
  if ((e = cudaMemcpyAsync(&overflow, flag, sizeof(int), cudaMemcpyDeviceToHost, s))) return cuda_error(e, "build");
  if ((e = cudaStreamSynchronize(s))) return cuda_error(e, "build");
  if (overflow) {
    // Diagnose which cell the reference would have named.
    const uint64_t nc = c.grid.ncells;
    int *sizes = nullptr, *off = nullptr, *fill = nullptr;
    int32_t* members = nullptr;
    unsigned long long* best = nullptr;
    void* tmp = nullptr;
    size_t tmp_bytes = 0;
    cudaMalloc(&sizes, nc * sizeof(int));
    cudaMalloc(&off, nc * sizeof(int));
    cudaMalloc(&fill, nc * sizeof(int));
    cudaMalloc(&members, n * sizeof(int32_t));
    cudaMalloc(&best, sizeof(unsigned long long));
    k_overflow_sizes<<<blocks(nc, 256), 256, 0, s>>>(c.grid, sizes);
    cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, sizes, off, (int)nc, s);
    cudaMalloc(&tmp, tmp_bytes);
    cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, sizes, off, (int)nc, s);
    cudaMemsetAsync(fill, 0, nc * sizeof(int), s);
    cudaMemsetAsync(best, 0xff, sizeof(unsigned long long), s);
    k_overflow_members<<<blocks(n, 256), 256, 0, s>>>(c.grid, c.pos, n, off, fill, members);
    k_overflow_pick<<<blocks(nc, 256), 256, 0, s>>>(c.grid, off, members, best);
    unsigned long long b = 0;
    cudaMemcpyAsync(&b, best, sizeof b, cudaMemcpyDeviceToHost, s);
    e = cudaStreamSynchronize(s);
    cudaFree(sizes);
    cudaFree(off);
    cudaFree(fill);
    cudaFree(members);
    cudaFree(best);
    cudaFree(tmp);
    if (e) return cuda_error(e, "build overflow");
    return set_error(GCMC_CELL_OVERFLOW, overflow_message(c, (int64_t)(b & 0xffffffffu), c.grid.cap));
  }
  k_sort_cells<<<blocks(c.grid.ncells, 256), 256, 0, s>>>(c.grid, c.rslot, c.st);
  if ((e = cudaGetLastError())) return cuda_error(e, "build");
  return mirror_build(c);
}

gcmc_status grid_check(Chain& c, std::string* issue) {
  issue->clear();
  const uint64_t n = c.st_host->n;
  const uint64_t nc = c.grid.ncells;
  cudaStream_t s = c.stream;
  int* fresh = nullptr;
  unsigned long long* first = nullptr;
  cudaError_t e;
  if ((e = cudaMalloc(&fresh, (nc ? nc : 1) * sizeof(int)))) return cuda_error(e, "rebuild_check");
  if ((e = cudaMalloc(&first, sizeof(unsigned long long)))) return cuda_error(e, "rebuild_check");
  cudaMemsetAsync(fresh, 0, (nc ? nc : 1) * sizeof(int), s);
  cudaMemsetAsync(first, 0xff, sizeof(unsigned long long), s);
  if (nc) {
    if (n) k_fresh_count<<<blocks(n, 256), 256, 0, s>>>(c.grid, c.pos, n, fresh);
    k_check_cells<<<blocks(nc, 256), 256, 0, s>>>(c.grid, c.pos, n, fresh, first);
  }
  unsigned long long* mfirst = reinterpret_cast<unsigned long long*>(c.iscratch);
  cudaMemsetAsync(mfirst, 0xff, sizeof(unsigned long long), s);
  if (n) k_check_mirror<<<blocks(n, 256), 256, 0, s>>>(c.grid, c.mirror, c.pos, c.rslot, n, mfirst);
  unsigned long long mf = 0;
  cudaMemcpyAsync(&mf, mfirst, sizeof mf, cudaMemcpyDeviceToHost, s);
  unsigned long long f = 0;
  int fr = 0, oc = 0;
  cudaMemcpyAsync(&f, first, sizeof f, cudaMemcpyDeviceToHost, s);
  e = cudaStreamSynchronize(s);
  if (!e && f != ~0ull) {
    const uint64_t cell = f >> 8;
    cudaMemcpy(&fr, fresh + cell, sizeof(int), cudaMemcpyDeviceToHost);
    cudaMemcpy(&oc, c.grid.occ + cell, sizeof(int), cudaMemcpyDeviceToHost);
  }
  cudaFree(fresh);
  cudaFree(first);
  if (e) return cuda_error(e, "rebuild_check");
  if (f == ~0ull) {
    if (mf != ~0ull) {
      std::ostringstream os;
      os << "coordinate mirror differs from the store (particle " << mf << ")";
      *issue = os.str();
    }
    return GCMC_OK;
  }
  const uint64_t cell = f >> 8;
  const int code = (int)(f & 0xff);
  const bool micro = c.grid.kind == GCMC_MICROCELL;
  std::ostringstream os;
  if (code == 1)
    os << "rebin overflow in " << (micro ? "microcell " : "cell ") << cell;
  else if (code == 2)
    os << (micro ? "microcell " : "cell ") << cell << ": occupancy " << oc << ", rebinned " << fr;
  else if (code == 3)
    os << (micro ? "microcell " : "cell ") << cell << ": occupant sets differ from fresh binning";
  else
    os << (micro ? "microcell " : "cell ") << cell << ": coordinate mirror differs from the store";
  *issue = os.str();
  return GCMC_OK;
}

gcmc_status commit_one(Chain& c, int kind, uint64_t pid, const double* p, uint64_t* new_pid) {
  const uint64_t n = c.st_host->n;
  c.e_valid = false;  // rebuilt before the next maintained-energy engine run
  CommitArgs a{kind, pid, n, p ? p[0] : 0.0, p ? p[1] : 0.0, p ? p[2] : 0.0};
  long long* out = reinterpret_cast<long long*>(c.dscratch);
  k_commit_one<<<1, 1, 0, c.stream>>>(c.grid, c.mirror, Store{c.pos, c.rslot}, c.st, a,
                                      out);
  long long h[4];
  cudaError_t e = cudaMemcpyAsync(h, out, sizeof h, cudaMemcpyDeviceToHost, c.stream);
  if (!e) e = cudaStreamSynchronize(c.stream);
  if (e) return cuda_error(e, "commit");
  if (h[0] == GCMC_CELL_OVERFLOW) {
    if (kind == 1) c.st_host->n = n + 1;  // store already appended (microcell_grid.hpp:254)
    if (h[3]) {
      std::ostringstream os;
      os << "mirror: brick " << h[1] << " exceeds capacity " << c.mirror.cap;
      return set_error(GCMC_CELL_OVERFLOW, os.str());
    }
    return set_error(GCMC_CELL_OVERFLOW, overflow_message(c, h[1], h[2]));
  }
  if (kind == 1) {
    if (new_pid) *new_pid = n;
    c.st_host->n = n + 1;
  } else if (kind == 2) {
    c.st_host->n = n - 1;
  }
  return GCMC_OK;
}

}  // namespace gcmcb
