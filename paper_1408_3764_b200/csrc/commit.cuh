// Incremental relink of the spatial index on an accepted move — the device
// form of commit_displace / commit_insert / commit_delete and their helpers
// insert_id / remove_id / relabel_id (microcell_grid.hpp:243-268, 472-513;
// cell_grid.hpp:140-166, 237-275; particles.hpp:28-41).
//
// Split in two so the loads leave the serial path:
//   commit_prefetch  (one warp, during the move's evaluation) loads every
//                    slot + coordinate-mirror record of the cell the particle
//                    leaves, the occupancy of the cell it enters, and for a
//                    deletion the last record and its cell;
//   commit_apply     (lane 0, after the move won the round) replays the
//                    reference's sequential bookkeeping on those copies and
//                    issues only stores.
// The evaluation state is the commit state (nothing changes in between), so
// the prefetched copies are exact. Slot order after every commit is
// byte-identical to the reference.
#pragma once
#include "common.cuh"

namespace gcmcb {

struct CellView {
  int cell, occ;
  int32_t ids[kMaxCap];
  double4 rec[kMaxCap];
};

struct CommitPlan {
  CellView a;        // cell the particle leaves (displace / remove)
  CellView l;        // cell of the last record (remove, pid != last)
  int cb, occb;      // cell entered (displace / insert) and its occupancy
  int ca, cl;
  double4 lastp;     // position of the last record (remove)
  int status;
  long long e1, e2;
};

__device__ __forceinline__ void load_view(const Grid& g, int cell, CellView& v, int lane) {
  if (lane == 0) {
    v.cell = cell;
    v.occ = ld_cg(g.occ + cell);
  }
  for (int k = lane; k < g.cap; k += 32) {
    const uint64_t s = slot_index(g, cell, k);
    v.ids[k] = ld_cg(g.slots + s);
    v.rec[k] = ld_cg(g.cellpos + s);
  }
}

// One warp. kind 0 displace (pid, old -> p), 1 insert (p), 2 remove (pid).
__device__ __forceinline__ void commit_prefetch(const Grid& g, const double4* pos, uint64_t n,
                                                int kind, uint64_t pid, double4 old, double px,
                                                double py, double pz, CommitPlan& cp) {
  const int lane = threadIdx.x & 31;
  if (g.kind == GCMC_ALL_PAIRS) {
    if (kind == 2 && lane == 0 && pid != n - 1) cp.lastp = ld_cg(pos + n - 1);
    return;
  }
  const int ca = (kind != 1) ? cell_of(g, old.x, old.y, old.z) : -1;
  const int cb = (kind != 2) ? cell_of(g, px, py, pz) : -1;
  if (lane == 0) {
    cp.ca = ca;
    cp.cb = cb;
    cp.occb = cb >= 0 ? ld_cg(g.occ + cb) : 0;
  }
  if (ca >= 0) load_view(g, ca, cp.a, lane);
  if (kind == 2 && pid != n - 1) {
    const double4 lp = ld_cg(pos + n - 1);
    const int cl = cell_of(g, lp.x, lp.y, lp.z);
    if (lane == 0) {
      cp.lastp = lp;
      cp.cl = cl;
    }
    if (cl != ca) load_view(g, cl, cp.l, lane);
  }
}

// Lane 0 only. Returns GCMC_OK or an error status (detail in cp.e1/e2).
__device__ __forceinline__ int commit_apply(const Grid& g, double4* pos, ChainState* st,
                                            uint64_t n, int kind, uint64_t pid, double px,
                                            double py, double pz, CommitPlan& cp) {
  const bool grid = g.kind != GCMC_ALL_PAIRS;
  const uint64_t last = n - 1;
  int status = GCMC_OK;
  cp.e1 = cp.e2 = 0;
  // store update (particles.hpp:28-41)
  if (kind == 0) st_cg(pos + pid, make_double4(px, py, pz, 0.0));
  if (kind == 1) st_cg(pos + n, make_double4(px, py, pz, 0.0));
  auto remove_from = [&](CellView& v, int32_t id) -> bool {
    for (int k = 0; k < v.occ; ++k) {
      if (v.ids[k] == id) {
        const int e = v.occ - 1;
        v.ids[k] = v.ids[e];
        v.rec[k] = v.rec[e];
        --v.occ;
        const uint64_t s = slot_index(g, v.cell, k);
        __stcg(g.slots + s, v.ids[k]);
        st_cg(g.cellpos + s, v.rec[k]);
        __stcg(g.occ + v.cell, v.occ);
        return true;
      }
    }
    status = GCMC_NOT_FOUND;
    cp.e1 = id;
    cp.e2 = v.cell;
    return false;
  };
  auto insert_into = [&](int cell, int occ, int32_t id, double x, double y, double z) {
    if (occ >= g.cap) {
      status = GCMC_CELL_OVERFLOW;
      cp.e1 = cell;
      cp.e2 = occ;
      return;
    }
    const uint64_t s = slot_index(g, cell, occ);
    __stcg(g.slots + s, id);
    st_cg(g.cellpos + s, make_double4(x, y, z, pid_bits((uint64_t)id)));
    __stcg(g.occ + cell, occ + 1);
    atomicMax(&st->peak, occ + 1);
  };
  if (grid) {
    if (kind == 0) {
      if (cp.ca == cp.cb) {  // same cell: slots unchanged, refresh the mirror record
        int k = 0;
        while (k < cp.a.occ && cp.a.ids[k] != (int32_t)pid) ++k;
        if (k == cp.a.occ) {
          status = GCMC_NOT_FOUND;
          cp.e1 = (long long)pid;
          cp.e2 = cp.ca;
        } else {
          st_cg(g.cellpos + slot_index(g, cp.ca, k), make_double4(px, py, pz, pid_bits(pid)));
        }
      } else if (remove_from(cp.a, (int32_t)pid)) {
        insert_into(cp.cb, cp.occb, (int32_t)pid, px, py, pz);
      }
    } else if (kind == 1) {
      insert_into(cp.cb, cp.occb, (int32_t)n, px, py, pz);
    } else if (remove_from(cp.a, (int32_t)pid) && pid != last) {
      CellView& v = cp.cl == cp.ca ? cp.a : cp.l;  // relabel last -> pid
      int k = 0;
      while (k < v.occ && v.ids[k] != (int32_t)last) ++k;
      if (k == v.occ) {
        status = GCMC_NOT_FOUND;
        cp.e1 = (long long)last;
        cp.e2 = cp.cl;
      } else {
        const uint64_t s = slot_index(g, cp.cl, k);
        __stcg(g.slots + s, (int32_t)pid);
        st_cg(g.cellpos + s, make_double4(cp.lastp.x, cp.lastp.y, cp.lastp.z, pid_bits(pid)));
      }
    }
  }
  if (kind == 2 && pid != last)
    st_cg(pos + pid, make_double4(cp.lastp.x, cp.lastp.y, cp.lastp.z, 0.0));
  cp.status = status;
  return status;
}

}  // namespace gcmcb
