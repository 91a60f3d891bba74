// Incremental relink of the spatial indexes on an accepted move — the device
// form of commit_displace / commit_insert / commit_delete and their helpers
// insert_id / remove_id / relabel_id (microcell_grid.hpp:243-268, 472-513;
// cell_grid.hpp:140-166, 237-275; particles.hpp:28-41).
//
// Two structures are maintained, both with the reference's swap-last
// semantics:
//   Grid    the strategy's reference layout (occ/slots), byte-identical to
//           occupancy_view()/slots_view() after every commit (a vacated slot
//           keeps its stale id exactly as remove_id leaves it);
//   Mirror  the brick records the ΔE kernels read (slot.cuh).
// Per-particle back-pointers rslot[i] (slot of i in its reference cell) and
// bslot[i] (record index of i in the mirror) replace the reference's linear
// "find id in cell" scans, so a commit is two dependent loads (occupancy,
// last occupant) and a fixed handful of stores.
//
// The mover's own inputs (old position and back-pointers) arrive in
// MoveData, loaded when the move was evaluated (the engine guarantees nothing
// changed them since); everything else — occupancies, last occupants, and
// for a deletion the last particle q = n-1 — is loaded here, so commits
// applied in move order by one thread are exact whatever the evaluation saw
// of earlier commits.
#pragma once
#include "mirror.cuh"

namespace gcmcb {

struct Store {
  double4* pos;    // (x, y, z, mirror back-pointer in the low word of w)
  int32_t* rslot;
};

struct MoveData {
  double nx, ny, nz;           // new position (displace / insert)
  double ox, oy, oz;           // old position of pid (displace / delete)
  int32_t rslot_pid, bslot_pid;
};

// Load MoveData's per-particle fields of the mover (one thread).
__device__ __forceinline__ void load_move(const Store& s, int kind, uint64_t pid, MoveData& d) {
  if (kind != 1) {
    const double4 o = ld_cg(s.pos + pid);
    d.ox = o.x;
    d.oy = o.y;
    d.oz = o.z;
    d.rslot_pid = __ldcg(s.rslot + pid);
    d.bslot_pid = bslot_in(o);
  }
}

// Everything a commit reads besides MoveData (two dependent L2 hops).
struct CommitIn {
  double qx, qy, qz;
  int32_t rslot_q, bslot_q;
  int32_t rslot_pid;  // slot of the mover in its reference cell (loaded here)
  int ca, cb, cl, occ_ca, occ_cb;
  int ba, bb, occ_ba, occ_bb, la;
  int32_t last_ca, last_bid;
  double lx, ly, lz;
  bool relabel, ref_move, mir_move;
};

// kind 0 displace (pid -> new), 1 insert (new, id n), 2 delete (pid; the last
// particle q = n-1 takes its id). n = store size before the move.
__device__ __forceinline__ void commit_load(const Grid& g, const Mirror& m, const Store& s,
                                            int kind, uint64_t pid, uint64_t n,
                                            const MoveData& d, CommitIn& c) {
  const bool grid = g.kind != GCMC_ALL_PAIRS;
  const uint64_t q = n - 1;
  c.relabel = kind == 2 && pid != q;
  // ---- hop 1: cells, occupancies, the last particle
  c.qx = c.qy = c.qz = 0.0;
  c.rslot_q = c.bslot_q = -1;
  c.rslot_pid = (kind != 1 && grid) ? __ldcg(s.rslot + pid) : -1;
  if (c.relabel) {
    const double4 o = ld_cg(s.pos + q);
    c.qx = o.x;
    c.qy = o.y;
    c.qz = o.z;
    c.rslot_q = __ldcg(s.rslot + q);
    c.bslot_q = bslot_in(o);
  }
  c.ca = c.cb = c.cl = -1;
  c.occ_ca = c.occ_cb = 0;
  c.ba = c.bb = -1;
  c.occ_ba = c.occ_bb = 0;
  if (kind != 1) {
    c.ba = (int)mbrick(m, mpoint(m, d.ox, d.oy, d.oz));
    c.occ_ba = __ldcg(m.occ + c.ba);
    if (grid) {
      c.ca = cell_of(g, d.ox, d.oy, d.oz);
      c.occ_ca = __ldcg(g.occ + c.ca);
    }
  }
  if (kind != 2) {
    c.bb = (int)mbrick(m, mpoint(m, d.nx, d.ny, d.nz));
    c.occ_bb = __ldcg(m.occ + c.bb);
    if (grid) {
      c.cb = cell_of(g, d.nx, d.ny, d.nz);
      c.occ_cb = __ldcg(g.occ + c.cb);
    }
  }
  if (grid && c.relabel) c.cl = cell_of(g, c.qx, c.qy, c.qz);
  c.ref_move = grid && (kind == 2 || (kind == 0 && c.ca != c.cb));
  c.mir_move = kind == 2 || (kind == 0 && c.ba != c.bb);
  // ---- hop 2: last occupants of the cell / brick left
  c.last_ca = c.last_bid = -1;
  c.lx = c.ly = c.lz = 0.0;
  c.la = c.ba * m.cap + c.occ_ba - 1;
  if (c.ref_move) c.last_ca = __ldcg(g.slots + slot_index(g, c.ca, c.occ_ca - 1));
  if (c.mir_move) {
    c.last_bid = __ldcg(m.rid + c.la);
    c.lx = __ldcg(m.rx + c.la);
    c.ly = __ldcg(m.ry + c.la);
    c.lz = __ldcg(m.rz + c.la);
  }
}

// Stores only. Returns GCMC_OK or GCMC_CELL_OVERFLOW (e1 = cell, e2 =
// occupancy; e3 = 1 for the mirror), after the reference's partial effects
// (store updated, particle removed from its old cell) as in
// commit_displace/commit_insert when insert_id throws.
__device__ __forceinline__ int commit_store(const Grid& g, const Mirror& m, const Store& s,
                                            int32_t* peak, int kind, uint64_t pid, uint64_t n,
                                            const MoveData& d, const CommitIn& c, long long& e1,
                                            long long& e2, long long& e3, bool skip_index = false) {
  const bool grid = g.kind != GCMC_ALL_PAIRS;
  const uint64_t q = n - 1;
  e1 = e2 = e3 = 0;
  int status = GCMC_OK;
  // ---- store (particles.hpp:28-41)
  if (kind == 0) st_xyz(s.pos + pid, d.nx, d.ny, d.nz);
  // skip_index: an insertion whose particle a later deletion of the same
  // batch relabels (and takes its data from registers) leaves index n unused
  if (kind == 1 && !skip_index) st_xyz(s.pos + n, d.nx, d.ny, d.nz);
  // ---- reference layout
  if (grid) {
    if (c.ref_move) {  // remove_id: the last id fills the hole
      const int k = c.rslot_pid, last = c.occ_ca - 1;
      if (k != last) {
        __stcg(g.slots + slot_index(g, c.ca, k), c.last_ca);
        if (!(c.relabel && c.last_ca == (int32_t)q)) __stcg(s.rslot + c.last_ca, k);
      }
      __stcg(g.occ + c.ca, last);
    }
    if (kind == 1 || (kind == 0 && c.ca != c.cb)) {  // insert_id
      if (c.occ_cb >= g.cap) {
        status = GCMC_CELL_OVERFLOW;
        e1 = c.cb;
        e2 = c.occ_cb;
      } else {
        const int32_t id = kind == 1 ? (int32_t)n : (int32_t)pid;
        __stcg(g.slots + slot_index(g, c.cb, c.occ_cb), id);
        if (!skip_index) __stcg(s.rslot + id, c.occ_cb);
        __stcg(g.occ + c.cb, c.occ_cb + 1);
        atomicMax(peak, c.occ_cb + 1);
      }
    }
    if (c.relabel) {  // relabel_id(last -> pid)
      const int rq = c.last_ca == (int32_t)q ? c.rslot_pid : c.rslot_q;
      __stcg(g.slots + slot_index(g, c.cl, rq), (int32_t)pid);
      __stcg(s.rslot + pid, rq);
    }
  }
  // ---- mirror
  if (kind == 0 && !c.mir_move) {
    __stcg(m.rx + d.bslot_pid, d.nx);
    __stcg(m.ry + d.bslot_pid, d.ny);
    __stcg(m.rz + d.bslot_pid, d.nz);
  } else {
    if (c.mir_move) {
      const int k = d.bslot_pid;
      if (k != c.la) {
        __stcg(m.rx + k, c.lx);
        __stcg(m.ry + k, c.ly);
        __stcg(m.rz + k, c.lz);
        __stcg(m.rid + k, c.last_bid);
        if (!(c.relabel && c.last_bid == (int32_t)q)) __stcg(bslot_of(s.pos, c.last_bid), k);
      }
      __stcg(m.occ + c.ba, c.occ_ba - 1);
    }
    if (kind != 2) {
      if (c.occ_bb >= m.cap) {
        if (status == GCMC_OK) {
          status = GCMC_CELL_OVERFLOW;
          e1 = c.bb;
          e2 = c.occ_bb;
          e3 = 1;
        }
      } else {
        const int32_t id = kind == 1 ? (int32_t)n : (int32_t)pid;
        const int k = c.bb * m.cap + c.occ_bb;
        __stcg(m.rx + k, d.nx);
        __stcg(m.ry + k, d.ny);
        __stcg(m.rz + k, d.nz);
        __stcg(m.rid + k, id);
        if (!skip_index) __stcg(bslot_of(s.pos, id), k);
        __stcg(m.occ + c.bb, c.occ_bb + 1);
      }
    }
    if (c.relabel) {
      const int bq = c.last_bid == (int32_t)q ? d.bslot_pid : c.bslot_q;
      __stcg(m.rid + bq, (int32_t)pid);
      __stcg(bslot_of(s.pos, pid), bq);
      st_xyz(s.pos + pid, c.qx, c.qy, c.qz);
    }
  }
  return status;
}

// What a commit touches (reads or writes), for ordering concurrent commits:
// reference cells, mirror bricks, particle indices.
struct Touch {
  int cell[3], brick[3];
  int64_t part[5];
};
__device__ __forceinline__ Touch touch_of(const Mirror& m, int kind, uint64_t pid, uint64_t n,
                                          const CommitIn& c) {
  Touch t;
  t.cell[0] = c.ca;
  t.cell[1] = c.cb;
  t.cell[2] = c.cl;
  t.brick[0] = c.ba;
  t.brick[1] = c.bb;
  t.brick[2] = c.relabel && c.bslot_q >= 0 ? c.bslot_q / m.cap : -1;
  t.part[0] = kind != 1 ? (int64_t)pid : (int64_t)n;
  t.part[1] = kind == 2 ? (int64_t)(n - 1) : -1;
  t.part[2] = c.last_ca;
  t.part[3] = c.last_bid;
  t.part[4] = -1;
  return t;
}
__device__ __forceinline__ bool touches(const Touch& a, const Touch& b) {
#pragma unroll
  for (int x = 0; x < 3; ++x)
#pragma unroll
    for (int y = 0; y < 3; ++y) {
      if (a.cell[x] >= 0 && a.cell[x] == b.cell[y]) return true;
      if (a.brick[x] >= 0 && a.brick[x] == b.brick[y]) return true;
    }
#pragma unroll
  for (int x = 0; x < 5; ++x)
#pragma unroll
    for (int y = 0; y < 5; ++y)
      if (a.part[x] >= 0 && a.part[x] == b.part[y]) return true;
  return false;
}

// One thread: load + store.
__device__ __forceinline__ int commit_move(const Grid& g, const Mirror& m, const Store& s,
                                           int32_t* peak, int kind, uint64_t pid, uint64_t n,
                                           const MoveData& d, long long& e1, long long& e2,
                                           long long& e3) {
  CommitIn c;
  commit_load(g, m, s, kind, pid, n, d, c);
  return commit_store(g, m, s, peak, kind, pid, n, d, c, e1, e2, e3);
}

}  // namespace gcmcb
