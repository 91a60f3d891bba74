// Device-side random initial configuration: random_initial_configuration()
// (init_config.hpp:19-64) on the B200, consuming the identical MT19937-64
// stream and producing bit-identical positions, acceptance order and final
// RNG state.
//
// The reference places candidates one at a time: three uniforms per
// candidate (rejected ones included), rejected when an already placed
// particle lies closer than min_sep (minimum image), with a coarse grid of
// side >= min_sep for the lookup. Every candidate's position is fixed by the
// stream before any decision, so candidates can be tested in blocks:
//
//   1. stream  (k_ic_stream, 1 CTA): MT19937-64 twisted block by block; the
//      uniforms and the untempered state of every 312-word block are kept
//      (the final RNG state is the block holding the next draw);
//   2. probe   (k_ic_probe): every candidate of the block against the
//      particles placed so far (27 grid cells, the reference's exact
//      minimum-image distance) -> blocked or survivor;
//   3. pairs   (k_ic_local, k_ic_pairs): survivors binned in a per-block grid;
//      each lists the EARLIER survivors (candidate order) within min_sep;
//   4. resolve (k_ic_resolve, 1 thread): candidates in order; a survivor is
//      placed unless an earlier survivor it lists was placed; ids in order,
//      the consecutive-rejection limit, the stop at the n-th placement;
//   5. commit  (k_ic_commit): placed particles into the grid and the output.
//
// Blocks are sized from the box (about one survivor neighbour pair per
// block at most), so step 4 stays short.
#include <algorithm>
#include <cstring>
#include <random>
#include <sstream>
#include <vector>

#include "internal.h"

namespace gcmcb {

namespace {

constexpr int NW = 312, MW = 156;
constexpr uint64_t MATRIX_A = 0xB5026F5AA96619E9ULL;
constexpr uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
constexpr int kCellCap = 16;     // placed particles per grid cell (side >= min_sep: <= 8 possible)
constexpr int kLocalCap = 16;    // survivors per cell of the per-block grid
constexpr int kNbr = 8;          // earlier survivors listed per survivor

__device__ __forceinline__ uint64_t temper64(uint64_t z) {
  z ^= (z >> 29) & 0x5555555555555555ULL;
  z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
  z ^= (z << 37) & 0xFFF7EEE000000000ULL;
  z ^= z >> 43;
  return z;
}

// nblocks twisted 312-word blocks after `state` (the last block, untempered):
// raw[b * 312 + k] untempered, uni[b * 312 + k] the uniform of that draw.
__global__ void __launch_bounds__(320) k_ic_stream(uint64_t* state, int nblocks, uint64_t* raw,
                                                   double* uni) {
  __shared__ uint64_t buf[2][NW];
  const int k = threadIdx.x;
  if (k < NW) buf[0][k] = state[k];
  __syncthreads();
  int cur = 0;
  for (int b = 0; b < nblocks; ++b) {
    const uint64_t* c = buf[cur];
    uint64_t* nx = buf[cur ^ 1];
    if (k < NW - MW) {
      const uint64_t y = (c[k] & UM) | (c[k + 1] & LM);
      nx[k] = c[k + MW] ^ (y >> 1) ^ ((y & 1) ? MATRIX_A : 0);
    }
    __syncthreads();
    if (k >= NW - MW && k < NW - 1) {
      const uint64_t y = (c[k] & UM) | (c[k + 1] & LM);
      nx[k] = nx[k - (NW - MW)] ^ (y >> 1) ^ ((y & 1) ? MATRIX_A : 0);
    } else if (k == NW - 1) {
      const uint64_t y = (c[NW - 1] & UM) | (nx[0] & LM);
      nx[NW - 1] = nx[MW - 1] ^ (y >> 1) ^ ((y & 1) ? MATRIX_A : 0);
    }
    __syncthreads();
    if (k < NW) {
      const uint64_t w = nx[k];
      raw[(size_t)b * NW + k] = w;
      uni[(size_t)b * NW + k] = __dmul_rn((double)(temper64(w) >> 11), 0x1.0p-53);  // rng.hpp:28-31
    }
    cur ^= 1;
  }
  if (k < NW) state[k] = buf[cur][k];
}

struct IcGrid {
  int dims;
  double inv_width;  // dims / L (init_config.hpp:26)
  double l, inv_l, min_sep2;
};

__device__ __forceinline__ int ic_coord(const IcGrid& g, double v) {
  const int c = (int)__dmul_rn(v, g.inv_width);
  return c < g.dims ? c : g.dims - 1;
}

// box.hpp:45-55, the reference's operation order (no contraction)
__device__ __forceinline__ double ic_dist2(const IcGrid& g, double ax, double ay, double az, double bx,
                                           double by, double bz) {
  double dx = __dsub_rn(ax, bx), dy = __dsub_rn(ay, by), dz = __dsub_rn(az, bz);
  dx = __dsub_rn(dx, __dmul_rn(g.l, rint(__dmul_rn(dx, g.inv_l))));
  dy = __dsub_rn(dy, __dmul_rn(g.l, rint(__dmul_rn(dy, g.inv_l))));
  dz = __dsub_rn(dz, __dmul_rn(g.l, rint(__dmul_rn(dz, g.inv_l))));
  return __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
}

// Candidate q of the block: position from draws 3 (c0 + q) .. + 2 (uniforms
// indexed from the start of the current stream buffer).
__device__ __forceinline__ void ic_cand(const IcGrid& g, const double* uni, uint64_t u0, double& x,
                                        double& y, double& z) {
  x = wrap_axis(__dmul_rn(uni[u0], g.l), g.l);
  y = wrap_axis(__dmul_rn(uni[u0 + 1], g.l), g.l);
  z = wrap_axis(__dmul_rn(uni[u0 + 2], g.l), g.l);
}

// the cube_cells(c, 1, dims) neighbourhood (grid_common.hpp), as api.cu's host form
__device__ __forceinline__ int ic_cell(const IcGrid& g, int cx, int cy, int cz, int t) {
  const int d = g.dims, span = d < 3 ? d : 3;
  const int a = t / (span * span), b = (t / span) % span, q = t % span;
  int ix = (cx - 1) % d, iy = (cy - 1) % d, iz = (cz - 1) % d;
  if (ix < 0) ix += d;
  if (iy < 0) iy += d;
  if (iz < 0) iz += d;
  ix = (ix + q) % d;
  iy = (iy + b) % d;
  iz = (iz + a) % d;
  return ix + d * (iy + d * iz);
}

// 2. probe against the placed particles; 3a. survivors into the block grid
__global__ void k_ic_probe(IcGrid g, const double* __restrict__ uni, uint64_t ubase, int nc,
                           const int* __restrict__ cnt, const int* __restrict__ slots,
                           const double* __restrict__ xyz, uint8_t* blocked, int* lcnt, int* lslots,
                           int* local_full) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nc) return;
  double x, y, z;
  ic_cand(g, uni, ubase + 3ull * q, x, y, z);
  const int cx = ic_coord(g, x), cy = ic_coord(g, y), cz = ic_coord(g, z);
  const int span = g.dims < 3 ? g.dims : 3, ncell = span * span * span;
  bool clash = false;
  for (int t = 0; t < ncell && !clash; ++t) {
    const int c = ic_cell(g, cx, cy, cz, t);
    const int m = cnt[c];
    for (int k = 0; k < m; ++k) {
      const int j = slots[(size_t)c * kCellCap + k];
      if (ic_dist2(g, x, y, z, xyz[3 * (size_t)j], xyz[3 * (size_t)j + 1], xyz[3 * (size_t)j + 2]) <
          g.min_sep2) {
        clash = true;
        break;
      }
    }
  }
  blocked[q] = clash ? 1 : 0;
  if (!clash) {
    const int c = cx + g.dims * (cy + g.dims * cz);
    const int s = atomicAdd(lcnt + c, 1);
    if (s < kLocalCap) lslots[(size_t)c * kLocalCap + s] = q;
    else atomicExch(local_full, 1);  // the block's survivor lists are incomplete
  }
}

// 3b. each survivor: the earlier survivors (candidate order) within min_sep
__global__ void k_ic_pairs(IcGrid g, const double* __restrict__ uni, uint64_t ubase, int nc,
                           const uint8_t* __restrict__ blocked, const int* __restrict__ lcnt,
                           const int* __restrict__ lslots, int* ncount, int* nlist) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nc || blocked[q]) return;
  double x, y, z;
  ic_cand(g, uni, ubase + 3ull * q, x, y, z);
  const int cx = ic_coord(g, x), cy = ic_coord(g, y), cz = ic_coord(g, z);
  const int span = g.dims < 3 ? g.dims : 3, ncell = span * span * span;
  int m = 0;
  for (int t = 0; t < ncell; ++t) {
    const int c = ic_cell(g, cx, cy, cz, t);
    const int lc = min(lcnt[c], kLocalCap);
    for (int k = 0; k < lc; ++k) {
      const int p = lslots[(size_t)c * kLocalCap + k];
      if (p >= q) continue;
      double px, py, pz;
      ic_cand(g, uni, ubase + 3ull * p, px, py, pz);
      if (ic_dist2(g, x, y, z, px, py, pz) < g.min_sep2) {
        if (m < kNbr) nlist[(size_t)q * kNbr + m] = p;
        ++m;
      }
    }
  }
  ncount[q] = m <= kNbr ? m : 255;  // 255: more than kNbr (resolved by a scan)
}

struct IcState {  // device-resident progress of the placement
  unsigned long long placed, run, consumed;  // particles placed, current rejection run, candidates consumed
  int error, pad;
};

// 4. candidates in order, decided in parallel where the order cannot matter:
// a blocked candidate is rejected, a survivor without an earlier survivor
// within min_sep is placed; only the survivors that have one (rare: blocks
// are sized to the box) are decided one by one, in order, from their lists
// (or by a scan of the block's earlier placed candidates when a list or the
// block's survivor grid overflowed). Then block scans give the ids, the stop
// at the n-th placement, and the consecutive-rejection limit (only the run
// before the block's first placement can reach it: later gaps are shorter
// than a block).
constexpr int kResolveThreads = 1024;
constexpr int kMaxBlock = 32768;

__device__ __forceinline__ int block_excl_scan(int v, int* wsum, int& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int incl = v;
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  __syncthreads();
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    int w = lane < kResolveThreads / 32 ? wsum[lane] : 0;
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += t;
    }
    if (lane < kResolveThreads / 32) wsum[lane] = w;
  }
  __syncthreads();
  total = wsum[kResolveThreads / 32 - 1];
  return incl - v + (warp ? wsum[warp - 1] : 0);
}

__global__ void __launch_bounds__(kResolveThreads)
    k_ic_resolve(IcGrid g, const double* __restrict__ uni, uint64_t ubase, int nc, uint64_t n,
                 unsigned long long max_rej, const uint8_t* __restrict__ blocked,
                 const int* __restrict__ ncount, const int* __restrict__ nlist,
                 const int* __restrict__ local_full, int* placed_id, IcState* st) {
  extern __shared__ uint8_t sm[];
  uint8_t* cnt8 = sm;                                        // [kMaxBlock] 0 blocked / no list, 1..8, 255 scan
  uint8_t* acc = sm + kMaxBlock;                             // [kMaxBlock] placed
  uint16_t* dl = reinterpret_cast<uint16_t*>(sm + 2 * kMaxBlock);  // [kMaxBlock] dependent survivors
  __shared__ int wsum[kResolveThreads / 32];
  __shared__ int s_first, s_cut;
  const bool scan_all = *local_full != 0;
  const int per = (nc + kResolveThreads - 1) / kResolveThreads;
  const int lo = threadIdx.x * per, hi = min(nc, lo + per);
  int ndep = 0;
  for (int q = lo; q < hi; ++q) {
    const bool surv = !blocked[q];
    const int c = surv ? ncount[q] : 0;
    const uint8_t m = !surv ? 0 : (scan_all ? 255 : (uint8_t)(c > 255 ? 255 : c));
    cnt8[q] = m;
    acc[q] = surv && m == 0 ? 1 : 0;
    ndep += surv && m != 0 ? 1 : 0;
  }
  int total_dep;
  int pos = block_excl_scan(ndep, wsum, total_dep);
  for (int q = lo; q < hi; ++q)
    if (!blocked[q] && cnt8[q] != 0) dl[pos++] = (uint16_t)q;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int t = 0; t < total_dep; ++t) {
      const int q = dl[t];
      const int m = cnt8[q];
      bool ok = true;
      if (m == 255) {
        double x, y, z;
        ic_cand(g, uni, ubase + 3ull * q, x, y, z);
        for (int p = 0; p < q && ok; ++p) {
          if (!acc[p]) continue;
          double px, py, pz;
          ic_cand(g, uni, ubase + 3ull * p, px, py, pz);
          if (ic_dist2(g, x, y, z, px, py, pz) < g.min_sep2) ok = false;
        }
      } else {
        for (int k = 0; k < m && ok; ++k)
          if (acc[nlist[(size_t)q * kNbr + k]]) ok = false;
      }
      acc[q] = ok ? 1 : 0;
    }
    s_first = nc;
    s_cut = nc;
  }
  __syncthreads();
  // ranks of the placed candidates; the first placement; the n-th placement
  int local = 0;
  for (int q = lo; q < hi; ++q) local += acc[q];
  int total_acc;
  int rank = block_excl_scan(local, wsum, total_acc);
  const unsigned long long placed0 = st->placed, run0 = st->run;
  const long long need = (long long)n - (long long)placed0;  // >= 1
  {
    int r = rank;
    for (int q = lo; q < hi; ++q)
      if (acc[q]) {
        if (r == 0) s_first = q;  // one thread holds rank 0
        if (r == need - 1) s_cut = q + 1;
        ++r;
      }
  }
  __syncthreads();
  int consumed = s_cut;
  bool error = false;
  // the run before the first placement (with the carried one) is the only
  // one that can reach max_rej inside a block
  if (run0 + (unsigned long long)min(s_first, consumed) >= max_rej) {
    consumed = (int)(max_rej - run0);  // the failing candidate included
    error = true;
  }
  for (int q = lo; q < hi; ++q) {
    const bool placed = acc[q] && q < consumed && !error;
    placed_id[q] = placed ? (int)(placed0 + rank) : -1;
    rank += acc[q];
  }
  if (threadIdx.x == 0) {
    if (error) {
      st->error = 1;
      st->run = max_rej;
    } else {
      const long long nplaced = need <= (long long)total_acc ? need : (long long)total_acc;
      st->placed = placed0 + (unsigned long long)nplaced;
      // rejections since the last placement within the consumed candidates
      if (nplaced == 0) st->run = run0 + (unsigned long long)consumed;
      else {
        int last = consumed - 1;
        while (last >= 0 && !acc[last]) --last;
        st->run = (unsigned long long)(consumed - 1 - last);
      }
    }
    st->consumed += (unsigned long long)consumed;
  }
}

// 5. placed particles into the grid and the output
__global__ void k_ic_commit(IcGrid g, const double* __restrict__ uni, uint64_t ubase, int nc,
                            const uint8_t* __restrict__ blocked, const int* __restrict__ placed_id,
                            int* cnt, int* slots, double* xyz, int* lcnt, int* overflow) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nc) return;
  const int id = placed_id[q];
  if (id < 0 && blocked[q]) return;
  double x, y, z;
  ic_cand(g, uni, ubase + 3ull * q, x, y, z);
  if (!blocked[q])  // the per-block grid, for the next block (every survivor's cell)
    lcnt[ic_coord(g, x) + g.dims * (ic_coord(g, y) + g.dims * ic_coord(g, z))] = 0;
  if (id < 0) return;
  xyz[3 * (size_t)id] = x;
  xyz[3 * (size_t)id + 1] = y;
  xyz[3 * (size_t)id + 2] = z;
  const int c = ic_coord(g, x) + g.dims * (ic_coord(g, y) + g.dims * ic_coord(g, z));
  const int s = atomicAdd(cnt + c, 1);
  if (s < kCellCap) slots[(size_t)c * kCellCap + s] = id;
  else atomicExch(overflow, 1);
}

struct DevBuf {
  void* p = nullptr;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
};

}  // namespace

gcmc_status device_initial_configuration(int device, uint64_t n, double l, double min_sep, uint64_t seed,
                                         double* out_xyz, uint64_t words[312], uint64_t* index,
                                         uint64_t* draws) {
  if (!(l > 0.0) || !(min_sep > 0.0)) return set_error(GCMC_ARG, "bad box or separation");
  cudaError_t e = cudaSetDevice(device);
  if (e) return cuda_error(e, "initial configuration");
  // the freshly seeded engine (rng.hpp:23): 312 words, _M_p = 312
  uint64_t seedw[313];
  {
    std::mt19937_64 eng(seed);
    std::ostringstream os;
    os << eng;
    std::istringstream is(os.str());
    for (auto& w : seedw) is >> w;
  }
  IcGrid g;
  g.dims = (int)(l / min_sep);
  if (g.dims < 1) g.dims = 1;
  g.inv_width = g.dims / l;
  g.l = l;
  g.inv_l = 1.0 / l;
  g.min_sep2 = min_sep * min_sep;
  const uint64_t ncells = (uint64_t)g.dims * g.dims * g.dims;
  // candidates per block: about vol / 8 (a few survivor pairs per block at
  // most), at most 32768
  const double vol = l * l * l;
  const int cap_b = (int)std::min((double)kMaxBlock, std::max(64.0, vol / 8.0));
  constexpr int kStreamBlocks = 4096;  // 312-word blocks per stream refill (1.28M draws)
  const uint64_t sdraws = (uint64_t)kStreamBlocks * NW;
  DevBuf bstate, braw, buni, bcnt, bslots, bxyz, bblk, blcnt, blslots, bnc, bnl, bpid, bst, bov, blf;
  cudaStream_t s = nullptr;
  auto ck = [&](cudaError_t x) { return x == cudaSuccess; };
  if (!ck(cudaMalloc(&bstate.p, NW * 8)) || !ck(cudaMalloc(&braw.p, 2 * sdraws * 8)) ||
      !ck(cudaMalloc(&buni.p, 2 * sdraws * 8)) || !ck(cudaMalloc(&bcnt.p, ncells * 4)) ||
      !ck(cudaMalloc(&bslots.p, ncells * kCellCap * 4)) || !ck(cudaMalloc(&bxyz.p, (n ? n : 1) * 24)) ||
      !ck(cudaMalloc(&bblk.p, 32768)) || !ck(cudaMalloc(&blcnt.p, ncells * 4)) ||
      !ck(cudaMalloc(&blslots.p, ncells * kLocalCap * 4)) || !ck(cudaMalloc(&bnc.p, 32768 * 4)) ||
      !ck(cudaMalloc(&bnl.p, 32768 * kNbr * 4)) || !ck(cudaMalloc(&bpid.p, 32768 * 4)) ||
      !ck(cudaMalloc(&bst.p, sizeof(IcState))) || !ck(cudaMalloc(&bov.p, 4)) ||
      !ck(cudaMalloc(&blf.p, 4)))
    return cuda_error(cudaGetLastError(), "initial configuration alloc");
  uint64_t* state = (uint64_t*)bstate.p;
  uint64_t* raw = (uint64_t*)braw.p;
  double* uni = (double*)buni.p;
  int *cnt = (int*)bcnt.p, *slots = (int*)bslots.p, *lcnt = (int*)blcnt.p, *lslots = (int*)blslots.p;
  int *ncount = (int*)bnc.p, *nlist = (int*)bnl.p, *pid = (int*)bpid.p, *ovf = (int*)bov.p;
  int* lfull = (int*)blf.p;
  const size_t rsmem = 4 * (size_t)kMaxBlock;
  if ((e = cudaFuncSetAttribute(k_ic_resolve, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rsmem)))
    return cuda_error(e, "initial configuration");
  uint8_t* blocked = (uint8_t*)bblk.p;
  double* xyz = (double*)bxyz.p;
  IcState* st = (IcState*)bst.p;
  cudaMemcpyAsync(state, seedw, NW * 8, cudaMemcpyHostToDevice, s);
  cudaMemsetAsync(cnt, 0, ncells * 4, s);
  cudaMemsetAsync(lcnt, 0, ncells * 4, s);
  cudaMemsetAsync(st, 0, sizeof(IcState), s);
  cudaMemsetAsync(ovf, 0, 4, s);
  // stream buffer: two halves of sdraws draws; draws [sbase, sbase + have)
  // are resident, the half holding draw D at ((D / sdraws) & 1)
  uint64_t sbase = 0, have = 0;  // first resident draw, resident draws
  static_assert((2ull * kStreamBlocks * NW) % 3 == 0, "the ring holds whole candidates");
  auto refill = [&]() {  // append sdraws draws (one half); when full, the oldest half goes
    if (have == 2 * sdraws) {
      sbase += sdraws;
      have -= sdraws;
    }
    const uint64_t half = ((sbase + have) / sdraws) & 1;
    k_ic_stream<<<1, 320, 0, s>>>(state, kStreamBlocks, raw + half * sdraws, uni + half * sdraws);
    have += sdraws;
  };
  refill();
  uint64_t consumed = 0;  // candidates consumed (3 draws each)
  IcState hs{};
  const unsigned long long max_rej = 1000000ull;  // init_config.hpp:22
  while (hs.placed < n && !hs.error) {
    // the block's draws must be resident and contiguous in one half-aligned
    // window: keep at least 3 * cap_b draws past the block start
    const uint64_t d0 = 3 * consumed;
    while (d0 + 3ull * cap_b > sbase + have) refill();
    // candidates of this block: draws d0 .. d0 + 3 nc within the resident window
    const uint64_t off = d0 % (2 * sdraws);
    int nc = cap_b;
    // the ring holds a multiple of 3 draws, so a block ends at its end at
    // worst (shorter block), and no candidate straddles it
    if (off + 3ull * nc > 2 * sdraws) nc = (int)((2 * sdraws - off) / 3);
    const double* u0 = uni;
    const unsigned nb = (unsigned)((nc + 255) / 256);
    cudaMemsetAsync(lfull, 0, 4, s);
    k_ic_probe<<<nb, 256, 0, s>>>(g, u0, off, nc, cnt, slots, xyz, blocked, lcnt, lslots, lfull);
    k_ic_pairs<<<nb, 256, 0, s>>>(g, u0, off, nc, blocked, lcnt, lslots, ncount, nlist);
    k_ic_resolve<<<1, kResolveThreads, rsmem, s>>>(g, u0, off, nc, n, max_rej, blocked, ncount, nlist,
                                                   lfull, pid, st);
    k_ic_commit<<<nb, 256, 0, s>>>(g, u0, off, nc, blocked, pid, cnt, slots, xyz, lcnt, ovf);
    IcState prev = hs;
    int hov = 0;
    cudaMemcpyAsync(&hs, st, sizeof hs, cudaMemcpyDeviceToHost, s);
    cudaMemcpyAsync(&hov, ovf, 4, cudaMemcpyDeviceToHost, s);
    if ((e = cudaStreamSynchronize(s))) return cuda_error(e, "initial configuration");
    if (hov) return set_error(GCMC_ARG, "initial configuration: device grid capacity exceeded");
    consumed += hs.consumed - prev.consumed;
  }
  if (hs.error)
    return set_error(GCMC_ARG, "initial configuration: 1000000 consecutive rejections; "
                               "density too high for the minimum separation");
  if (n && (e = cudaMemcpy(out_xyz, xyz, n * 24, cudaMemcpyDeviceToHost)))
    return cuda_error(e, "initial configuration");
  // RNG state after 3 * consumed draws: the block holding the next draw
  // (lazy twist: after a whole block the index is 312 and the state that block)
  const uint64_t dtot = 3 * consumed;
  uint64_t blk, idx;
  if (dtot == 0) {
    std::memcpy(words, seedw, NW * 8);
    *index = NW;
  } else {
    blk = (dtot - 1) / NW;  // block of the last consumed draw
    idx = dtot - blk * NW;  // 1..312
    const uint64_t first = blk * NW;
    if (first < sbase) return set_error(GCMC_STATE, "initial configuration: stream window lost");
    const uint64_t pos = first % (2 * sdraws);
    if ((e = cudaMemcpy(words, raw + pos, NW * 8, cudaMemcpyDeviceToHost)))
      return cuda_error(e, "initial configuration");
    *index = idx;
  }
  if (draws) *draws = dtot;
  return GCMC_OK;
}

}  // namespace gcmcb
