// Proposal generation: the reference's RngStream (std::mt19937_64,
// rng.hpp:26-31,84) reproduced bit-for-bit on the device, and the move
// stream parsed out of it.
//
// Every move consumes a fixed number of draws for its kind, accepted or not
// (engine.hpp:207-213): displace = selector, pick, u1, u2, u3, accept (6);
// insert = selector, source, u1, u2, u3, accept (6); remove = selector,
// source, pick, accept (4); the accept draw is taken before ΔE
// (engine.hpp:352-354, 381-382, 397-398). Kinds, targets and accept draws
// are therefore state-independent: only pid = index_from(pick, N) needs the
// state. This kernel turns the MT stream into Proposal records ahead of the
// engine, and leaves the MT state exactly where libstdc++ would be after
// those moves (lazy twist: _M_p == 312 until the next draw).
//
// One CTA: 312 threads twist a 312-word block in two dependent phases,
// temper it into doubles; warp 0 parses the block with a 6-state finite
// automaton per 10-draw lane segment (move starts are reachable only at
// offsets 0..5 into a segment), composes the lane maps with a warp scan, then
// re-walks and emits.
#include <cstdlib>

#include <vector>

#include "internal.h"
#include "mirror.cuh"

namespace gcmcb {

namespace {

constexpr int N = 312, M = 156;
constexpr uint64_t MATRIX_A = 0xB5026F5AA96619E9ULL;
constexpr uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
constexpr int kThreads = 320;
constexpr int kSeg = 10;

__device__ __forceinline__ uint64_t temper(uint64_t z) {
  z ^= (z >> 29) & 0x5555555555555555ULL;
  z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
  z ^= (z << 37) & 0xFFF7EEE000000000ULL;
  z ^= z >> 43;
  return z;
}

__device__ __forceinline__ double to_uniform(uint64_t z) {
  return __dmul_rn((double)(z >> 11), 0x1.0p-53);  // rng.hpp:28-31
}

// next = twist(cur); both in shared memory; all threads participate.
__device__ void twist(const uint64_t* cur, uint64_t* nxt) {
  const int k = threadIdx.x;
  if (k < N - M) {
    const uint64_t y = (cur[k] & UM) | (cur[k + 1] & LM);
    nxt[k] = cur[k + M] ^ (y >> 1) ^ ((y & 1) ? MATRIX_A : 0);
  }
  __syncthreads();
  if (k >= N - M && k < N - 1) {
    const uint64_t y = (cur[k] & UM) | (cur[k + 1] & LM);
    nxt[k] = nxt[k - (N - M)] ^ (y >> 1) ^ ((y & 1) ? MATRIX_A : 0);
  } else if (k == N - 1) {
    const uint64_t y = (cur[N - 1] & UM) | (nxt[0] & LM);
    nxt[N - 1] = nxt[M - 1] ^ (y >> 1) ^ ((y & 1) ? MATRIX_A : 0);
  }
  __syncthreads();
}

struct GenArgs {
  uint64_t* mt;      // [312 words, idx, draws]
  Proposal* out;
  uint64_t nmoves;
  double dp;         // displace_percent
  double l;          // box length
  int raw_disp;      // max_displacement > 0: keep u1..u3 raw
};

// KB blocks of 312 draws per iteration. All threads twist and temper the KB
// blocks in sequence (the MT recurrence is serial); then warp w parses block
// w for all six possible entry offsets at once (lane segment maps composed by
// a warp scan -> the block's entry->exit map), one thread chains the KB block
// maps from the known entry, and every warp emits its block's moves at its
// resolved entry and move index (KB x fewer serial parse steps than parsing
// one block at a time).
constexpr int KB = 8;

__device__ __forceinline__ uint32_t compose6(uint32_t g, uint32_t h) {  // (g o h)(x) = g(h(x))
  uint32_t comp = 0;
#pragma unroll
  for (int x = 0; x < 6; ++x) {
    const uint32_t hx = (h >> (3 * x)) & 7u;
    comp |= ((g >> (3 * hx)) & 7u) << (3 * x);
  }
  return comp;
}

// One chain per CTA: the arguments by value (one chain) or from a device
// list indexed by blockIdx.x (K chains in one launch).
template <bool kMulti>
__global__ void __launch_bounds__(kThreads) k_gen2(GenArgs one, const GenArgs* __restrict__ list) {
  const GenArgs a = kMulti ? list[blockIdx.x] : one;
  __shared__ uint64_t rawb[KB + 1][N];  // raw MT words of the iteration's blocks
  __shared__ double dr[KB + 1][N];      // their uniforms
  __shared__ uint32_t s_map[KB];
  __shared__ int s_entry[KB + 1], s_base[KB + 1], s_cnt[KB], s_endb, s_endp, s_done;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (a.nmoves == 0) return;
  if (tid < N) rawb[0][tid] = a.mt[tid];
  const uint64_t idx0 = a.mt[N];
  const uint64_t draws0 = a.mt[N + 1];
  __syncthreads();
  int entry;
  if (idx0 >= (uint64_t)N) {
    twist(rawb[0], rawb[1]);
    if (tid < N) rawb[0][tid] = rawb[1][tid];
    __syncthreads();
    entry = 0;
  } else {
    entry = (int)idx0;
  }
  if (tid < N) dr[0][tid] = to_uniform(temper(rawb[0][tid]));
  uint64_t emitted = 0, consumed = 0;
  bool firstit = true;
  for (;;) {
    // a resumed stream may start deep inside block 0: its segments then start
    // at the entry (the automaton covers entry offsets 0..5 of a segment)
    const int org0 = firstit && entry >= 6 ? entry : 0;
    for (int b = 1; b <= KB; ++b) {  // the MT recurrence: serial over blocks
      twist(rawb[b - 1], rawb[b]);
      if (tid < N) dr[b][tid] = to_uniform(temper(rawb[b][tid]));
    }
    __syncthreads();
    // ---- phase A: warp w parses block w for all six entry offsets
    const int wb = warp < KB ? warp : 0;
    const double* d0 = dr[wb];
    const double* d1 = dr[wb + 1];
    auto D = [&](int p) { return p < N ? d0[p] : d1[p - N]; };
    auto len_at = [&](int p) {
      if (D(p) < a.dp) return 6;              // displace (engine.hpp:296)
      return D(p + 1) < 0.5 ? 4 : 6;          // remove : insert (engine.hpp:298)
    };
    const int seg0 = (warp == 0 ? org0 : 0) + kSeg * lane;
    const int seg1 = min(seg0 + kSeg, N);
    const bool active = seg0 < N;
    uint32_t cnts = 0, g = 0;
    if (warp < KB) {
      uint32_t fmap = 0;
      for (int x = 0; x < 6; ++x) {
        int p = seg0 + x, c = 0;
        if (active)
          while (p < seg1) {
            p += len_at(p);
            ++c;
          }
        const int ex = active ? p - seg1 : x;
        fmap |= (uint32_t)ex << (3 * x);
        cnts |= (uint32_t)c << (3 * x);
      }
      g = fmap;  // inclusive composition G_l = f_l o ... o f_0
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t h = __shfl_up_sync(0xffffffffu, g, o);
        if (lane >= o) g = compose6(g, h);
      }
      if (lane == 31) s_map[warp] = g;
    }
    __syncthreads();
    // ---- phase B: chain the block maps from the known entry
    if (tid == 0) {
      int e = entry - org0;
      for (int b = 0; b < KB; ++b) {
        s_entry[b] = e;
        e = (int)((s_map[b] >> (3 * e)) & 7u);
      }
      s_entry[KB] = e;
    }
    __syncthreads();
    // ---- phase C: moves per lane at the resolved entry, per-block totals
    int x_in = 0, my_cnt = 0, incl = 0;
    if (warp < KB) {
      const int eb = s_entry[warp];
      const uint32_t gprev = __shfl_up_sync(0xffffffffu, g, 1);
      x_in = lane == 0 ? eb : (int)((gprev >> (3 * eb)) & 7u);
      my_cnt = active ? (int)((cnts >> (3 * x_in)) & 7u) : 0;
      incl = my_cnt;
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
      }
      if (lane == 31) s_cnt[warp] = incl;
    }
    __syncthreads();
    if (tid == 0) {
      int base = 0;
      s_done = 0;
      s_endb = -1;
      for (int b = 0; b < KB; ++b) {
        s_base[b] = base;
        if (!s_done && emitted + (uint64_t)(base + s_cnt[b]) >= a.nmoves) {
          s_done = 1;
          s_endb = b;
        }
        base += s_cnt[b];
      }
      s_base[KB] = base;
      s_endp = -1;
    }
    __syncthreads();
    // ---- phase D: emit
    if (warp < KB) {
      uint64_t mi = emitted + (uint64_t)(s_base[warp] + incl - my_cnt);
      int p = seg0 + x_in;
      if (active)
        while (p < seg1) {
          const int len = len_at(p);
          if (mi < a.nmoves) {
            Proposal pr;
            pr.wmask = kNoMask;
            pr.bpt = 0;
            pr.cell = 0;
            const double sel = D(p);
            if (sel < a.dp) {
              pr.kind = 0;
              pr.pick = D(p + 1);
              const double u1 = D(p + 2), u2 = D(p + 3), u3 = D(p + 4);
              if (a.raw_disp) {
                pr.x = u1;
                pr.y = u2;
                pr.z = u3;
              } else {  // point_from (engine.hpp:345-348)
                pr.x = wrap_axis(__dmul_rn(u1, a.l), a.l);
                pr.y = wrap_axis(__dmul_rn(u2, a.l), a.l);
                pr.z = wrap_axis(__dmul_rn(u3, a.l), a.l);
              }
              pr.acc = D(p + 5);
            } else if (D(p + 1) < 0.5) {
              pr.kind = 2;
              pr.pick = D(p + 2);
              pr.acc = D(p + 3);
              pr.x = pr.y = pr.z = 0.0;
            } else {
              pr.kind = 1;
              pr.pick = 0.0;
              pr.x = wrap_axis(__dmul_rn(D(p + 2), a.l), a.l);
              pr.y = wrap_axis(__dmul_rn(D(p + 3), a.l), a.l);
              pr.z = wrap_axis(__dmul_rn(D(p + 4), a.l), a.l);
              pr.acc = D(p + 5);
            }
            a.out[mi] = pr;
            if (mi == a.nmoves - 1) s_endp = p + len;  // in block s_endb, may pass its end
          }
          ++mi;
          p += len;
        }
    }
    __syncthreads();
    if (s_done) {
      const int eb = s_endb, endp = s_endp;
      consumed += (uint64_t)(eb * N + endp - entry);
      const int fb = endp <= N ? eb : eb + 1;  // block holding the next draw (lazy twist at N)
      const int fidx = endp <= N ? endp : endp - N;
      if (tid < N) a.mt[tid] = rawb[fb][tid];
      if (tid == 0) {
        a.mt[N] = (uint64_t)fidx;
        a.mt[N + 1] = draws0 + consumed;
      }
      return;
    }
    emitted += (uint64_t)s_base[KB];
    consumed += (uint64_t)(KB * N + s_entry[KB] - entry);
    entry = s_entry[KB];
    firstit = false;
    if (tid < N) {  // block KB is block 0 of the next iteration
      rawb[0][tid] = rawb[KB][tid];
      dr[0][tid] = dr[KB][tid];
    }
    __syncthreads();
  }
}

// The state-independent part of each proposal's evaluation, once per
// proposal and off the engine's critical path: the pruned brick window of the
// new position (window_keep, the same arithmetic as the engine's own
// window_bricks_warp), its packed brick point and reference-grid cell.
// Deletions and max_displacement displacements (new position relative to the
// mover) get kNoMask and are computed in the engine.
struct AnnArgs {
  Proposal* p;
  uint64_t n;
  Mirror m;
  Box b;
  Grid g;
  int raw;
};
template <bool kMulti>
__global__ void __launch_bounds__(256) k_annotate(AnnArgs one, const AnnArgs* __restrict__ list) {
  const AnnArgs& A = kMulti ? list[blockIdx.y] : one;
  Proposal* const p = A.p;
  const uint64_t n = A.n;
  const Mirror m = A.m;
  const Box b = A.b;
  const Grid g = A.g;
  const int raw = A.raw;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    Proposal& q = p[i];
    uint32_t mask = kNoMask, bpt = 0;
    int cell = 0;
    if (q.kind != 2 && !(q.kind == 0 && raw) && m.dims >= 3) {
      const double x = q.x, y = q.y, z = q.z;
      const int bx = mcoord(m, x), by = mcoord(m, y), bz = mcoord(m, z);
      mask = 0;
      for (int l = 0; l < 27; ++l) {
        uint32_t id;
        if (window_keep(m, b, x, y, z, bx, by, bz, l, id)) mask |= 1u << l;
      }
      bpt = (uint32_t)bx | ((uint32_t)by << 8) | ((uint32_t)bz << 16);
      if (g.kind != GCMC_ALL_PAIRS) cell = cell_of(g, x, y, z);
    }
    q.wmask = mask;
    q.bpt = bpt;
    q.cell = cell;
  }
}

}  // namespace

gcmc_status gen_proposals(Chain& c, uint64_t n, cudaStream_t s) {
  return gen_proposals_into(c, c.mt, c.props, n, s);
}

gcmc_status gen_proposals_into(Chain& c, uint64_t* mt, Proposal* out, uint64_t n, cudaStream_t s) {
  if (n == 0) return GCMC_OK;
  GenArgs a{mt, out, n, c.params.displace_percent, c.box.l,
            c.params.max_displacement > 0.0 ? 1 : 0};
  k_gen2<false><<<1, kThreads, 0, s>>>(a, nullptr);
  const unsigned blocks = (unsigned)((n + 255) / 256 < 1024 ? (n + 255) / 256 : 1024);
  k_annotate<false><<<blocks, 256, 0, s>>>(AnnArgs{out, n, c.mirror, c.box, c.grid, a.raw_disp}, nullptr);
  cudaError_t e = cudaGetLastError();
  if (e) return cuda_error(e, "gen_proposals");
  return GCMC_OK;
}

gcmc_status gen_proposals_many(Chain* const* cs, int k, const uint64_t* n, cudaStream_t s) {
  std::vector<GenArgs> ga;
  std::vector<AnnArgs> aa;
  uint64_t nmax = 0;
  for (int i = 0; i < k; ++i) {
    if (n[i] == 0) continue;
    Chain& c = *cs[i];
    ga.push_back(GenArgs{c.mt, c.props, n[i], c.params.displace_percent, c.box.l,
                         c.params.max_displacement > 0.0 ? 1 : 0});
    aa.push_back(AnnArgs{c.props, n[i], c.mirror, c.box, c.grid, ga.back().raw_disp});
    nmax = n[i] > nmax ? n[i] : nmax;
  }
  if (ga.empty()) return GCMC_OK;
  const int kk = (int)ga.size();
  void* d = nullptr;
  const size_t bytes = kk * (sizeof(GenArgs) + sizeof(AnnArgs));
  cudaError_t e = cudaMallocAsync(&d, bytes, s);
  if (e) return cuda_error(e, "gen_proposals args");
  GenArgs* dg = static_cast<GenArgs*>(d);
  AnnArgs* da = reinterpret_cast<AnnArgs*>(dg + kk);
  if ((e = cudaMemcpyAsync(dg, ga.data(), kk * sizeof(GenArgs), cudaMemcpyHostToDevice, s)) ||
      (e = cudaMemcpyAsync(da, aa.data(), kk * sizeof(AnnArgs), cudaMemcpyHostToDevice, s)))
    return cuda_error(e, "gen_proposals args");
  k_gen2<true><<<kk, kThreads, 0, s>>>(GenArgs{}, dg);
  const unsigned blocks = (unsigned)((nmax + 255) / 256 < 64 ? (nmax + 255) / 256 : 64);
  k_annotate<true><<<dim3(blocks, kk), 256, 0, s>>>(AnnArgs{}, da);
  e = cudaGetLastError();
  cudaFreeAsync(d, s);
  if (e) return cuda_error(e, "gen_proposals");
  return GCMC_OK;
}

}  // namespace gcmcb
