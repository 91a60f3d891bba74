// Trial-move ΔE for explicit proposals (the per-move plugin API):
// NeighborStrategy::delta_displace / delta_insert / delta_delete
// (strategy.hpp:36-38). One 256-thread CTA per proposal running the same
// group evaluator as the engine (slot.cuh), all proposals against the same
// state.
#include "internal.h"
#include "slot.cuh"

namespace gcmcb {

namespace {

constexpr int kT = 256;

__global__ void __launch_bounds__(kT)
    k_delta_batch(Mirror m, Box b, const double4* __restrict__ pos,
                  uint64_t n, bool all_pairs, uint64_t count,
                  const int32_t* __restrict__ kinds, const uint64_t* __restrict__ pids,
                  const double* __restrict__ xyz, double* du, double* dw) {
  __shared__ WinWs<kT> ws;
  const uint64_t q = blockIdx.x;
  if (q >= count) return;
  const int kind = kinds[q];
  const int lane = threadIdx.x & 31;
  long long exclude = -1;
  if (threadIdx.x < 32) {
    if (lane == 0) {
      ws.excl = -1;
      ws.nwin = 1;
      ws.sign1 = -1;
      ws.cx[0] = xyz[3 * q];
      ws.cy[0] = xyz[3 * q + 1];
      ws.cz[0] = xyz[3 * q + 2];
      if (kind != 1) {
        const uint64_t pid = pids[q];
        const double4 o = ld_cg(pos + pid);
        ws.excl = bslot_in(o);
        const int e = kind == 0 ? 1 : 0;
        ws.nwin = kind == 0 ? 2 : 1;
        ws.cx[e] = o.x;
        ws.cy[e] = o.y;
        ws.cz[e] = o.z;
      }
    }
    __syncwarp();
    if (!all_pairs) win_setup_warp<kT>(m, b, ws, nullptr, lane);
  }
  if (kind != 1) exclude = (long long)pids[q];
  __syncthreads();
  double su, sw;
  if (all_pairs)
    allpairs_sums<kT>(b, pos, n, ws, exclude, threadIdx.x, su, sw);
  else
    win_sums<kT>(m, b, ws, threadIdx.x, su, sw);
  group_reduce<kT>(ws, su, sw, 1, threadIdx.x);
  if (threadIdx.x == 0) {
    du[q] = kind == 2 ? -su : su;
    dw[q] = kind == 2 ? -sw : sw;
  }
}

}  // namespace

gcmc_status delta_batch(Chain& c, uint64_t count, const int32_t* kinds_d, const uint64_t* pids_d,
                        const double* xyz_d, double* du_d, double* dw_d) {
  if (!count) return GCMC_OK;
  k_delta_batch<<<(unsigned)count, kT, 0, c.stream>>>(
      c.mirror, c.box, c.pos, c.st_host->n, c.grid.kind == GCMC_ALL_PAIRS, count, kinds_d,
      pids_d, xyz_d, du_d, dw_d);
  cudaError_t e = cudaGetLastError();
  if (e) return cuda_error(e, "delta");
  return GCMC_OK;
}

}  // namespace gcmcb
