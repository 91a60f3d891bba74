// Trial-move ΔE for explicit proposals (the per-move plugin API):
// NeighborStrategy::delta_displace / delta_insert / delta_delete
// (strategy.hpp:36-38). One 512-thread CTA per proposal (the same
// cta_window_sums the engine uses), all proposals against the same state.
#include "cta_window.cuh"
#include "internal.h"

namespace gcmcb {

namespace {

constexpr int kCtaThreads = 512;

__global__ void __launch_bounds__(kCtaThreads)
    k_delta_batch(Grid g, Box b, const double4* __restrict__ pos, uint64_t n, uint64_t count,
                  const int32_t* __restrict__ kinds, const uint64_t* __restrict__ pids,
                  const double* __restrict__ xyz, double* du, double* dw) {
  __shared__ GroupReduce<kCtaThreads> red;
  __shared__ MoveCtx ctx;
  const uint64_t q = blockIdx.x;
  if (q >= count) return;
  const int kind = kinds[q];
  if (threadIdx.x < 32) {
    if (threadIdx.x == 0) {
      ctx.exclude = (long long)n;
      ctx.np = 1;
      ctx.x[0] = xyz[3 * q];
      ctx.y[0] = xyz[3 * q + 1];
      ctx.z[0] = xyz[3 * q + 2];
      if (kind == 0 || kind == 2) {
        const uint64_t pid = pids[q];
        const double4 o = ld_cg(pos + pid);
        ctx.exclude = (long long)pid;
        const int e = kind == 0 ? 1 : 0;
        ctx.np = kind == 0 ? 2 : 1;
        ctx.x[e] = o.x;
        ctx.y[e] = o.y;
        ctx.z[e] = o.z;
      }
    }
    __syncwarp();
    setup_runs(g, b, ctx);
  }
  __syncthreads();
  double du_s, dw_s;
  group_delta<kCtaThreads>(g, b, pos, n, ctx, red, 1, du_s, dw_s);
  if (threadIdx.x == 0) {
    du[q] = kind == 2 ? -du_s : du_s;
    dw[q] = kind == 2 ? -dw_s : dw_s;
  }
}

}  // namespace

gcmc_status delta_batch(Chain& c, uint64_t count, const int32_t* kinds_d, const uint64_t* pids_d,
                        const double* xyz_d, double* du_d, double* dw_d) {
  if (!count) return GCMC_OK;
  k_delta_batch<<<(unsigned)count, kCtaThreads, 0, c.stream>>>(c.grid, c.box, c.pos,
                                                              c.st_host->n, count, kinds_d,
                                                              pids_d, xyz_d, du_d, dw_d);
  cudaError_t e = cudaGetLastError();
  if (e) return cuda_error(e, "delta");
  return GCMC_OK;
}

}  // namespace gcmcb
