// Latency microbenchmarks for the engine's critical path (single thread).
// Build and run (writes the JSON line bench.py's latency floor reads):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -std=c++17 \
//        -I paper_1408_3764_b200/csrc -I include -o /tmp/ubench tools/ubench/ubench.cu
//   /tmp/ubench --json 2> profiles/ubench.json
#include <cstdio>
#include <cstring>
#include <cstdint>
#include <cuda_runtime.h>
#include "common.cuh"
using namespace gcmcb;

__global__ void k_lat(const int* chase, int steps, const double4* recs, Box b, unsigned long long* out, double* sink) {
  if (threadIdx.x) return;
  // L2 (.cg) pointer chase
  int p = 0;
  unsigned long long t0 = clock64();
  for (int i = 0; i < steps; ++i) p = __ldcg(chase + p);
  unsigned long long t1 = clock64();
  out[0] = (t1 - t0) / steps;
  // default-cached chase (L1)
  p = 0;
  t0 = clock64();
  for (int i = 0; i < steps; ++i) p = chase[p];
  t1 = clock64();
  out[1] = (t1 - t0) / steps;
  // dependent DADD chain
  double x = sink[0];
  t0 = clock64();
  for (int i = 0; i < steps; ++i) x = __dadd_rn(x, 1.0);
  t1 = clock64();
  out[2] = (t1 - t0) / steps;
  // rint chain
  t0 = clock64();
  for (int i = 0; i < steps; ++i) x = rint(__dadd_rn(x, 0.3));
  t1 = clock64();
  out[3] = (t1 - t0) / steps;
  // div chain
  double y = 1.7;
  t0 = clock64();
  for (int i = 0; i < steps; ++i) y = __ddiv_rn(1.3, __dadd_rn(y, 1.0));
  t1 = clock64();
  out[4] = (t1 - t0) / steps;
  // full pair term (min image + LJ) chained through r2 perturbation
  double acc = 0.0;
  double px = 1.0, py = 2.0, pz = 3.0;
  t0 = clock64();
  for (int i = 0; i < steps; ++i) {
    const double4 r = make_double4(1.5 + acc * 1e-30, 2.2, 3.1, 0.0);
    const double r2 = min_image_dist2(px, py, pz, r.x, r.y, r.z, b);
    double u, w;
    lj_pair_clamped(r2, b, u, w);
    acc = __dadd_rn(acc, u);
  }
  t1 = clock64();
  out[5] = (t1 - t0) / steps;
  // exp chain
  t0 = clock64();
  for (int i = 0; i < steps; ++i) y = exp(-__dmul_rn(y, 1e-3));
  t1 = clock64();
  out[6] = (t1 - t0) / steps;
  // 8 independent .cg loads then use (MLP): time per batch
  t0 = clock64();
  int q = 0;
  for (int i = 0; i < steps / 8; ++i) {
    int v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = __ldcg(chase + ((q + k * 977) & 65535));
    int s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += v[k];
    q = s & 65535;
  }
  t1 = clock64();
  out[7] = (t1 - t0) / (steps / 8);
  // double4 ld_cg chase via pid field
  long long pid = 0;
  t0 = clock64();
  for (int i = 0; i < steps; ++i) {
    const double4 r = ld_cg(recs + pid);
    pid = bits_pid(r.w);
  }
  t1 = clock64();
  out[8] = (t1 - t0) / steps;
  sink[0] = x + y + acc + p + q + pid;
}

// Dependent warp reduction step: one shuffle + one DADD.
__global__ void k_shfl(int steps, double seed, unsigned long long* out, double* sink) {
  double x = seed + threadIdx.x;
  const unsigned long long t0 = clock64();
  for (int i = 0; i < steps; ++i) x = __dadd_rn(x, __shfl_xor_sync(0xffffffffu, x, 1 + (i & 15)));
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0) {
    out[0] = (t1 - t0) / steps;
    sink[0] = x;
  }
}

__device__ __forceinline__ unsigned long long ldr(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void str(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// Two CTAs on different SMs bounce a counter through global memory:
// per iteration = two one-way store->load visibility latencies.
__global__ void k_pingpong(unsigned long long* flag, unsigned long long* ack, int iters,
                           unsigned long long* out) {
  if (threadIdx.x) return;
  unsigned smid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  if (blockIdx.x == 0) {
    const unsigned long long t0 = clock64();
    for (int i = 1; i <= iters; ++i) {
      str(flag, i);
      while (ldr(ack) != (unsigned long long)i) {}
    }
    out[0] = (clock64() - t0) / iters;
    out[2] = smid;
  } else {
    for (int i = 1; i <= iters; ++i) {
      while (ldr(flag) != (unsigned long long)i) {}
      str(ack, i);
    }
    out[3] = smid;
  }
}
__global__ void k_relaxed_chase(const unsigned long long* chase, int steps, unsigned long long* out) {
  if (threadIdx.x) return;
  unsigned long long p = 0;
  const unsigned long long t0 = clock64();
  for (int i = 0; i < steps; ++i) p = ldr(chase + p);
  out[1] = (clock64() - t0) / steps + (p == 12345678 ? 1 : 0);
}

int main(int argc, char** argv) {
  const bool json = argc > 1 && !strcmp(argv[1], "--json");
  if (json) freopen("/dev/null", "w", stdout);
  const int N = 1 << 16;
  int* h = new int[N];
  // random cyclic permutation
  unsigned s = 12345;
  int* perm = new int[N];
  for (int i = 0; i < N; ++i) perm[i] = i;
  for (int i = N - 1; i > 0; --i) { s = s * 1103515245u + 12345u; int j = s % (i + 1); int t = perm[i]; perm[i] = perm[j]; perm[j] = t; }
  for (int i = 0; i < N; ++i) h[perm[i]] = perm[(i + 1) % N];
  double4* hr = new double4[N];
  for (int i = 0; i < N; ++i) hr[perm[i]] = make_double4(0, 0, 0, [&]{ long long v = perm[(i + 1) % N]; double dd; memcpy(&dd, &v, 8); return dd; }());
  int* d; double4* dr; unsigned long long* o; double* sink;
  cudaMalloc(&d, N * 4); cudaMalloc(&dr, N * 32); cudaMalloc(&o, 16 * 8); cudaMalloc(&sink, 8);
  cudaMemcpy(d, h, N * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dr, hr, N * 32, cudaMemcpyHostToDevice);
  cudaMemset(sink, 0, 8);
  Box b{};
  b.l = 36.57; b.inv_l = 1.0 / b.l; b.eps = 1; b.sigma = 1; b.sigma2 = 1; b.rc = 2.5; b.rc2 = 6.25; b.four_eps = 4; b.tf_eps = 24;
  for (int rep = 0; rep < 2; ++rep) k_lat<<<1, 32>>>(d, 4096, dr, b, o, sink);
  unsigned long long ho[16];
  cudaMemcpy(ho, o, 16 * 8, cudaMemcpyDeviceToHost);
  const char* names[] = {"ld.cg chase", "ld chase", "dadd", "rint+dadd", "ddiv+dadd", "pair_term", "exp", "8x ld.cg batch", "double4 ld.cg chase"};
  for (int i = 0; i < 9; ++i) printf("%-22s %6llu cycles\n", names[i], ho[i]);
  unsigned long long pp_max = 0, chase_relaxed = 0, shfl = 0;
  {
    unsigned long long *flag, *ack, *po, *ch;
    cudaMalloc(&flag, 4096); cudaMalloc(&ack, 4096); cudaMalloc(&po, 64); cudaMalloc(&ch, N * 8);
    unsigned long long* hc = new unsigned long long[N];
    for (int i = 0; i < N; ++i) hc[perm[i]] = perm[(i + 1) % N];
    cudaMemcpy(ch, hc, N * 8, cudaMemcpyHostToDevice);
    for (int grid : {2, 74, 148}) {
      cudaMemset(flag, 0, 4096); cudaMemset(ack, 0, 4096);
      k_pingpong<<<grid, 32>>>(flag, ack + 64, 2000, po);  // (blocks >1 idle)
      cudaDeviceSynchronize();
      unsigned long long hp[4];
      cudaMemcpy(hp, po, 32, cudaMemcpyDeviceToHost);
      printf("pingpong grid %3d (sm %llu <-> sm %llu): %llu cycles per round trip\n", grid, hp[2], hp[3], hp[0]);
      if (hp[0] > pp_max) pp_max = hp[0];
    }
    k_relaxed_chase<<<1, 32>>>(ch, 4096, po);
    cudaDeviceSynchronize();
    unsigned long long hp[2];
    cudaMemcpy(hp, po, 16, cudaMemcpyDeviceToHost);
    printf("ld.relaxed.gpu chase: %llu cycles\n", hp[1]);
    chase_relaxed = hp[1];
  }
  {
    unsigned long long* so;
    double* ss;
    cudaMalloc(&so, 8);
    cudaMalloc(&ss, 8);
    k_shfl<<<1, 32>>>(4096, 1.0, so, ss);
    cudaMemcpy(&shfl, so, 8, cudaMemcpyDeviceToHost);
    printf("shfl+dadd chain: %llu cycles\n", shfl);
  }
  if (json) {
    int khz = 0;
    cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
    cudaDeviceProp prop;
    cudaGetDeviceProperties(&prop, 0);
    fprintf(stderr,
            "{\"source\": \"tools/ubench/ubench.cu on %s\", \"sm_ghz\": %.4f, \"l2_chase_cycles\": %llu, "
            "\"l2_relaxed_chase_cycles\": %llu, \"pingpong_cycles\": %llu, \"pair_term_cycles\": %llu, "
            "\"shfl_dadd_cycles\": %llu, \"double4_chase_cycles\": %llu}\n",
            prop.name, khz / 1e6, ho[0], chase_relaxed, pp_max, ho[5], shfl, ho[8]);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
