// TEST INFRASTRUCTURE ONLY — drop-in check of include/gcmc_b200_strategy.hpp.
//
// Built here against the UNMODIFIED reference headers (oracle/Makefile,
// target `shim`) into oracle/_ref/shim_check, linked to the product's
// libgcmc_b200.so; run on the GPU box by tests/test_gpu_parity.py. The
// reference's own strategy (the oracle) and the B200 strategy index two
// copies of the same ParticleStore and receive the same proposals and
// commits, in the spirit of validate::cross_strategy_equivalence
// (validate.hpp:44-93) and grid_rebin_consistency (:108-148):
//   * every delta_* within 1e-10 relative (T/test_grids.cpp:255-259),
//   * after every commit: identical store, byte-identical occupancy/slots,
//     clean rebuild_check, identical peak occupancy.
//
//   shim_check <microcell|cell_list|all_pairs> <n0> <proposals> <seed>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "gcmc/cell_grid.hpp"
#include "gcmc/init_config.hpp"
#include "gcmc/microcell_grid.hpp"
#include "gcmc/rng.hpp"
#include "gcmc/strategy.hpp"
#include "gcmc_b200_strategy.hpp"

namespace {

double rel(double a, double b) { return std::fabs(a - b) / std::max(1.0, std::fabs(b)); }

}  // namespace

int main(int argc, char** argv) {
  const std::string kind = argc > 1 ? argv[1] : "microcell";
  const std::size_t n0 = argc > 2 ? std::strtoull(argv[2], nullptr, 10) : 4096;
  const int nprop = argc > 3 ? std::atoi(argv[3]) : 3000;
  const std::uint64_t seed = argc > 4 ? std::strtoull(argv[4], nullptr, 10) : 5;
  const double l = std::cbrt((double)n0 / 0.67);
  gcmc::SimBox box(l);
  gcmc::LjParams lj(1.0, 1.0, 2.5);
  gcmc::RngStream init_rng(seed);
  gcmc::ParticleStore s_ref = gcmc::random_initial_configuration(n0, box, 0.85, init_rng);
  gcmc::ParticleStore s_gpu = s_ref;

  std::unique_ptr<gcmc::NeighborStrategy> ref;
  int k = GCMC_MICROCELL;
  if (kind == "microcell") {
    ref = std::make_unique<gcmc::MicrocellGridStrategy>(s_ref, box, lj, 5);
  } else if (kind == "cell_list") {
    ref = std::make_unique<gcmc::CellGridStrategy>(s_ref, box, lj, 0);
    k = GCMC_CELL_LIST;
  } else {
    ref = std::make_unique<gcmc::AllPairsStrategy>(s_ref, box, lj);
    k = GCMC_ALL_PAIRS;
  }
  gcmc_b200::GpuNeighborStrategy gpu(s_gpu, box, lj, k, kind == "microcell" ? 5 : 0);

  gcmc::RngStream rng(seed + 1000);
  double worst = 0.0;
  int commits = 0, fails = 0;
  auto grids_equal = [&]() -> bool {
    if (k == GCMC_ALL_PAIRS) return true;
    int32_t dims = 0, cap = 0;
    uint64_t nc = 0;
    gcmc_b200::check(gcmc_grid_info(gpu.handle(), &dims, &cap, &nc));
    std::vector<int32_t> occ(nc), slots(nc * (uint64_t)cap);
    gcmc_b200::check(gcmc_download_grid(gpu.handle(), occ.data(), slots.data()));
    std::span<const std::int32_t> ro, rs;
    if (k == GCMC_MICROCELL) {
      auto* m = static_cast<gcmc::MicrocellGridStrategy*>(ref.get());
      ro = m->occupancy_view();
      rs = m->slots_view();
    } else {
      auto* c = static_cast<gcmc::CellGridStrategy*>(ref.get());
      ro = c->occupancy_view();
      rs = c->slots_view();
    }
    return ro.size() == occ.size() && rs.size() == slots.size() &&
           std::memcmp(ro.data(), occ.data(), occ.size() * 4) == 0 &&
           std::memcmp(rs.data(), slots.data(), slots.size() * 4) == 0;
  };
  if (!grids_equal()) {
    std::printf("FAIL build: grids differ\n");
    return 1;
  }
  for (int t = 0; t < nprop; ++t) {
    const int mk = (int)rng.index_from(rng.uniform(), 3);
    const gcmc::Vec3 p{rng.uniform() * l, rng.uniform() * l, rng.uniform() * l};
    const std::size_t n = s_ref.size();
    const std::size_t pid = n ? rng.index_from(rng.uniform(), n) : 0;
    gcmc::PairInteraction a, b;
    if (mk == 0 && n) {
      a = ref->delta_displace(pid, p);
      b = gpu.delta_displace(pid, p);
    } else if (mk == 2 && n) {
      a = ref->delta_delete(pid);
      b = gpu.delta_delete(pid);
    } else {
      a = ref->delta_insert(p);
      b = gpu.delta_insert(p);
    }
    if (a.u < 1e29) worst = std::max(worst, std::max(rel(b.u, a.u), rel(b.w, a.w)));
    // commit roughly one proposal in four that is not an overlap
    if (a.u < 50.0 && rng.uniform() < 0.25) {
      if (mk == 0 && n) {
        ref->commit_displace(pid, p);
        gpu.commit_displace(pid, p);
      } else if (mk == 2 && n) {
        ref->commit_delete(pid);
        gpu.commit_delete(pid);
      } else {
        const std::size_t ia = ref->commit_insert(p), ib = gpu.commit_insert(p);
        if (ia != ib) ++fails;
      }
      ++commits;
      if (commits % 50 == 0 || t == nprop - 1) {
        if (!grids_equal()) ++fails;
        if (gpu.rebuild_check()) ++fails;
        if (ref->peak_cell_occupancy() != gpu.peak_cell_occupancy()) ++fails;
      }
    }
  }
  // the GPU strategy kept the caller's store in step
  bool same = s_ref.size() == s_gpu.size();
  for (std::size_t i = 0; same && i < s_ref.size(); ++i)
    same = s_ref[i].x == s_gpu[i].x && s_ref[i].y == s_gpu[i].y && s_ref[i].z == s_gpu[i].z;
  std::vector<double> dev(3 * s_ref.size() + 3);
  uint64_t cnt = 0;
  gcmc_b200::check(gcmc_download_positions(gpu.handle(), dev.data(), dev.size(), &cnt));
  for (std::size_t i = 0; same && i < cnt; ++i)
    same = dev[3 * i] == s_ref[i].x && dev[3 * i + 1] == s_ref[i].y && dev[3 * i + 2] == s_ref[i].z;
  // error path: the reference's exception types and messages
  bool err_ok = false;
  try {
    gpu.delta_delete(s_gpu.size() + 5);
  } catch (const std::out_of_range& e) {
    try {
      ref->delta_delete(s_ref.size() + 5);
    } catch (const std::out_of_range& f) {
      err_ok = std::string(e.what()) == f.what();
    }
  }
  std::printf("%s n0=%zu proposals=%d commits=%d worst_rel=%.3e store_equal=%d errors_equal=%d fails=%d\n",
              kind.c_str(), n0, nprop, commits, worst, (int)same, (int)err_ok, fails);
  return (worst <= 1e-10 && same && err_ok && fails == 0) ? 0 : 1;
}
