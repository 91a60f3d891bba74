// gcmc_b200_strategy.hpp — drop-in gcmc::NeighborStrategy backed by the
// B200 C ABI (gcmc_b200.h). Header-only; include it next to the reference's
// headers (proj/include) and add one case to make_strategy
// (engine.hpp:189-202), see INTEGRATION.md.
//
// Semantics follow NeighborStrategy (strategy.hpp:27-50): delta_* are const
// and repeatable, commit_* update both the spatial index and the caller's
// ParticleStore (so Simulation keeps reading N and positions from it), errors
// are rethrown as the reference's exception types with its messages
// (std::out_of_range for a bad id, std::runtime_error for "cell C exceeds
// capacity K" / "not found in cell C").
#pragma once

#include <cstddef>
#include <cstdint>
#include <optional>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

#include "gcmc/strategy.hpp"
#include "gcmc_b200.h"

namespace gcmc_b200 {

inline void check(gcmc_status s) {
  if (s == GCMC_OK) return;
  const std::string msg = gcmc_last_error();
  switch (s) {
    case GCMC_INVALID_PID: throw std::out_of_range(msg);
    case GCMC_ARG: throw std::invalid_argument(msg);
    default: throw std::runtime_error(msg);
  }
}

class GpuNeighborStrategy final : public gcmc::NeighborStrategy {
 public:
  // kind: GCMC_ALL_PAIRS / GCMC_CELL_LIST / GCMC_MICROCELL; capacity 0 = the
  // reference default (cell_grid.hpp:36-38, microcell_grid.hpp:149).
  GpuNeighborStrategy(gcmc::ParticleStore& store, const gcmc::SimBox& box,
                      const gcmc::LjParams& lj, int kind, int capacity = 0, int device = 0)
      : store_(store), kind_(kind) {
    gcmc_params p{};
    p.box_length = box.side_length;
    p.epsilon = lj.epsilon;
    p.sigma = lj.sigma;
    p.r_cut = lj.r_cut;
    p.temperature = 1.0;
    p.lambda = 1.0;
    p.sampling_interval = 1;
    p.strategy = kind;
    if (kind == GCMC_CELL_LIST) p.cell_capacity = capacity;
    if (kind == GCMC_MICROCELL) p.microcell_capacity = capacity;
    check(gcmc_create(&p, device, &h_));
    build();  // the reference ctors build immediately
  }
  ~GpuNeighborStrategy() override { gcmc_destroy(h_); }
  GpuNeighborStrategy(const GpuNeighborStrategy&) = delete;
  GpuNeighborStrategy& operator=(const GpuNeighborStrategy&) = delete;

  std::string_view name() const override {
    return kind_ == GCMC_MICROCELL ? "microcell" : (kind_ == GCMC_CELL_LIST ? "cell_list" : "all_pairs");
  }

  // Re-uploads the store (positions may have been edited behind our back).
  void build() override {
    const auto pos = store_.positions();
    std::vector<double> xyz(3 * pos.size());
    for (std::size_t i = 0; i < pos.size(); ++i) {
      xyz[3 * i] = pos[i].x;
      xyz[3 * i + 1] = pos[i].y;
      xyz[3 * i + 2] = pos[i].z;
    }
    check(gcmc_upload_positions(h_, xyz.data(), pos.size()));
  }

  gcmc::PairInteraction delta_displace(std::size_t pid, const gcmc::Vec3& p) const override {
    const double q[3] = {p.x, p.y, p.z};
    gcmc::PairInteraction r;
    check(gcmc_delta_displace(h_, pid, q, &r.u, &r.w));
    return r;
  }
  gcmc::PairInteraction delta_insert(const gcmc::Vec3& p) const override {
    const double q[3] = {p.x, p.y, p.z};
    gcmc::PairInteraction r;
    check(gcmc_delta_insert(h_, q, &r.u, &r.w));
    return r;
  }
  gcmc::PairInteraction delta_delete(std::size_t pid) const override {
    gcmc::PairInteraction r;
    check(gcmc_delta_delete(h_, pid, &r.u, &r.w));
    return r;
  }

  void commit_displace(std::size_t pid, const gcmc::Vec3& p) override {
    const double q[3] = {p.x, p.y, p.z};
    check(gcmc_commit_displace(h_, pid, q));
    store_.set(pid, p);
  }
  std::size_t commit_insert(const gcmc::Vec3& p) override {
    const double q[3] = {p.x, p.y, p.z};
    uint64_t pid = 0;
    const gcmc_status s = gcmc_commit_insert(h_, q, &pid);
    // On a cell overflow the device store has already appended the particle,
    // as the reference's does before insert_id throws (microcell_grid.hpp:253-256).
    if (s == GCMC_OK || s == GCMC_CELL_OVERFLOW) store_.append(p);
    check(s);
    return static_cast<std::size_t>(pid);
  }
  void commit_delete(std::size_t pid) override {
    check(gcmc_commit_delete(h_, pid));
    store_.remove_swap_last(pid);
  }

  std::optional<std::string> rebuild_check() const override {
    char msg[512];
    int32_t clean = 0;
    check(gcmc_rebuild_check(h_, msg, sizeof msg, &clean));
    if (clean) return std::nullopt;
    return std::string(msg);
  }
  int peak_cell_occupancy() const override {
    int32_t p = 0;
    check(gcmc_peak_occupancy(h_, &p));
    return p;
  }

  gcmc_dev* handle() const { return h_; }

 private:
  gcmc::ParticleStore& store_;
  int kind_;
  gcmc_dev* h_ = nullptr;
};

}  // namespace gcmc_b200
