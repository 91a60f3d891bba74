// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// A thin C ABI over the UNMODIFIED reference headers
// (/root/reference/proj/include/gcmc/*.hpp, included by path at compile
// time, never copied). `oracle/Makefile` compiles this file with the
// reference's own Release flags (g++ -std=c++20 -O3 -DNDEBUG, no -march,
// matching proj/CMakeLists.txt:6-8) into oracle/_ref/libgcmc_ref.so.
//
// Used by tests/ (parity checker), tests/golden/make_golden.py (fixture
// generator) and bench.py's reference arm / cpu_baseline leg (timing of the
// reference's own Simulation::step loop, proj/include/gcmc/bench.hpp:95).
#include <chrono>
#include <cstdint>
#include <cstring>
#include <filesystem>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "gcmc/bench.hpp"
#include "gcmc/checkpoint.hpp"
#include "gcmc/driver.hpp"
#include "gcmc/engine.hpp"
#include "gcmc/validate.hpp"

using namespace gcmc;

extern "C" {

// Mirrors gcmc::RunConfig (proj/include/gcmc/config.hpp:42-64).
struct ref_config {
  double temperature, chemical_potential, lambda, epsilon, sigma, r_cut;
  double box_length;
  uint64_t initial_particles;
  double density;
  double displace_percent;
  uint64_t steps, seed, checkpoint_interval;
  int32_t strategy;  // 0 all_pairs, 1 cell_list, 2 microcell
  int32_t tail_corrections;
  int32_t cell_capacity, microcell_capacity;
  uint64_t equilibration_steps, sampling_interval;
  double max_displacement;
};

// Mirrors gcmc::MoveOutcome (engine.hpp:104-110) plus the post-move N.
struct ref_outcome {
  int32_t kind;  // 0 displace, 1 insert, 2 remove
  int32_t accepted;
  double delta_u, delta_w, acceptance_prob;
  uint64_t n_after;
};

// SystemState + RunStatistics + step/draws (engine.hpp:112-140).
struct ref_state {
  uint64_t step, n;
  double energy, virial;
  uint64_t attempted[3], accepted[3];
  uint64_t samples;
  double sum_u, sum_p, sum_n, sum_n2;
  uint64_t draws;
  int32_t peak_occupancy, pad;
  double pressure, reported_energy;
};
}

namespace {

thread_local std::string g_err;

int fail(const std::exception& e, int code) {
  g_err = e.what();
  return code;
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const AuditFailure& e) {
    return fail(e, 5);
  } catch (const std::out_of_range& e) {
    return fail(e, 1);
  } catch (const std::domain_error& e) {
    return fail(e, 3);
  } catch (const std::invalid_argument& e) {
    return fail(e, 4);
  } catch (const std::runtime_error& e) {
    return fail(e, 2);
  } catch (const std::exception& e) {
    return fail(e, 9);
  }
}

RunConfig to_cfg(const ref_config& c) {
  RunConfig r;
  r.temperature = c.temperature;
  r.chemical_potential = c.chemical_potential;
  r.lambda = c.lambda;
  r.epsilon = c.epsilon;
  r.sigma = c.sigma;
  r.r_cut = c.r_cut;
  r.box_length = c.box_length;
  r.initial_particles = c.initial_particles;
  r.density = c.density;
  r.displace_percent = c.displace_percent;
  r.steps = c.steps;
  r.seed = c.seed;
  r.checkpoint_interval = c.checkpoint_interval;
  r.strategy = static_cast<Strategy>(c.strategy);
  r.tail_corrections = c.tail_corrections != 0;
  r.cell_capacity = c.cell_capacity;
  r.microcell_capacity = c.microcell_capacity;
  r.equilibration_steps = c.equilibration_steps;
  r.sampling_interval = c.sampling_interval;
  r.max_displacement = c.max_displacement;
  return r;
}

void from_cfg(const RunConfig& r, ref_config* c) {
  c->temperature = r.temperature;
  c->chemical_potential = r.chemical_potential;
  c->lambda = r.lambda;
  c->epsilon = r.epsilon;
  c->sigma = r.sigma;
  c->r_cut = r.r_cut;
  c->box_length = r.box_length;
  c->initial_particles = r.initial_particles;
  c->density = r.density;
  c->displace_percent = r.displace_percent;
  c->steps = r.steps;
  c->seed = r.seed;
  c->checkpoint_interval = r.checkpoint_interval;
  c->strategy = static_cast<int32_t>(r.strategy);
  c->tail_corrections = r.tail_corrections ? 1 : 0;
  c->cell_capacity = r.cell_capacity;
  c->microcell_capacity = r.microcell_capacity;
  c->equilibration_steps = r.equilibration_steps;
  c->sampling_interval = r.sampling_interval;
  c->max_displacement = r.max_displacement;
}

std::vector<Vec3> to_vec(const double* xyz, uint64_t n) {
  std::vector<Vec3> v(n);
  for (uint64_t i = 0; i < n; ++i) v[i] = {xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]};
  return v;
}

void copy_str(const std::string& s, char* buf, uint64_t cap) {
  if (!buf || cap == 0) return;
  const uint64_t n = s.size() < cap - 1 ? s.size() : cap - 1;
  std::memcpy(buf, s.data(), n);
  buf[n] = 0;
}

// A standalone strategy over its own store (validate.hpp:51-53 pattern).
struct StratBox {
  ParticleStore store;
  SimBox box{1.0};
  LjParams lj;
  std::unique_ptr<NeighborStrategy> s;
  int kind = 0;
};

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---------------------------------------------------------------- config I/O
int ref_parse_config(const char* text, ref_config* out) {
  return guarded([&] { from_cfg(parse_config_text(text), out); });
}

int ref_serialize_config(const ref_config* c, char* buf, uint64_t cap) {
  return guarded([&] { copy_str(to_cfg(*c).serialize(), buf, cap); });
}

// ---------------------------------------------------------------- primitives
int ref_mt_uniforms(uint64_t seed, uint64_t skip, uint64_t n, double* out) {
  return guarded([&] {
    RngStream r(seed);
    for (uint64_t i = 0; i < skip; ++i) r.uniform();
    for (uint64_t i = 0; i < n; ++i) out[i] = r.uniform();
  });
}

int ref_rng_hex(uint64_t seed, uint64_t skip, char* buf, uint64_t cap) {
  return guarded([&] {
    RngStream r(seed);
    for (uint64_t i = 0; i < skip; ++i) r.uniform();
    copy_str(r.serialize_hex(), buf, cap);
  });
}

uint64_t ref_index_from(double u, uint64_t n) { return RngStream::index_from(u, n); }

int ref_wrap_position(const double* p, double l, double* out) {
  return guarded([&] {
    const Vec3 w = wrap_position({p[0], p[1], p[2]}, SimBox(l));
    out[0] = w.x;
    out[1] = w.y;
    out[2] = w.z;
  });
}

double ref_min_image_dist2(const double* a, const double* b, double l) {
  return min_image_dist2({a[0], a[1], a[2]}, {b[0], b[1], b[2]}, SimBox(l));
}

int ref_lj_pair(double r2, double eps, double sigma, double rc, int clamped, double* u, double* w) {
  return guarded([&] {
    const LjParams lj(eps, sigma, rc);
    const auto p = clamped ? lj_pair_clamped(r2, lj) : lj_pair(r2, lj);
    *u = p.u;
    *w = p.w;
  });
}

void ref_tail_corrections(double rho, double eps, double sigma, double rc, double* u, double* p) {
  const auto t = tail_corrections(rho, eps, sigma, rc);
  *u = t.u_per_particle;
  *p = t.pressure;
}

double ref_displacement_acceptance(double du, double beta) {
  return displacement_acceptance(du, beta);
}
double ref_insertion_acceptance(double du, uint64_t n, double v, double beta, double mu,
                                double lambda) {
  return insertion_acceptance(du, n, v, beta, mu, lambda);
}
double ref_deletion_acceptance(double du, uint64_t n, double v, double beta, double mu,
                               double lambda) {
  return deletion_acceptance(du, n, v, beta, mu, lambda);
}

void ref_compute_cell_dims(double l, double rc, int32_t* dims, double* size) {
  const auto d = compute_cell_dims(l, rc);
  *dims = d.cells_per_dim;
  *size = d.cell_size;
}
int32_t ref_default_cell_capacity(double rc, double sigma) { return default_cell_capacity(rc, sigma); }
void ref_microcell_dims(double l, double sigma, int32_t* dims, double* last_w) {
  const auto d = microcell_dims(l, sigma);
  *dims = d.dims;
  *last_w = d.last_cell_width;
}
int32_t ref_microcell_extent(double rc, double sigma) { return microcell_extent(rc, sigma); }
void ref_microcell_axis_window(int32_t center, double rc, double sigma, int32_t dims, double last_w,
                               int32_t* lo, int32_t* count) {
  const auto w = microcell_axis_window(center, rc, sigma, dims, last_w);
  *lo = w.lo;
  *count = w.count;
}
void ref_microcell_axis_arc(double x, double rc, double sigma, double l, int32_t dims,
                            int32_t* first, int32_t* count) {
  const auto a = microcell_axis_arc(x, rc, sigma, l, dims);
  *first = a.first;
  *count = a.count;
}
uint64_t ref_cube_cells(int32_t cx, int32_t cy, int32_t cz, int32_t h, int32_t dims, int32_t* out,
                        uint64_t cap) {
  const auto v = detail::cube_cells(cx, cy, cz, h, dims);
  for (uint64_t i = 0; i < v.size() && i < cap; ++i) out[i] = v[i];
  return v.size();
}

int ref_total_energy(const double* xyz, uint64_t n, double l, double eps, double sigma, double rc,
                     double* u, double* w) {
  return guarded([&] {
    const ParticleStore store(to_vec(xyz, n));
    const auto e = total_energy(store, SimBox(l), LjParams(eps, sigma, rc));
    *u = e.u;
    *w = e.w;
  });
}

// Random sequential insertion (init_config.hpp:19-64) from a fresh seed.
// Writes positions and the RNG state (hex) left behind for the MC stream.
int ref_random_initial_configuration(uint64_t n, double l, double min_sep, uint64_t seed,
                                     double* out_xyz, char* rng_hex, uint64_t hex_cap) {
  return guarded([&] {
    RngStream r(seed);
    const auto store = random_initial_configuration(n, SimBox(l), min_sep, r);
    for (uint64_t i = 0; i < store.size(); ++i) {
      out_xyz[3 * i] = store[i].x;
      out_xyz[3 * i + 1] = store[i].y;
      out_xyz[3 * i + 2] = store[i].z;
    }
    copy_str(r.serialize_hex(), rng_hex, hex_cap);
  });
}

// ---------------------------------------------------------------- strategies
int ref_strat_create(int32_t kind, const double* xyz, uint64_t n, double l, double eps, double sigma,
                     double rc, int32_t capacity, void** out) {
  return guarded([&] {
    auto b = std::make_unique<StratBox>();
    b->store = ParticleStore(to_vec(xyz, n));
    b->box = SimBox(l);
    b->lj = LjParams(eps, sigma, rc);
    b->kind = kind;
    if (kind == 0)
      b->s = std::make_unique<AllPairsStrategy>(b->store, b->box, b->lj);
    else if (kind == 1)
      b->s = std::make_unique<CellGridStrategy>(b->store, b->box, b->lj, capacity);
    else
      b->s = std::make_unique<MicrocellGridStrategy>(b->store, b->box, b->lj, capacity);
    *out = b.release();
  });
}

void ref_strat_destroy(void* h) { delete static_cast<StratBox*>(h); }

int ref_strat_delta_displace(void* h, uint64_t pid, const double* p, double* du, double* dw) {
  return guarded([&] {
    const auto d = static_cast<StratBox*>(h)->s->delta_displace(pid, {p[0], p[1], p[2]});
    *du = d.u;
    *dw = d.w;
  });
}
int ref_strat_delta_insert(void* h, const double* p, double* du, double* dw) {
  return guarded([&] {
    const auto d = static_cast<StratBox*>(h)->s->delta_insert({p[0], p[1], p[2]});
    *du = d.u;
    *dw = d.w;
  });
}
int ref_strat_delta_delete(void* h, uint64_t pid, double* du, double* dw) {
  return guarded([&] {
    const auto d = static_cast<StratBox*>(h)->s->delta_delete(pid);
    *du = d.u;
    *dw = d.w;
  });
}
int ref_strat_commit_displace(void* h, uint64_t pid, const double* p) {
  return guarded([&] { static_cast<StratBox*>(h)->s->commit_displace(pid, {p[0], p[1], p[2]}); });
}
int ref_strat_commit_insert(void* h, const double* p, uint64_t* pid) {
  return guarded([&] { *pid = static_cast<StratBox*>(h)->s->commit_insert({p[0], p[1], p[2]}); });
}
int ref_strat_commit_delete(void* h, uint64_t pid) {
  return guarded([&] { static_cast<StratBox*>(h)->s->commit_delete(pid); });
}
int ref_strat_build(void* h) {
  return guarded([&] { static_cast<StratBox*>(h)->s->build(); });
}
uint64_t ref_strat_size(void* h) { return static_cast<StratBox*>(h)->store.size(); }
void ref_strat_positions(void* h, double* out) {
  const auto& st = static_cast<StratBox*>(h)->store;
  for (uint64_t i = 0; i < st.size(); ++i) {
    out[3 * i] = st[i].x;
    out[3 * i + 1] = st[i].y;
    out[3 * i + 2] = st[i].z;
  }
}
int32_t ref_strat_peak(void* h) { return static_cast<StratBox*>(h)->s->peak_cell_occupancy(); }

// dims, capacity and cell count of the grid (0 for all_pairs).
void ref_strat_grid_info(void* h, int32_t* dims, int32_t* capacity, uint64_t* ncells) {
  auto* b = static_cast<StratBox*>(h);
  *dims = 0;
  *capacity = 0;
  *ncells = 0;
  if (b->kind == 1) {
    auto& g = static_cast<CellGridStrategy&>(*b->s);
    *dims = g.cells_per_dim();
    *capacity = g.capacity_per_cell();
    *ncells = g.cell_count();
  } else if (b->kind == 2) {
    auto& g = static_cast<MicrocellGridStrategy&>(*b->s);
    *dims = g.dims();
    *capacity = g.capacity_per_cell();
    *ncells = g.cell_count();
  }
}
void ref_strat_grid(void* h, int32_t* occ, int32_t* slots) {
  auto* b = static_cast<StratBox*>(h);
  std::span<const int32_t> o, s;
  if (b->kind == 1) {
    auto& g = static_cast<CellGridStrategy&>(*b->s);
    o = g.occupancy_view();
    s = g.slots_view();
  } else if (b->kind == 2) {
    auto& g = static_cast<MicrocellGridStrategy&>(*b->s);
    o = g.occupancy_view();
    s = g.slots_view();
  }
  std::memcpy(occ, o.data(), o.size() * 4);
  std::memcpy(slots, s.data(), s.size() * 4);
}
int32_t ref_strat_cell_of(void* h, const double* p) {
  auto* b = static_cast<StratBox*>(h);
  if (b->kind == 1) return static_cast<CellGridStrategy&>(*b->s).cell_of({p[0], p[1], p[2]});
  if (b->kind == 2) return static_cast<MicrocellGridStrategy&>(*b->s).cell_of({p[0], p[1], p[2]});
  return -1;
}
// Cells the delta path scans: by cell (cell_list table / microcell window) or,
// for microcell, by position (arc product).
uint64_t ref_strat_neighborhood_of_cell(void* h, int32_t cell, int32_t* out, uint64_t cap) {
  auto* b = static_cast<StratBox*>(h);
  std::vector<int32_t> v;
  if (b->kind == 1) v = static_cast<CellGridStrategy&>(*b->s).neighborhood_cells(cell);
  if (b->kind == 2) v = static_cast<MicrocellGridStrategy&>(*b->s).neighborhood_cells(cell);
  for (uint64_t i = 0; i < v.size() && i < cap; ++i) out[i] = v[i];
  return v.size();
}
uint64_t ref_strat_neighborhood_of_pos(void* h, const double* p, int32_t* out, uint64_t cap) {
  auto* b = static_cast<StratBox*>(h);
  std::vector<int32_t> v;
  if (b->kind == 2)
    v = static_cast<MicrocellGridStrategy&>(*b->s).neighborhood_cells(Vec3{p[0], p[1], p[2]});
  for (uint64_t i = 0; i < v.size() && i < cap; ++i) out[i] = v[i];
  return v.size();
}
int ref_strat_rebuild_check(void* h, char* msg, uint64_t cap, int32_t* clean) {
  return guarded([&] {
    const auto issue = static_cast<StratBox*>(h)->s->rebuild_check();
    *clean = issue ? 0 : 1;
    copy_str(issue ? *issue : std::string(), msg, cap);
  });
}

// ---------------------------------------------------------------- simulation
// mode 0: Simulation(cfg) (fresh: init config + O(N^2) total energy)
// mode 1: Simulation(cfg, store, rng)            (prepared, total energy)
// mode 2: Simulation(cfg, store, rng, step, U, W) (resume, nothing recomputed)
int ref_sim_create(const ref_config* c, int32_t mode, const double* xyz, uint64_t n,
                   const char* rng_hex, uint64_t step, double energy, double virial, void** out) {
  return guarded([&] {
    const RunConfig cfg = to_cfg(*c);
    Simulation* s = nullptr;
    if (mode == 0)
      s = new Simulation(cfg);
    else if (mode == 1)
      s = new Simulation(cfg, ParticleStore(to_vec(xyz, n)), RngStream::deserialize_hex(rng_hex));
    else
      s = new Simulation(cfg, ParticleStore(to_vec(xyz, n)), RngStream::deserialize_hex(rng_hex),
                         step, energy, virial);
    *out = s;
  });
}

void ref_sim_destroy(void* h) { delete static_cast<Simulation*>(h); }

// Runs n steps; optional per-move trace. Returns the move-loop seconds
// (steady_clock, as bench.hpp:92-108) through *seconds.
int ref_sim_run(void* h, uint64_t n, ref_outcome* trace, double* seconds) {
  return guarded([&] {
    auto* s = static_cast<Simulation*>(h);
    const auto t0 = std::chrono::steady_clock::now();
    if (trace) {
      for (uint64_t i = 0; i < n; ++i) {
        const auto o = s->step();
        trace[i] = {static_cast<int32_t>(o.kind), o.accepted ? 1 : 0, o.delta_u, o.delta_w,
                    o.acceptance_prob, s->particle_count()};
      }
    } else {
      for (uint64_t i = 0; i < n; ++i) s->step();
    }
    const auto t1 = std::chrono::steady_clock::now();
    if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
  });
}

void ref_sim_state(void* h, ref_state* out) {
  auto* s = static_cast<Simulation*>(h);
  out->step = s->current_step();
  out->n = s->particle_count();
  out->energy = s->state().energy;
  out->virial = s->state().virial;
  for (int k = 0; k < 3; ++k) {
    out->attempted[k] = s->state().attempted[k];
    out->accepted[k] = s->state().accepted[k];
  }
  out->samples = s->statistics().samples;
  out->sum_u = s->statistics().sum_u;
  out->sum_p = s->statistics().sum_p;
  out->sum_n = s->statistics().sum_n;
  out->sum_n2 = s->statistics().sum_n2;
  out->draws = s->rng().draw_count();
  out->peak_occupancy = s->strategy().peak_cell_occupancy();
  out->pressure = s->pressure();
  out->reported_energy = s->reported_energy();
}

void ref_sim_positions(void* h, double* out) {
  const auto& st = static_cast<Simulation*>(h)->particles();
  for (uint64_t i = 0; i < st.size(); ++i) {
    out[3 * i] = st[i].x;
    out[3 * i + 1] = st[i].y;
    out[3 * i + 2] = st[i].z;
  }
}

void ref_sim_rng_hex(void* h, char* buf, uint64_t cap) {
  copy_str(static_cast<Simulation*>(h)->rng().serialize_hex(), buf, cap);
}

int ref_sim_audit(void* h, double* u_rec, double* w_rec, int32_t* passed, char* msg, uint64_t cap) {
  return guarded([&] {
    const auto r = static_cast<Simulation*>(h)->audit();
    *u_rec = r.u_recomputed;
    *w_rec = r.w_recomputed;
    *passed = r.passed() ? 1 : 0;
    copy_str(r.describe(), msg, cap);
  });
}

// Reference-format checkpoint text (checkpoint.hpp:45-58) of a live sim.
int ref_sim_checkpoint_text(void* h, char* buf, uint64_t cap, uint64_t* needed) {
  return guarded([&] {
    const std::string t = to_text(snapshot(*static_cast<Simulation*>(h)));
    *needed = t.size() + 1;
    copy_str(t, buf, cap);
  });
}

int ref_sim_stats_row(void* h, char* buf, uint64_t cap) {
  return guarded([&] { copy_str(stats_csv_row(*static_cast<Simulation*>(h)), buf, cap); });
}

// The reference grid of a live Simulation's strategy (occupancy_view() /
// slots_view(), microcell_grid.hpp:167-168, cell_grid.hpp:78-79): the engine
// path's commits (remove_id / relabel_id slot order) are byte-compared
// against it. dims = capacity = ncells = 0 for all_pairs.
void ref_sim_grid_info(void* h, int32_t* dims, int32_t* capacity, uint64_t* ncells) {
  const NeighborStrategy& s = static_cast<Simulation*>(h)->strategy();
  *dims = 0;
  *capacity = 0;
  *ncells = 0;
  if (const auto* g = dynamic_cast<const CellGridStrategy*>(&s)) {
    *dims = g->cells_per_dim();
    *capacity = g->capacity_per_cell();
    *ncells = g->cell_count();
  } else if (const auto* m = dynamic_cast<const MicrocellGridStrategy*>(&s)) {
    *dims = m->dims();
    *capacity = m->capacity_per_cell();
    *ncells = m->cell_count();
  }
}
void ref_sim_grid(void* h, int32_t* occ, int32_t* slots) {
  const NeighborStrategy& s = static_cast<Simulation*>(h)->strategy();
  std::span<const int32_t> o, sl;
  if (const auto* g = dynamic_cast<const CellGridStrategy*>(&s)) {
    o = g->occupancy_view();
    sl = g->slots_view();
  } else if (const auto* m = dynamic_cast<const MicrocellGridStrategy*>(&s)) {
    o = m->occupancy_view();
    sl = m->slots_view();
  }
  if (!o.empty()) std::memcpy(occ, o.data(), o.size() * 4);
  if (!sl.empty()) std::memcpy(slots, sl.data(), sl.size() * 4);
}

// ParticleStore::set (particles.hpp:26) on a live Simulation: moves particle
// i "behind the engine's back", as T/test_engine.cpp:186-192 does.
int ref_sim_store_set(void* h, uint64_t i, const double* p) {
  return guarded([&] {
    auto* s = static_cast<Simulation*>(h);
    if (i >= s->particles().size()) throw std::out_of_range("store: invalid particle id");
    s->particles().set(i, {p[0], p[1], p[2]});
  });
}

// run_with_files (driver.hpp:47-116) with a config given as key=value text
// (config.hpp:128-211); resume may be null. Returns the final step.
int ref_run_with_files(const char* cfg_text, const char* out_dir, const char* resume,
                       uint64_t* final_step) {
  return guarded([&] {
    const RunConfig cfg = parse_config_text(cfg_text);
    std::optional<std::filesystem::path> rp;
    if (resume && *resume) rp = std::filesystem::path(resume);
    const auto r = run_with_files(cfg, out_dir, rp);
    if (final_step) *final_step = r.final_step;
  });
}

// text.hpp:14-18 (std::to_chars general, precision 17).
void ref_format_g17(double v, char* buf, uint64_t cap) { copy_str(format_g17(v), buf, cap); }

// Restores a Simulation from reference checkpoint text (checkpoint.hpp:24-28).
int ref_sim_from_checkpoint(const char* text, void** out) {
  return guarded([&] {
    const Checkpoint c = checkpoint_from_text(text);
    *out = new Simulation(c.config, ParticleStore(c.positions),
                          RngStream::deserialize_hex(c.rng_state_hex), c.step, c.energy, c.virial);
  });
}

// P independent chains on P host threads, each its own resumed Simulation
// from the same start, seeds seed0+k: the multi-core comparator
// (BASELINE.md §4.6). Returns aggregate moves/s.
int ref_run_concurrent(const ref_config* c, const double* xyz, uint64_t n, const char* rng_hex,
                       double energy, double virial, int32_t threads, uint64_t steps_each,
                       double* agg_moves_per_s) {
  return guarded([&] {
    std::vector<std::thread> ts;
    std::vector<double> secs(static_cast<size_t>(threads), 0.0);
    const RunConfig cfg = to_cfg(*c);
    const auto start = to_vec(xyz, n);
    const auto t0 = std::chrono::steady_clock::now();
    for (int k = 0; k < threads; ++k) {
      ts.emplace_back([&, k] {
        Simulation s(cfg, ParticleStore(start), RngStream::deserialize_hex(rng_hex), 0, energy,
                     virial);
        for (uint64_t i = 0; i < steps_each; ++i) s.step();
      });
    }
    for (auto& t : ts) t.join();
    const double dt =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    *agg_moves_per_s = static_cast<double>(steps_each) * threads / dt;
  });
}

// ---------------------------------------------------------------- validate
int ref_cross_strategy_equivalence(uint64_t particles, double density, double rc, int32_t per_kind,
                                   double tol, uint64_t seed, double* max_u, double* max_w,
                                   int32_t* passed) {
  return guarded([&] {
    const auto r = validate::cross_strategy_equivalence(particles, density, rc, per_kind, tol, seed);
    *max_u = r.max_rel_u;
    *max_w = r.max_rel_w;
    *passed = r.result.passed ? 1 : 0;
  });
}

}  // extern "C"
