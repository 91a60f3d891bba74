/* gcmc_b200 — B200-native grand-canonical Monte Carlo per-move energy path.
 *
 * Plain C ABI (no CUDA or torch types). One opaque handle = one Markov chain
 * on one device; host buffers are copied, the device owns the state. Every
 * call returns gcmc_status; gcmc_last_error() gives a thread-local message
 * whose text matches the exception the reference would have thrown.
 *
 * Each entry point replaces a reference interface (paths relative to
 * /root/reference/proj/include/gcmc/):
 *
 *   gcmc_create / gcmc_destroy      make_strategy + strategy ctor            engine.hpp:189-202,
 *                                                                            microcell_grid.hpp:140-156,
 *                                                                            cell_grid.hpp:48-68
 *   gcmc_upload_positions           ParticleStore(std::vector<Vec3>)         particles.hpp:19
 *   gcmc_download_positions         ParticleStore::positions()               particles.hpp:26
 *   gcmc_store_set                  ParticleStore::set()                     particles.hpp:26
 *   gcmc_build                      NeighborStrategy::build()                strategy.hpp:34
 *   gcmc_delta_displace/insert/     NeighborStrategy::delta_*                strategy.hpp:36-38
 *     delete, gcmc_delta_batch
 *   gcmc_commit_displace/insert/    NeighborStrategy::commit_*               strategy.hpp:40-42
 *     delete
 *   gcmc_rebuild_check              NeighborStrategy::rebuild_check()        strategy.hpp:46
 *   gcmc_peak_occupancy             NeighborStrategy::peak_cell_occupancy()  strategy.hpp:49
 *   gcmc_download_grid              occupancy_view() / slots_view()          microcell_grid.hpp:167-168,
 *                                                                            cell_grid.hpp:78-79
 *   gcmc_total_energy               total_energy()                           engine.hpp:74-94
 *   gcmc_set/get_rng_state          RngStream engine state                   rng.hpp:47-77
 *   gcmc_set/get_state              SystemState / RunStatistics / step_      engine.hpp:112-140, 244-252
 *   gcmc_run_moves                  Simulation::step() x n  (run_to loop)    engine.hpp:293-325
 *   gcmc_random_initial_configuration  random_initial_configuration()        init_config.hpp:19-64
 *   gcmc_device_initial_configuration  (the same, on the device)              init_config.hpp:19-64
 *   gcmc_run_chains                 (no reference counterpart: K independent Simulations, e.g. the
 *                                   points of a mu/T sweep, advanced concurrently on one device;
 *                                   PAPER.md:632 future work)
 */
#ifndef GCMC_B200_H
#define GCMC_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum gcmc_status {
  GCMC_OK = 0,
  GCMC_INVALID_PID = 1,   /* std::out_of_range ("...: invalid particle id")          */
  GCMC_CELL_OVERFLOW = 2, /* std::runtime_error ("...: cell C exceeds capacity K...") */
  GCMC_NOT_FOUND = 3,     /* std::runtime_error ("...not found in cell C")           */
  GCMC_OVERLAP = 4,       /* std::runtime_error ("total_energy: particles i and j overlap") */
  GCMC_CUDA = 5,          /* CUDA runtime failure                                     */
  GCMC_ARG = 6,           /* std::invalid_argument / config error                     */
  GCMC_STATE = 7          /* call not valid in the current state                      */
} gcmc_status;

/* Strategy enum values match gcmc::Strategy (config.hpp:16). */
enum { GCMC_ALL_PAIRS = 0, GCMC_CELL_LIST = 1, GCMC_MICROCELL = 2 };

/* RunConfig subset the per-move path needs (config.hpp:42-64). */
typedef struct gcmc_params {
  double box_length;
  double epsilon, sigma, r_cut;
  double temperature, chemical_potential, lambda;
  double displace_percent, max_displacement;
  uint64_t equilibration_steps, sampling_interval;
  int32_t strategy;
  int32_t cell_capacity;      /* 0 = default_cell_capacity() (cell_grid.hpp:36-38) */
  int32_t microcell_capacity; /* 0 = 5 (microcell_grid.hpp:149) */
  int32_t tail_corrections;
  uint64_t max_particles;     /* initial store capacity (0 = automatic: as many particles as the
                                 reference grid and the evaluation mirror can hold); the store
                                 grows as needed, like the reference's std::vector */
  int32_t engine_ctas;        /* engine CTAs: 1 sequencer + evaluators (0 = every SM but one; engine2: fewer in small boxes) */
  int32_t engine_group;       /* threads per evaluation slot: 128/256/512 (0 = 256 per-window engine, 128 engine2) */
  int32_t engine_variants;    /* per-window engine: N-variants per displace/delete proposal
                                 after the first (0 = 11, at most 15) */
  int32_t engine_bias;        /* initial variant order: -1 N expected to fall, +1 rise (0 = -1) */
  int32_t engine_mode;        /* 0 = maintained-energy engine where supported (brick strategies,
                                 max_displacement = 0; the chain-per-SM engine when
                                 engine_share >= 12), 1 = per-window engine always,
                                 2 = chain-per-SM engine (one CTA per chain; brick
                                 strategies, max_displacement = 0, else as 0) */
  int32_t engine_share;       /* chains that share the device (gcmc_run_chains): with engine_ctas
                                 = 0 this chain's engine takes (SMs - share) / share CTAs
                                 (0 or 1 = the whole device) */
} gcmc_params;

/* SystemState + RunStatistics + step counter (engine.hpp:112-140, 436). */
typedef struct gcmc_state {
  uint64_t step;
  uint64_t n;
  double energy, virial;
  uint64_t attempted[3], accepted[3]; /* index = MoveKind: displace, insert, remove */
  uint64_t samples;
  double sum_u, sum_p, sum_n, sum_n2;
  int32_t peak_occupancy;
  int32_t pad;
} gcmc_state;

/* One MoveOutcome (engine.hpp:104-110) plus N after the move. */
typedef struct gcmc_trace_rec {
  int32_t kind; /* 0 displace, 1 insert, 2 remove */
  int32_t accepted;
  double delta_u, delta_w, acceptance_prob;
  uint64_t n_after;
} gcmc_trace_rec;

typedef struct gcmc_run_result {
  gcmc_state state;   /* after the run */
  uint64_t moves;     /* moves executed by this call */
  uint64_t rounds;    /* speculative evaluation rounds the device used */
  double device_ms;   /* device time of the move loop (CUDA events) */
  double gen_ms;      /* device time of proposal generation */
  uint64_t pair_evals; /* FP64 pair evaluations (minimum image + cutoff test) the device
                          performed for this call: windows, energy updates, all-pairs scans */
  int32_t engine;     /* engine that ran the moves: 1 per-window (engine.cu), 2 multi-SM
                         maintained-energy (engine2.cu), 3 chain-per-SM (engine_sm.cu) */
  int32_t pad;
} gcmc_run_result;

typedef struct gcmc_dev gcmc_dev;

const char* gcmc_last_error(void);
const char* gcmc_version(void);

gcmc_status gcmc_create(const gcmc_params* params, int device, gcmc_dev** out);
gcmc_status gcmc_destroy(gcmc_dev* h);

/* Positions are AoS xyz doubles (Vec3, vec3.hpp:7-27). Upload replaces the
 * store and rebuilds the grid (the strategy ctor builds immediately). */
gcmc_status gcmc_upload_positions(gcmc_dev* h, const double* xyz, uint64_t n);
gcmc_status gcmc_download_positions(gcmc_dev* h, double* xyz, uint64_t capacity, uint64_t* n);
gcmc_status gcmc_build(gcmc_dev* h);
/* Overwrites particle pid's position in the store only — the grid is NOT
 * updated, exactly like ParticleStore::set under a live strategy. For audits'
 * fault-injection tests (T/test_engine.cpp:186-192). */
gcmc_status gcmc_store_set(gcmc_dev* h, uint64_t pid, const double pos[3]);

/* Grid geometry: cells per axis, slots per cell, total cells. */
gcmc_status gcmc_grid_info(gcmc_dev* h, int32_t* dims, int32_t* capacity, uint64_t* ncells);
gcmc_status gcmc_download_grid(gcmc_dev* h, int32_t* occ, int32_t* slots);
gcmc_status gcmc_rebuild_check(gcmc_dev* h, char* msg, size_t msg_cap, int32_t* clean);
gcmc_status gcmc_peak_occupancy(gcmc_dev* h, int32_t* peak);

gcmc_status gcmc_delta_displace(gcmc_dev* h, uint64_t pid, const double pos[3], double* du,
                                double* dw);
gcmc_status gcmc_delta_insert(gcmc_dev* h, const double pos[3], double* du, double* dw);
gcmc_status gcmc_delta_delete(gcmc_dev* h, uint64_t pid, double* du, double* dw);
/* n proposals against the same state: kinds[i] 0/1/2, pids[i], xyz[3i..3i+2]. */
gcmc_status gcmc_delta_batch(gcmc_dev* h, uint64_t n, const int32_t* kinds, const uint64_t* pids,
                             const double* xyz, double* du, double* dw);

gcmc_status gcmc_commit_displace(gcmc_dev* h, uint64_t pid, const double pos[3]);
gcmc_status gcmc_commit_insert(gcmc_dev* h, const double pos[3], uint64_t* pid);
gcmc_status gcmc_commit_delete(gcmc_dev* h, uint64_t pid);

gcmc_status gcmc_total_energy(gcmc_dev* h, double* u, double* w);

/* Diagnostic (no reference counterpart): largest |e_i - fresh e_i| over the
 * per-particle pair energies / virials the maintained-energy engine carries
 * across moves, against a from-scratch evaluation (0, 0 when not in use). */
gcmc_status gcmc_energy_drift(gcmc_dev* h, double* max_du, double* max_dw);

/* Diagnostic: total_energy() as the reference computes it — every pair i < j,
 * no cell structure (engine.hpp:74-94's O(N^2) loop) — on the device. A
 * cross-check of gcmc_total_energy's cell-based pass (~1 s at 1M). */
gcmc_status gcmc_total_energy_bruteforce(gcmc_dev* h, double* u, double* w);

/* Diagnostic (no reference counterpart): device time of the last
 * gcmc_total_energy (CUDA events on the chain's stream): the whole pass
 * (binning, sort, pair sums, reduction) and the pair-sum kernel alone. */
gcmc_status gcmc_energy_timing(gcmc_dev* h, double* pass_ms, double* kernel_ms);

/* std::mt19937_64 state in libstdc++ order: 312 words + position (_M_p),
 * plus RngStream's draw counter. */
gcmc_status gcmc_seed_rng(gcmc_dev* h, uint64_t seed);
gcmc_status gcmc_set_rng_state(gcmc_dev* h, const uint64_t words[312], uint64_t index,
                               uint64_t draws);
gcmc_status gcmc_get_rng_state(gcmc_dev* h, uint64_t words[312], uint64_t* index,
                               uint64_t* draws);

gcmc_status gcmc_set_state(gcmc_dev* h, const gcmc_state* s); /* resume (n is ignored) */
gcmc_status gcmc_get_state(gcmc_dev* h, gcmc_state* s);

/* Runs n Simulation::step()s on the device: proposals from the device MT
 * stream, exact speculative evaluation, on-device acceptance, commit and
 * statistics. `trace` (host, nullable) receives one record per move. */
gcmc_status gcmc_run_moves(gcmc_dev* h, uint64_t n, gcmc_trace_rec* trace,
                           gcmc_run_result* out);

/* K chains (distinct handles, any devices) each run n[i] moves concurrently,
 * exactly as K gcmc_run_moves calls would; out (nullable) receives K results.
 * Create each chain with gcmc_params.engine_share = K (or an explicit
 * engine_ctas) so that the K engines and their K proposal generators fit the
 * device together. Returns the first failing chain's status;
 * the message names the chain. */
gcmc_status gcmc_run_chains(gcmc_dev* const* hs, int32_t k, const uint64_t* n,
                            gcmc_run_result* out);

/* random_initial_configuration (init_config.hpp:19-64) on the device: the
 * same MT19937-64 stream, bit-identical positions in the same order, the same
 * RNG state afterwards and the same error after 10^6 consecutive rejections;
 * candidates are tested in parallel blocks against the particles placed so
 * far, and within a block in candidate order. */
gcmc_status gcmc_device_initial_configuration(int device, uint64_t n, double box_length,
                                              double min_sep, uint64_t seed, double* out_xyz,
                                              uint64_t words[312], uint64_t* index, uint64_t* draws);

/* Host-side initial configuration (init_config.hpp:19-64) consuming the
 * identical MT stream; returns the RNG state left for the MC stream. */
gcmc_status gcmc_random_initial_configuration(uint64_t n, double box_length, double min_sep,
                                              uint64_t seed, double* out_xyz,
                                              uint64_t words[312], uint64_t* index,
                                              uint64_t* draws);

#ifdef __cplusplus
}
#endif
#endif /* GCMC_B200_H */
