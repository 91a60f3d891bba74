/* TEST INFRASTRUCTURE ONLY — the CPU restatement ("port") of the reference's
 * per-move energy path, used as the parity checker by tests/ and as the
 * cpu_baseline "port" leg of bench.py. Never linked into the product.
 *
 * Every function restates a reference routine; the .c file cites the
 * reference file:line for each. Paths are relative to
 * /root/reference/proj/include/gcmc/.
 *
 * Parity of this restatement is pinned (tests/test_oracle_cpu.py) against:
 *   - the compiled reference (oracle/_ref/libgcmc_ref.so) when present,
 *   - golden vectors in tests/golden/ generated from that reference by
 *     tests/golden/make_golden.py,
 *   - the C++ standard's mt19937_64 known-answer value (10000th output of
 *     the default-seeded engine = 9981545732273789042).
 */
#ifndef GCMC_ORACLE_H
#define GCMC_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* std::mt19937_64 (rng.hpp:84): 312 words + position, libstdc++ layout. */
typedef struct {
  uint64_t mt[312];
  uint64_t idx;   /* libstdc++ _M_p: 312 right after seeding */
  uint64_t draws; /* RngStream::draws_ (rng.hpp:44) */
} orc_rng;

void orc_rng_seed(orc_rng* r, uint64_t seed);
uint64_t orc_rng_next(orc_rng* r);
double orc_uniform(orc_rng* r);
uint64_t orc_index_from(double u, uint64_t n);

double orc_wrap_axis(double v, double l);
int orc_wrap_position(const double* p, double l, double* out); /* -1 on non-finite */
double orc_min_image_dist2(const double* a, const double* b, double l);

typedef struct {
  double epsilon, sigma, r_cut, sigma2, r_cut2;
} orc_lj;
orc_lj orc_lj_make(double eps, double sigma, double rc);
int orc_lj_pair(double r2, const orc_lj* p, double* u, double* w); /* -1 if r2 <= 0 */
void orc_lj_pair_clamped(double r2, const orc_lj* p, double* u, double* w);
void orc_tail_corrections(double rho, double eps, double sigma, double rc, double* u, double* pr);

double orc_displacement_acceptance(double du, double beta);
double orc_insertion_acceptance(double du, uint64_t n, double v, double beta, double mu, double lam);
double orc_deletion_acceptance(double du, uint64_t n, double v, double beta, double mu, double lam);

void orc_compute_cell_dims(double l, double rc, int32_t* dims, double* size);
int32_t orc_default_cell_capacity(double rc, double sigma);
void orc_microcell_dims(double l, double sigma, int32_t* dims, double* last_w);
int32_t orc_microcell_extent(double rc, double sigma);
void orc_microcell_axis_window(int32_t center, double rc, double sigma, int32_t dims, double last_w,
                               int32_t* lo, int32_t* count);
void orc_microcell_axis_arc(double x, double rc, double sigma, double l, int32_t dims,
                            int32_t* first, int32_t* count);

/* ---------------------------------------------------------------- grid */
enum { ORC_ALL_PAIRS = 0, ORC_CELL_LIST = 1, ORC_MICROCELL = 2 };

enum {
  ORC_OK = 0,
  ORC_INVALID_PID = 1,
  ORC_CELL_OVERFLOW = 2,
  ORC_NOT_FOUND = 3,
  ORC_OVERLAP = 4,
  ORC_ARG = 5
};

typedef struct orc_grid orc_grid; /* strategy + its particle store */

orc_grid* orc_grid_create(int32_t kind, const double* xyz, uint64_t n, uint64_t capacity_n,
                          double l, double eps, double sigma, double rc, int32_t cell_cap,
                          int32_t* status);
void orc_grid_destroy(orc_grid* g);
int32_t orc_grid_build(orc_grid* g);
uint64_t orc_grid_size(const orc_grid* g);
const double* orc_grid_positions(const orc_grid* g); /* xyz AoS, size() records */
void orc_grid_info(const orc_grid* g, int32_t* dims, int32_t* cap, uint64_t* ncells);
const int32_t* orc_grid_occ(const orc_grid* g);
const int32_t* orc_grid_slots(const orc_grid* g);
int32_t orc_grid_peak(const orc_grid* g);
int32_t orc_grid_cell_of(const orc_grid* g, const double* p);

int32_t orc_delta_displace(const orc_grid* g, uint64_t pid, const double* p, double* du, double* dw);
int32_t orc_delta_insert(const orc_grid* g, const double* p, double* du, double* dw);
int32_t orc_delta_delete(const orc_grid* g, uint64_t pid, double* du, double* dw);
int32_t orc_commit_displace(orc_grid* g, uint64_t pid, const double* p);
int32_t orc_commit_insert(orc_grid* g, const double* p, uint64_t* pid);
int32_t orc_commit_delete(orc_grid* g, uint64_t pid);
int32_t orc_rebuild_check(const orc_grid* g); /* 1 clean, 0 inconsistent */
const char* orc_last_error(void);

int32_t orc_total_energy(const double* xyz, uint64_t n, double l, double eps, double sigma,
                         double rc, double* u, double* w);

/* init_config.hpp:19-64 */
int32_t orc_random_initial_configuration(uint64_t n, double l, double min_sep, orc_rng* r,
                                         double* out_xyz);

/* ---------------------------------------------------------------- engine */
typedef struct {
  double temperature, chemical_potential, lambda, epsilon, sigma, r_cut, box_length;
  double displace_percent, max_displacement;
  uint64_t equilibration_steps, sampling_interval;
  int32_t strategy, tail_corrections, cell_capacity, microcell_capacity;
} orc_params;

typedef struct {
  int32_t kind, accepted;
  double delta_u, delta_w, acceptance_prob;
  uint64_t n_after;
} orc_outcome;

typedef struct {
  uint64_t step;
  double energy, virial;
  uint64_t attempted[3], accepted[3];
  uint64_t samples;
  double sum_u, sum_p, sum_n, sum_n2;
} orc_state;

typedef struct orc_sim orc_sim;
orc_sim* orc_sim_create(const orc_params* p, const double* xyz, uint64_t n, const orc_rng* rng,
                        uint64_t step, double energy, double virial, int32_t* status);
void orc_sim_destroy(orc_sim* s);
int32_t orc_sim_run(orc_sim* s, uint64_t n, orc_outcome* trace);
void orc_sim_state(const orc_sim* s, orc_state* out);
const orc_grid* orc_sim_grid(const orc_sim* s);
const orc_rng* orc_sim_rng(const orc_sim* s);

#ifdef __cplusplus
}
#endif
#endif
