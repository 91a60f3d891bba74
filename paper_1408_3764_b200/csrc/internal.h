// Host-side internals shared by the translation units of libgcmc_b200.so.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <string>

#include "common.cuh"

namespace gcmcb {

// Per-chain device handle (what gcmc_dev* points at).
struct Chain {
  int device = 0;
  gcmc_params params{};
  Box box{};
  Grid grid{};
  Mirror mirror{};               // evaluation mirror (bricks >= r_cut)
  double4* pos = nullptr;        // [capn] (inside the hot arena)
  void* arena = nullptr;         // mirror planes + brick occupancy + store (L2-persisting)
  size_t arena_bytes = 0;
  int32_t* rslot = nullptr;      // [capn] slot of particle i in its reference cell
  uint64_t capn = 0;
  ChainState* st = nullptr;      // device
  ChainState* st_host = nullptr; // pinned mirror
  // device MT19937-64 state: 312 words + position + draw counter
  uint64_t* mt = nullptr;        // [312 + 2]
  // proposal ring (engine input)
  Proposal* props = nullptr;
  uint64_t props_cap = 0;
  // proposals generated ahead for the next batch (on gen_stream, on the SM
  // the engine leaves free) and the MT state after them
  Proposal* props_next = nullptr;
  uint64_t* mt_next = nullptr;
  uint64_t ahead_n = 0;
  cudaEvent_t ev_mt = nullptr, ev_ahead = nullptr;
  gcmc_trace_rec* trace = nullptr;
  uint64_t trace_cap = 0;
  // scratch for single-move API / batches
  double* dscratch = nullptr;    // [2 * batch_cap]
  int32_t* iscratch = nullptr;
  uint64_t batch_cap = 0;
  // energy grid scratch (counting sort)
  void* egrid = nullptr;
  size_t egrid_bytes = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t gen_stream = nullptr;
  cudaEvent_t ev[4] = {};
  cudaEvent_t ev_e[4] = {};      // total_energy: pass start, k_energy start / end, pass end
  float energy_ms[2] = {0.f, 0.f};  // last total_energy: whole pass, k_energy alone
  int sm_count = 0;
  int engine_ctas = 0;        // sequencer + evaluator CTAs
  int engine2_ctas = 0;       // ... of engine2 (fewer in small boxes)
  int engine_group = 256;     // threads per evaluation slot (per-window engine)
  int engine2_group = 128;    // threads per evaluation slot (engine2)
  int engine_variants = 11;   // N-variants per displace/delete proposal (after the first)
  int engine_bias = -1;       // initial variant order (+1: N expected to grow)
  uint64_t* eng_dec = nullptr;  // engine communication buffers (engine.cu)
  uint64_t* eng_res = nullptr;
  void* eng_ext = nullptr;
  bool built = false;
  bool mirror_full = false;      // the last mirror_build overflowed a brick
  // maintained per-particle pair energy / virial (engine2.cu)
  double2* ep = nullptr;         // [capn]
  bool e_valid = false;
  void* eng2_buf = nullptr;
  size_t eng2_bytes = 0;
  int last_engine = 0;           // gcmc_run_result.engine of the last engine_run
  unsigned long long* prof = nullptr;
  unsigned long long* stamp = nullptr;  // per-round global timestamps (GCMC_ENGINE_LATENCY=1)
};

// Experiment knobs (A/B timing of engine variants, tools/build_variant.py
// NAME -DGCMC_EXPERIMENTS): read from the environment only in that build; the
// product library ignores them.
inline const char* knob(const char* name) {
#ifdef GCMC_EXPERIMENTS
  return std::getenv(name);
#else
  (void)name;
  return nullptr;
#endif
}

// Thread-local error plumbing (api.cu).
gcmc_status set_error(gcmc_status s, const std::string& msg);
gcmc_status cuda_error(cudaError_t e, const char* where);

// grid.cu
gcmc_status grid_build(Chain& c);                              // occ/slots + mirror from pos
gcmc_status mirror_build(Chain& c);
gcmc_status grid_check(Chain& c, std::string* issue);          // rebuild_check
gcmc_status commit_one(Chain& c, int kind, uint64_t pid, const double* p, uint64_t* new_pid);

// delta.cu
gcmc_status delta_batch(Chain& c, uint64_t n, const int32_t* kinds_d, const uint64_t* pids_d,
                        const double* xyz_d, double* du_d, double* dw_d);

// energy.cu
gcmc_status total_energy(Chain& c, double* u, double* w);
gcmc_status total_energy_bruteforce(Chain& c, double* u, double* w);

// gen.cu: parse the next `n` moves of the MT stream into c.props[0..n).
gcmc_status gen_proposals(Chain& c, uint64_t n, cudaStream_t s);
gcmc_status gen_proposals_into(Chain& c, uint64_t* mt, Proposal* out, uint64_t n, cudaStream_t s);
// K chains in one launch (one CTA each): c.props[0..n[i]) from c.mt
gcmc_status gen_proposals_many(Chain* const* cs, int k, const uint64_t* n, cudaStream_t s);

// engine.cu: run n moves from c.props; optional device trace.
gcmc_status engine_run(Chain& c, uint64_t n, gcmc_trace_rec* trace_d, cudaStream_t s);
size_t engine_buffer_bytes(int nslots, size_t* dec, size_t* res, size_t* ext);
int engine_max_slots();

// engine2.cu: maintained-energy engine (one slot per move)
bool engine2_supported(const Chain& c);
gcmc_status engine2_run(Chain& c, uint64_t n, gcmc_trace_rec* trace_d, cudaStream_t s);
gcmc_status epart_build(Chain& c, double2* out);
gcmc_status epart_drift(Chain& c, double* du, double* dw);
gcmc_status epart_dump(Chain& c, double* maint, double* fresh);

// engine_sm.cu: the chain-per-SM engine (one CTA; engine_mode = 2)
bool engine_sm_supported(const Chain& c);
gcmc_status engine_sm_run(Chain& c, uint64_t n, gcmc_trace_rec* trace_d, cudaStream_t s);
// k chains (one CTA each) in one launch on stream s; proposals in each c.props
gcmc_status engine_sm_run_many(Chain* const* cs, int k, const uint64_t* n, cudaStream_t s);

// initcfg.cu: random_initial_configuration on the device (same stream and result)
gcmc_status device_initial_configuration(int device, uint64_t n, double l, double min_sep, uint64_t seed,
                                         double* out_xyz, uint64_t words[312], uint64_t* index,
                                         uint64_t* draws);

// Error text in the reference's wording.
std::string overflow_message(const Chain& c, int64_t cell, int64_t occ);
std::string strategy_name(int kind);

}  // namespace gcmcb
