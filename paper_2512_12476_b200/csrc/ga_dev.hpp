// Device-resident GA offspring loop: the state one run of
// ga_run (reference search.cpp:437-565) keeps between evaluation waves, laid
// out for a persistent kernel in which every warp is a worker. Host and device
// share these definitions.
//
// Per run, the record pool holds fixed-stride slots:
//   0                          best inserted member (ga_search's result)
//   1                          plan of the latest improvement (incumbent)
//   [2, 2 + pop_cap)           population members (pop_slot maps rank -> slot;
//                              entries past n_pop are the free slots)
//   2 + pop_cap + b*max_wave   stage buffer b (0/1) of max_wave records
// A wave always goes to the buffer that does not hold the current child, so
// the child (and a speculative stage kept for the next offspring) survive it.
#pragma once

#include <cstdint>

#include "common.hpp"
#include "rng.hpp"

namespace hpg {

constexpr int kGaTrials = 8;      // mutation tries per offspring (search.cpp:490-500)
constexpr int kGaMaxPop = 64;     // population knob limit of the device path
constexpr int kGaMaxSps = 16;     // swap_pair_sample limit of the device path
constexpr int kGaStreakCap = 64;  // infeasible-offspring streak (search.cpp:481)
constexpr int kGaJumps = 127;     // jump polynomials per gen_draws: lane offsets of a 4-warp team

// a mutation stage: ntr mutated trials + the unmutated parent at
// stage buffer `buf`, indices [base, base + ntr]
struct alignas(16) GaStage {
  int32_t buf, base, ntr, pad;
  Rng start, after_all;
  Rng snaps[kGaTrials];
};

enum GaState : int32_t {
  kGaLoop = 0,
  kGaMut = 1,
  kGaSwap = 2,
  kGaRedraw = 3,
  kGaDone = 4,
  kGaInit = 5,      // draw the next init chunk
  kGaInitDone = 6,  // take the chunk's results
  kGaSwap3 = 7,     // throughput mode: the L3-only swap wave finished
};

struct alignas(16) GaRun {
  // ---- set by the host ----
  int64_t slice;
  int64_t pool_off;    // byte offset of this run's record pool
  int32_t rec_stride;  // bytes per record slot (multiple of 16)
  int32_t ng;          // task groups
  int32_t gstart[kMaxTasks + 1];
  int32_t gslot[kMaxTasks];  // task slots, group by group (ArmEnv::tg order)
  int32_t counts[kMaxTasks];  // devices per group
  int32_t opt_off[kMaxTasks + 1];  // layout options of gslot[k]: opts[opt_base + opt_off[k] ...]
  int64_t opt_base;
  int32_t gen_draws;    // RNG draws per make_candidate (gen_draws_per_candidate)
  int32_t jump_off;     // jumps[jump_off + L - 1] = x^(L*gen_draws) mod p, L = 1..31
  int32_t init_target;  // ga_run init (search.cpp:437-450)
  int64_t attempt_cap, attempts, combo, chunk;
  // ---- GA state (host initialises after the init phase) ----
  Rng rng;
  int64_t used, streak, seq;
  double best;
  double best_member_cost;
  int32_t n_pop, state;
  int32_t pending;  // evaluations outstanding in the current wave
  int32_t wave_buf, wave_n;
  int32_t have_spec;
  int32_t best_member_flags;  // bit0: has a best member, bit1: replaced on the device
  int32_t impr_flags;         // bit0: improvement plan replaced on the device
  int32_t child_buf, child_idx;
  double child_cost;
  int32_t n3, n5, m5, pad0;
  Rng before3, before5, b5;
  Rng spec_from;  // stream position of the swap wave's speculative stage
  int64_t n_offspring, n_waves, n_evals, pad1;
  unsigned long long impr_time;  // globaltimer at the latest improvement
  int32_t pop_slot[kGaMaxPop];
  double pop_cost[kGaMaxPop];
  uint64_t pop_seq[kGaMaxPop];
  GaStage cur, spec;
  Rng snaps3[kGaMaxSps], snaps5[kGaMaxSps];
};

// one improvement of a run's incumbent (Improvement, search.cpp:456-460)
struct GaImpr {
  int32_t run, pad;
  int64_t local_idx;
  double cost;
  unsigned long long t;
};

// control words, one 128-byte line each
enum GaCtl : int {
  kGaCtlHead = 0,
  kGaCtlTail = 16,
  kGaCtlDone = 32,     // runs finished
  kGaCtlStop = 48,     // all runs finished: workers exit
  kGaCtlImpr = 64,     // improvements appended
  kGaCtlEvals = 80,    // plans evaluated
  kGaCtlBytes = 96,    // canonical bytes of the evaluated plans
  kGaCtlT0 = 112,      // globaltimer at kernel start
  kGaCtlProf = 120,    // diagnostics: step cycles, steps, eval cycles, evals
  kGaCtlWords = 128,
};

struct GaParams {
  GaRun* runs;
  int32_t n_runs, pop_cap, sps, max_wave;
  uint8_t* pool;
  EvalResult* res;  // [run][2][max_wave]
  const int32_t* id_rank;     // device -> lexicographic id rank
  const int32_t* by_id_rank;  // id rank -> device
  // work queue: payload (run, index; index 0xffffffff = GA step) and the
  // ticket that published it (Vyukov-style bounded ring)
  uint2* q_pay;
  unsigned long long* q_seq;
  unsigned long long q_mask;
  unsigned long long* ctl;  // kGaCtlWords words
  GaImpr* impr;
  int64_t impr_cap;
  int32_t kb_flags, n_tasks;
  // init phase: candidate generation (make_candidate on the device)
  const short4* opts;        // layout options (dp, pp, tp, -)
  Rng* init_snaps;           // [run][init_cap] stream after each init candidate
  const uint64_t* jumps;     // jump polynomials (rng_jump.hpp), 4 words each
  uint8_t* gen_scratch;      // per worker: 32 lanes x gen_smem bytes
  int32_t init_cap, res_per_run;
  int32_t gen_smem;          // scratch bytes per generating lane
  int32_t n_regions, n_nodes, max_nodes_per_region, n_dev;
  int32_t gen_in_smem;       // generation scratch in shared memory (else gen_scratch)
  double bias;               // locality_bias
  const int32_t* region_off;
  const int32_t* node_off;
  const uint8_t* node_devs;
  const int16_t* node_rank;
  int64_t task_nl[kMaxTasks];
  int32_t max_stride;  // record slot stride (multiple of 16)
  int32_t split_runs;  // more live runs than this: swap waves without L5 / speculation up front
  int32_t prof;        // diagnostics: cycle counters in ctl[kGaCtlProf..]
};

}  // namespace hpg
