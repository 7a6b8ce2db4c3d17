// dw_walk.cuh -- walk-path kernel interface shared by dw_walk.cu and dw_capi.cu.
#pragma once
#include "dw_models.cuh"

namespace dwb {

// Counter slots of the per-run device accumulator (RunStats, runtime.hpp:53-73).
enum Counter : int {
    kCQueries = 0,
    kCQueryErrors,
    kCDeadEnds,
    kCTrials,
    kCWeightReads,
    kCRngDraws,
    kCFallbacks,
    kCAlgBytes,           // SURVEY §8(d) minimal-sector bytes (roofline numerator)
    kCHist,               // [33][2] selection_by_degree
    kCNum = kCHist + 66
};

struct WalkParams {
    DevGraph g;
    const uint32_t* queries;
    unsigned long long nq;
    unsigned long long qid_base;
    const unsigned long long* qids;  // [nq] global walker ids (RNG keys), or null: qid_base + i
    uint32_t* paths;        // [nq][stride] or null
    uint32_t* lengths;      // [nq] or null
    uint32_t stride;        // walk_length + 1
    uint32_t target;        // min(walk_length, max_steps)
    uint32_t seed_lo, seed_hi;
    PhiloxKeys rk;          // round keys of seed (dw_common.cuh philox_keys)
    unsigned long long cap_per_degree;
    double ratio;
    double handoff;         // tier-2 eRJS hand-off (dw_run_opts.erjs_handoff), 0 = off
    unsigned long long* counters;     // [kCNum]
    unsigned long long* next_walker;  // queue head
    int* error;                       // first DevError
    unsigned long long* error_info;   // offending query index
    ModelParams mp;
    // direct compact output (dw_capi.cu run_direct): paths is the flat id
    // array and walker i's path starts at offs[i] (offs: [nq + 1], the scan
    // of the predicted lengths); null: paths is [nq][stride]
    const unsigned long long* offs;
    unsigned int* chunk_done;         // [nq >> chunk_shift] finished walkers, or null
    unsigned int* chunk_flag;         // host-mapped: 1 once every walker of the chunk is final
    unsigned int chunk_shift;
};

enum Mode : int { kAdaptive = 0, kForceErvs = 1, kForceErjs = 2, kErvsNoJump = 3 };

#ifndef __CUDACC_RTC__
// Launches the walk over p.nq walkers on `stream`; returns the CUDA error.
cudaError_t launch_walk(int model_kind, bool weighted, int mode, const WalkParams& p,
                        int num_sms, cudaStream_t stream);
#endif

}  // namespace dwb
