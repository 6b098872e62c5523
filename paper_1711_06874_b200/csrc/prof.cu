// prof.cu — opt-in per-stage device timing: CUDA events recorded on the launching stream around
// each stage's launches (tucker_profile_enable / tucker_profile_read).  Used by bench.py to time
// the dominant kernel inside the timed region without a profiler; off by default (no events).
#include <mutex>
#include <vector>

#include "common.cuh"
#include "prof.h"

namespace tk {
namespace {
struct Rec {
    int tag;
    cudaEvent_t a, b;
};
struct State {
    std::mutex mu;
    bool on = false;
    std::vector<Rec> recs;
    std::vector<cudaEvent_t> pool;
};
State& state() {
    static State s;
    return s;
}
cudaEvent_t take(State& s) {
    if (!s.pool.empty()) {
        cudaEvent_t e = s.pool.back();
        s.pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
    return e;
}
}  // namespace

ProfScope::ProfScope(int tag, cudaStream_t st) : tag_(tag), st_(st), a_(nullptr) {
    if (tag < 0) return;  // (a nested scope that must not count twice)
    State& s = state();
    std::lock_guard<std::mutex> g(s.mu);
    if (!s.on) return;
    a_ = take(s);
    if (a_ && cudaEventRecord(a_, st_) != cudaSuccess) {
        s.pool.push_back(a_);
        a_ = nullptr;
    }
}

ProfScope::~ProfScope() {
    if (!a_) return;
    State& s = state();
    std::lock_guard<std::mutex> g(s.mu);
    cudaEvent_t b = take(s);
    if (!b || cudaEventRecord(b, st_) != cudaSuccess) {
        s.pool.push_back(a_);
        if (b) s.pool.push_back(b);
        return;
    }
    s.recs.push_back(Rec{tag_, a_, b});
}

}  // namespace tk

extern "C" {

int tucker_profile_enable(int32_t on) {
    tk::State& s = tk::state();
    std::lock_guard<std::mutex> g(s.mu);
    s.on = on != 0;
    return TUCKER_OK;
}

int tucker_profile_read(double* ms, int64_t* count) {
    if (!ms || !count) return TUCKER_ERR_INVALID_ARG;
    tk::State& s = tk::state();
    std::lock_guard<std::mutex> g(s.mu);
    for (int t = 0; t < TUCKER_PROF_NSTAGES; ++t) {
        ms[t] = 0.0;
        count[t] = 0;
    }
    int rc = TUCKER_OK;
    for (const tk::Rec& r : s.recs) {
        float x = 0.f;
        if (cudaEventSynchronize(r.b) != cudaSuccess || cudaEventElapsedTime(&x, r.a, r.b) != cudaSuccess)
            rc = TUCKER_ERR_CUDA;
        if (r.tag >= 0 && r.tag < TUCKER_PROF_NSTAGES) {
            ms[r.tag] += x;
            count[r.tag] += 1;
        }
        s.pool.push_back(r.a);
        s.pool.push_back(r.b);
    }
    s.recs.clear();
    return rc;
}

}  // extern "C"
