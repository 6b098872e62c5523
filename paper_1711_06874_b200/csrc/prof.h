// prof.h — RAII stage scope for the opt-in device timing of prof.cu (tucker_profile_enable).
#pragma once

#include <cuda_runtime.h>

#include "../../include/tucker.h"

namespace tk {

class ProfScope {
  public:
    ProfScope(int tag, cudaStream_t st);
    ~ProfScope();
    ProfScope(const ProfScope&) = delete;
    ProfScope& operator=(const ProfScope&) = delete;

  private:
    int tag_;
    cudaStream_t st_;
    cudaEvent_t a_;
};

}  // namespace tk

#define TK_PROF_CAT2(a, b) a##b
#define TK_PROF_CAT(a, b) TK_PROF_CAT2(a, b)
#define TK_PROF(tag, st) ::tk::ProfScope TK_PROF_CAT(tk_prof_, __LINE__)((tag), (st))
