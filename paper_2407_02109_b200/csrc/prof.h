// RAII scope around one kernel launch: counts launches and, when profiling is enabled
// (pscwin_profile_enable), records CUDA events on the launching stream before and after it.
#pragma once
#include <cuda_runtime.h>
#include <string.h>

namespace pscwin {
class ProfScope {
 public:
  ProfScope(const char* name, cudaStream_t s);
  ~ProfScope();

 private:
  const char* name_;
  cudaStream_t s_;
  void* a_;
};
}  // namespace pscwin
#define PSCWIN_PROF(name, stream) ::pscwin::ProfScope _pscwin_prof_scope_(name, stream)
