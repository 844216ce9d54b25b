// Cycle scan — placeholder until the chunked closed-form kernels land.
#include "../../include/pscwin.h"
#include "pscwin_internal.h"

namespace pscwin {
int cycle_scan_module(const void*, const void*, const void*, void*, void*, size_t, size_t, size_t, size_t, size_t,
                      cudaStream_t) {
  return PSCWIN_ERR_UNSUPPORTED;
}
}  // namespace pscwin

extern "C" size_t pscwin_scan_workspace_bytes(const pscwin_scan_desc*) { return 256; }
extern "C" int pscwin_cycle_scan(const pscwin_scan_desc*, const void*, const void*, const float*, const float*,
                                 const void*, const float*, const float*, const float*, const float*, void*, void*,
                                 size_t, void*) {
  return PSCWIN_ERR_UNSUPPORTED;
}
