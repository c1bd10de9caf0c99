// NVTX phase ranges of the solver (SURVEY section 5 "tracing"): header-only NVTX3, a no-op unless a
// tool (ncu --nvtx, nsys) is attached. Ranges: one per outer iteration phase of Algorithm 2
// and one per trust-region / truncated-CG call, so that `ncu --nvtx --nvtx-include
// "drsdp:tcg/"` captures the kernels of one phase only.
#pragma once
#include <nvtx3/nvToolsExt.h>

namespace drsdp {

struct NvtxRange {
  explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange &) = delete;
  NvtxRange &operator=(const NvtxRange &) = delete;
};

// consecutive phases inside one scope: set() closes the previous phase; the destructor closes the last
// (so `continue`, `break` and early returns leave no range open)
struct NvtxPhase {
  bool open = false;
  void set(const char *name) {
    if (open) nvtxRangePop();
    nvtxRangePushA(name);
    open = true;
  }
  void end() {
    if (open) nvtxRangePop();
    open = false;
  }
  ~NvtxPhase() { end(); }
};

}  // namespace drsdp
