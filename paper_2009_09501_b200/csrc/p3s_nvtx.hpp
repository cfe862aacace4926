// NVTX ranges on the host threads (nvtx3, header-only: a no-op unless a profiler such as
// Nsight Systems injects itself), so a timeline shows each p3s_convert, its enqueue and its
// wait, each video frame and each sequence frame next to the kernels they launch.
#pragma once

#include <nvtx3/nvToolsExt.h>

namespace p3s {

class NvtxRange {
public:
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

}  // namespace p3s
