// Plan-specialised fused stem chains compiled with NVRTC (chain_jit.cpp).
#pragma once

#include <string>
#include <vector>

#include "kernels.h"

namespace stn {

struct ChainJitSpec {
  const ChainGeom *geom;
  const ChainTables *tables;  // host copy
};

bool chain_jit_available();
// Compiles one kernel per chain (one NVRTC program, cached per process and device);
// fns[i] receives chain i's CUfunction. False (and *log) if NVRTC is unavailable or
// the compilation failed: the chains then run on kernels_chain.cu.
bool chain_jit_compile(const std::vector<ChainJitSpec> &chains, bool exact, int device,
                       std::vector<void *> *fns, std::string *log);
// NVRTC compilation alone (no device needed): the CPU check that generated code builds.
bool chain_jit_compile_only(const std::vector<ChainJitSpec> &chains, bool exact,
                            std::string *log);
cudaError_t chain_jit_launch(void *fn, const ChainGeom &g, const ChainTables *T_device,
                             const BatchPtrs &p, cudaStream_t stream);

}  // namespace stn
