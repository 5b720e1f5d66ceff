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
// log2 of the widest tile access group the specialised kernels use (1: 16 B, 2: 32 B)
int chain_vec_max();
// Compiles one kernel per chain (one NVRTC program, cached per process and device);
// fns[i] receives chain i's CUfunction. False (and *log) if NVRTC is unavailable or
// the compilation failed: the chains then run on kernels_chain.cu.
bool chain_jit_compile(const std::vector<ChainJitSpec> &chains, bool exact, int device,
                       std::vector<void *> *fns, std::string *log,
                       std::vector<int> *local_bytes = nullptr,
                       std::vector<void *> *alt_fns = nullptr);
// NVRTC compilation alone (no device needed): the CPU check that generated code builds.
bool chain_jit_compile_only(const std::vector<ChainJitSpec> &chains, bool exact,
                            std::string *log);
// Lane / tile exchange that makes a tile's warp accesses whole 32-byte sectors: when
// tensor position 0 is a lane bit and position 1 a tile line, lane bit *j and tile
// slot bit *s swap roles through warp shuffles (the tile then holds positions 0 and 1:
// 32-byte accesses). False when no exchange helps. lane_off / elem_off: offsets of
// the lane bits / tile elements (ChainTables xl, xin or ol, oout).
bool chain_lane_swap(const int64_t *lane_off, const int64_t *elem_off, int n_log, int *j, int *s);
// Whether a chain's kernel may use those exchanges (register budget), and whether it
// software-pipelines its rows.
bool chain_swaps_allowed(const ChainGeom &g);
bool chain_prefetch(const ChainGeom &g);
// The offsets after that exchange (physical access pattern).
void chain_apply_swap(const int64_t *lane_off, const int64_t *elem_off, int n_log, int j, int s,
                      int64_t *lane_out, int64_t *elem_out);
cudaError_t chain_jit_launch(void *fn, const ChainGeom &g, const ChainTables *T_device,
                             const BatchPtrs &p, cudaStream_t stream);

}  // namespace stn
