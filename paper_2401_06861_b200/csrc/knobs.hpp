// Environment options, in one place.
//
// Supported runtime options:
//   NQ_JIT=off|sync|auto    pass-specialised kernels (auto: compiled in the
//                           background, the generic pass kernel meanwhile)
//   NQ_JIT_PX=0             register permutations applied eagerly instead of
//                           pending (the plain path the PX machinery is checked against)
//   NQ_TILE_SV, NQ_TILE_DM  tile qubits per CTA (default 11)
//   NQ_EXCHANGE=nccl        sharded exchanges through NCCL send/recv instead of
//                           CUDA-IPC peer memory
//   NQ_FUSED_EXCHANGE=0     no exchange fused into the preceding pass
//                           (=staged: the staged form even when a second copy fits)
//   NQ_COMM=host            sharded ranks coordinate through host shared memory
//                           instead of NCCL (ranks may share one GPU: tests)
//   NQ_NCCL_LIB             libnccl.so.2 to bind when none is loaded yet
// Diagnostics (no effect on plans or results):
//   NQ_PLAN_TRACE, NQ_SHARD_TRACE, NQ_SHARD_TIMING, NQ_JIT_DUMP,
//   NQ_BATCH_TIMING, NQ_SEGV_TRACE
// A/B switches: alternatives measured on B200 and kept for re-measurement
// (DESIGN.md §5 lists each with its measurement).  They are read only in a
// build made with `make AB=1` (-DNQ_AB_KNOBS); the product build compiles the
// default in and ignores the environment.
#pragma once

#include <cstdint>
#include <string>

namespace nqe {

// A supported option: the integer value of `name`, `dflt` if unset.
int env_option(const char* name, int dflt);
// A supported string option ("" if unset).
std::string env_option_str(const char* name);
// An A/B switch: `dflt` unless built with NQ_AB_KNOBS.
int ab_knob(const char* name, int dflt);
// Every NQ_* variable that can change a plan, a kernel or an exchange
// ("NAME=value;" sorted; diagnostics excluded).  Sharded states check at
// creation that all ranks agree, since each rank plans its flushes alone.
std::string plan_env_fingerprint();

}  // namespace nqe
