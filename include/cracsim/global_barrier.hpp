// cracsim B200 build — the host barrier that marks a consistent global
// checkpoint across the per-GPU processes of one job (SURVEY §8(e),
// BASELINE.json north_star: "only a host-side barrier marks a consistent global
// checkpoint").
//
// The reference is single-process (/root/reference/proj/src/ckpt_engine.cpp:29-61
// quiesces one DispatchTable); the B200 box runs one process per GPU, each with
// its own Session and drain.  A Session may carry a GlobalBarrier hook; every
// checkpoint entry point calls it at two points:
//
//   kPhaseQuiesced   inside the quiesce, before any state is read: returning
//                    means every rank's application is stopped with its queued
//                    device work drained, so no rank's application runs past
//                    the checkpoint line while another's is still running.
//   kPhaseImageComplete  after this rank's image is complete in host memory
//                    (after the shadow / pre-copy D2H for the split drains):
//                    returning means every rank's image is complete, i.e. the
//                    global checkpoint is committed.
//   kPhasePersisted  checkpoint_to_file only, after the file write + fdatasync.
//
// A hook returning nonzero fails the checkpoint with QuiesceTimeout (the
// application is resumed; no image is committed).
//
// ShmBarrier is the built-in hook for ranks on one node: a sense-reversing
// barrier in a POSIX shared-memory segment, one 64-bit word (generation,
// arrivals) updated by CAS, so an arrival that times out can be withdrawn and
// the barrier stays usable.  Multi-node jobs pass their own hook (e.g. an
// MPI_Barrier wrapper) through the same C-ABI.
#pragma once

#include <atomic>
#include <chrono>
#include <cstdint>
#include <string>

namespace cracsim {

enum GlobalPhase : int {
  kPhaseQuiesced = 0,
  kPhaseImageComplete = 1,
  kPhasePersisted = 2,
};

struct GlobalBarrier {
  int (*fn)(void* ctx, int phase) = nullptr;  // 0 = all ranks arrived
  void* ctx = nullptr;
  explicit operator bool() const { return fn != nullptr; }
};

class ShmBarrier {
 public:
  // Opens (creating on first use) the segment `name` ("/crac_..." as for
  // shm_open) for `world` ranks.  Every rank of the job opens the same name
  // with the same world; ranks may open in any order.
  ShmBarrier(const std::string& name, uint32_t world, uint32_t rank,
             std::chrono::milliseconds timeout);
  ~ShmBarrier();
  ShmBarrier(const ShmBarrier&) = delete;
  ShmBarrier& operator=(const ShmBarrier&) = delete;

  // One arrival.  Returns true when all `world` ranks arrived, false on
  // timeout (the arrival is withdrawn first).
  bool wait();
  uint64_t generation() const;
  uint32_t world() const { return world_; }
  uint32_t rank() const { return rank_; }
  void unlink_on_close() { unlink_ = true; }
  // the crac_barrier_fn-compatible entry (ctx = ShmBarrier*)
  static int hook(void* ctx, int phase);

  struct Shared {
    std::atomic<uint32_t> state;  // 0 fresh, 1 initialising, 2 ready
    uint32_t world;
    std::atomic<uint64_t> word;   // generation << 32 | arrivals
    std::atomic<uint64_t> waits;  // completed barrier episodes (diagnostic)
  };

 private:
  std::string name_;
  uint32_t world_, rank_;
  std::chrono::milliseconds timeout_;
  Shared* sh_ = nullptr;
  bool unlink_ = false;
};

}  // namespace cracsim
