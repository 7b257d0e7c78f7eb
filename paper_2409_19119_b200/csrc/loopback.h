// loopback.h -- the single-GPU loopback group (internal; the ABI is nek_loopback_* in nek.h).
//
// P virtual ranks in one process, one host thread and one context per rank, all on one device
// (SURVEY 4 "loopback comm backend"; SPEC S:196/S:235 runs ranks under one scheduler).  The
// contexts exchange exactly like one-process-per-GPU ranks -- the same halo pack/unpack, mailbox
// and split-wave kernels -- but their peer pointers come from the sibling contexts (host allgather
// through this group) instead of CUDA IPC, and every step that consumes another rank's data is
// stage-serialised: each rank records an event after its producers, the ranks swap events through
// the group, and the consumer's stream waits for all of them.  No kernel ever spins on a rank whose
// producer has not been launched, so the ranks cannot deadlock on one GPU.
#pragma once
#include <condition_variable>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <vector>

namespace nekb200 {

struct LoopGroup {
    int nranks = 0;
    int transport = 0;          // 0: peer-memory kernels (the NVLink path); 1: staged (the NCCL-path kernels)
    double timeout_s = 60.0;    // a barrier that waits longer aborts the group (error, not a hang)
    std::mutex m;
    std::condition_variable cv;
    int arrived = 0;
    uint64_t generation = 0;
    bool aborted = false;
    std::vector<const void *> slot;   // per-rank host pointers published for an allgather
    std::vector<size_t> slot_bytes;

    // all ranks arrive; false on timeout or abort
    bool barrier();
    void abort();
    // every rank's `bytes` of `mine` into all[nranks * bytes] (rank order); false on failure
    bool allgather(int rank, const void *mine, size_t bytes, void *all);
};

constexpr char LOOP_TAG[8] = {'N', 'E', 'K', 'L', 'O', 'O', 'P', '1'};

inline LoopGroup *loop_group_of(const unsigned char id[128])
{
    if (std::memcmp(id, LOOP_TAG, 8) != 0) return nullptr;
    LoopGroup *g = nullptr;
    std::memcpy(&g, id + 8, sizeof(g));
    return g;
}

}  // namespace nekb200
