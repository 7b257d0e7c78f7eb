// loopback.cpp -- host side of the loopback group (loopback.h) and its ABI (nek_loopback_*).
#include "loopback.h"

#include <chrono>
#include <cstdlib>
#include <new>

#include "nek.h"

namespace nekb200 {

bool LoopGroup::barrier()
{
    std::unique_lock<std::mutex> lk(m);
    if (aborted) return false;
    const uint64_t gen = generation;
    if (++arrived == nranks) {
        arrived = 0;
        ++generation;
        cv.notify_all();
        return true;
    }
    const bool ok = cv.wait_for(lk, std::chrono::duration<double>(timeout_s),
                                [&] { return generation != gen || aborted; });
    if (!ok || aborted) {
        aborted = true;
        cv.notify_all();
        return false;
    }
    return true;
}

void LoopGroup::abort()
{
    std::lock_guard<std::mutex> lk(m);
    aborted = true;
    cv.notify_all();
}

bool LoopGroup::allgather(int rank, const void *mine, size_t bytes, void *all)
{
    {
        std::lock_guard<std::mutex> lk(m);
        slot[rank] = mine;
        slot_bytes[rank] = bytes;
    }
    if (!barrier()) return false;
    bool same = true;
    for (int q = 0; q < nranks; ++q) {
        same &= slot_bytes[q] == bytes;
        if (same) std::memcpy(static_cast<char *>(all) + (size_t)q * bytes, slot[q], bytes);
    }
    if (!barrier()) return false;   // nobody republishes before every rank has copied
    if (!same) abort();
    return same;
}

}  // namespace nekb200

struct nek_loopback {
    nekb200::LoopGroup g;
};

extern "C" {

int nek_loopback_create(int nranks, int transport, nek_loopback **out)
{
    if (!out || nranks < 1 || nranks > 64 || (transport != 0 && transport != 1)) return NEK_EINVAL;
    nek_loopback *lb = new (std::nothrow) nek_loopback();
    if (!lb) return NEK_ENOMEM;
    lb->g.nranks = nranks;
    lb->g.transport = transport;
    lb->g.slot.assign(nranks, nullptr);
    lb->g.slot_bytes.assign(nranks, 0);
    if (const char *e = std::getenv("NEK_LOOPBACK_TIMEOUT_S")) lb->g.timeout_s = std::atof(e);
    *out = lb;
    return NEK_OK;
}

int nek_loopback_comm(nek_loopback *lb, int rank, nek_comm *comm)
{
    if (!lb || !comm || rank < 0 || rank >= lb->g.nranks) return NEK_EINVAL;
    std::memset(comm, 0, sizeof(*comm));
    comm->rank = rank;
    comm->nranks = lb->g.nranks;
    std::memcpy(comm->nccl_id, nekb200::LOOP_TAG, 8);
    nekb200::LoopGroup *g = &lb->g;
    std::memcpy(comm->nccl_id + 8, &g, sizeof(g));
    return NEK_OK;
}

int nek_loopback_abort(nek_loopback *lb)
{
    if (!lb) return NEK_EINVAL;
    lb->g.abort();
    return NEK_OK;
}

int nek_loopback_free(nek_loopback *lb)
{
    delete lb;
    return NEK_OK;
}

}  // extern "C"
