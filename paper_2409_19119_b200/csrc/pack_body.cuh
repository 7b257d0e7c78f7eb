// pack_body.cuh -- one halo send slot of the NVLink peer-memory exchange (shared by the pack kernel of
// gs.cu and the queue-mode Ax kernel of ax.cu): the interface run's local copies folded in canonical
// order (reading 7), the partial kept for the unpack, and the value stored straight into the
// neighbour's receive buffer half of this epoch's parity.
#pragma once

namespace nekb200 {

template <class T>
__device__ __forceinline__ void pack_slot(int64_t sidx, const int32_t *__restrict__ perm,
                                          const int32_t *__restrict__ offs, const T *__restrict__ v,
                                          T *__restrict__ partial, const int32_t *__restrict__ send_run,
                                          const int32_t *__restrict__ slot_nbr, double *const *peer_recv,
                                          const int64_t *__restrict__ remote_off,
                                          const int64_t *__restrict__ send_offs,
                                          const int64_t *__restrict__ remote_half, int nnbr, int64_t par,
                                          const int4 *__restrict__ pack4)
{
    // the slot lists are read every iteration next to the streamed metric factors: keep them in L2
    const uint64_t keep = tma::policy_evict_last();
    const int run = (int)tma::ldu(reinterpret_cast<const uint32_t *>(send_run) + sidx, keep);
    T s;
    const int4 c4 = pack4 ? tma::ldi4(pack4 + sidx, keep) : make_int4(-2, -1, -1, -1);
    if (c4.x >= 0) {                     // <= 4 local copies, listed per slot (one dependent level)
        s = v[c4.x];
        if (c4.y >= 0) s += v[c4.y];
        if (c4.z >= 0) s += v[c4.z];
        if (c4.w >= 0) s += v[c4.w];
    } else {
        const int o0 = offs[run], o1 = offs[run + 1];
        s = v[perm[o0]];
        for (int c = o0 + 1; c < o1; ++c) s += v[perm[c]];
    }
    partial[run] = s;
    const int k = (int)tma::ldu(reinterpret_cast<const uint32_t *>(slot_nbr) + sidx, keep);
    NEK_CHECK(k >= 0 && k < nnbr && sidx >= send_offs[k] && sidx < send_offs[k + 1] && remote_off[k] >= 0 &&
              remote_off[k] + (sidx - send_offs[k]) < remote_half[k]);
    reinterpret_cast<T *>(peer_recv[k])[par * remote_half[k] + remote_off[k] + (sidx - send_offs[k])] = s;
}

}  // namespace nekb200
