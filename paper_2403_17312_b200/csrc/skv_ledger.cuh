// skv_ledger.cuh -- per-step KV residency bookkeeping on device.
//
// Device form of the reference's token-granular ledger and the per-step
// action sets of the three-phase schedule:
//   * KvLedger tiers (memsim.hpp:72-215): one u8 per (layer, sequence, token):
//     0 Device, 1 Host, 2 Deleted, 255 not stored;
//   * step_actions (scheduler.hpp:320-381): offload the oldest device tokens
//     outside the local window until the host tier holds ceil(alpha*existing);
//     in Phase III delete the oldest ceil(beta*host_after) host tokens; selected
//     tokens that are host-resident or just offloaded are reloaded, deleted ones
//     recomputed; the current token (not yet stored) is skipped;
//   * apply_actions (engine.hpp:686-716) on the tiers.
// One CTA per sequence; every list is built with order-preserving block scans,
// so the lists are exactly the reference's (ascending / selection order).
#pragma once

#include "skv_topk.cuh"

namespace skvd {

constexpr int kLedgerThreads = 256;
enum : uint8_t { kTierDevice = 0, kTierHost = 1, kTierDeleted = 2, kTierAbsent = 255 };

// Device-side status of a cache, in mapped pinned host memory: the first
// ledger failure (KvLedger's OutOfDeviceMemory, memsim.hpp:193-200) or
// residency violation (engine.hpp:625-628) seen by a kernel. The host
// reports it from the next entry point (sticky).
struct DevStatus {
    int code;          // 0 ok, 2 OOM (SKV_ERR_OOM), 1 residency (SKV_ERR_CONTRACT)
    int layer;
    int seq;
    int token;
    long long step;
    unsigned long long needed;    // bytes the failing mutation needed (reference message)
    unsigned long long capacity;  // bytes
};

// Byte totals of the KvLedger (memsim.hpp:77-215) over every layer and
// sequence, in tokens of tok_bytes each (device memory).
struct LedgerTotals {
    unsigned long long dev_tokens, host_tokens, peak_dev_tokens;
    unsigned long long exhausted;  // failed slot allocations of the running layer-step (paged)
    unsigned long long moved[4];   // cumulative rows offloaded, deleted, reloaded, recomputed
    unsigned long long kept;       // cumulative reloads of rows offloaded in the same step (no copy in)
};

__device__ __forceinline__ void report_status_inl(DevStatus* st, int code, int layer, int seq, int token, long long step,
                                              unsigned long long needed, unsigned long long cap) {
    if (st == nullptr) return;
    if (atomicCAS(&st->code, 0, -1) == 0) {  // first failure wins
        st->layer = layer;
        st->seq = seq;
        st->token = token;
        st->step = step;
        st->needed = needed;
        st->capacity = cap;
        __threadfence_system();
        atomicExch(&st->code, code);
    }
}
// Out of line for the attend kernel (a cold path that must not cost it
// registers); kernels with room call report_status_inl.
static __device__ __noinline__ void report_status(DevStatus* st, int code, int layer, int seq, int token, long long step,
                                              unsigned long long needed, unsigned long long cap) {
    report_status_inl(st, code, layer, seq, token, step, needed, cap);
}

// Paged store: every (layer, sequence) owns `pcap` token slots of the pool;
// slot[t] maps token t to its slot (-1: not on device) and a FIFO ring of
// free slots (fq, head/tail counters) hands them out. Frees of a step go to
// the tail, allocations come from the head, so a slot freed by this step's
// offload is reused only when the older free slots run out ("recycled").
struct PagedSlots {
    int* slot;          // [B][slot_ld] token -> slot, -1 none
    long long slot_ld;  // Ncap
    int* fq;            // [B][pcap] free ring
    unsigned* fq_ht;    // [B][2] head, tail (monotonic)
    int pcap;
};

// A layer of the cache as the write / read kernels see it.
struct CacheView {
    uint8_t* kv;         // layer base: [B][kv_ncap][2][H][row]
    int Ncap;            // token stride of importance / tiers / slot rows
    int kv_ncap;         // token (slot) stride of the K/V storage: Ncap, or pcap when paged
    int* slot;           // paged: [B][Ncap] token -> slot (nullptr: slot = token)
    unsigned* fq_ht;     // paged: [B][2] FIFO (head, free count)
    LedgerTotals* tot;   // ledger totals (store_new accounting), nullable
};

struct LedgerParams {
    uint8_t* tiers;  // [B][tier_ld]
    long long tier_ld;
    const int* sel;  // [B][sel_ld] ascending selection of this step (SparseSelection::all)
    long long sel_ld;
    int m, k;
    int existing;      // tokens stored before this step (input_len + j)
    int phase;         // phase_of_step (scheduler.hpp:52-60), host-computed
    long long target;  // ceil(alpha * existing), host-computed in double
    double beta;
    int* lists;        // [B][4][list_ld]: offload, delete, reload, recompute
    long long list_ld;
    int* counts;       // [B][4]
    int apply;         // update tiers (apply_actions)
    int store_current; // mark token `existing` stored on device afterwards (store_new)
    // paged store (slot.slot != nullptr): slots freed / allocated with the tiers
    PagedSlots slots;
    int* act_slots;    // [B][4][list_ld] slot of each list entry (offload: source, reload/recompute: destination)
    int* aux;          // [B][4]: [0] reload-list index from which destinations are recycled slots
    // KvLedger byte accounting (apply only; tot nullptr: none)
    LedgerTotals* tot;
    unsigned* arrive;  // this layer's arrival counter (0 between launches)
    unsigned long long* layer_allocs;  // this layer's allocation count accumulator (0 between launches)
    unsigned long long cap_bytes, tok_bytes;
    unsigned long long cap_tokens;  // floor(cap_bytes / tok_bytes), host-computed (no 64-bit division on device)
    int layer;
    long long step;
    DevStatus* status;
};

// apply_actions data movement (engine.hpp:686-716) for one layer: the rows of
// the tokens in one action list move between the device cache and the pinned,
// device-mapped host tier ([B][Ncap][2][H][row] on the host; the device side
// is the same layout, or the paged pool [B][pcap] addressed by slot).
struct MoveParams {
    uint8_t* dev;        // layer base of the device cache / pool
    uint8_t* host;       // layer base of the host tier (mapped pinned memory)
    const int* lists;    // [B][4][list_ld]
    const int* counts;   // [B][4]
    const int* act_slots;  // [B][4][list_ld] device slots (paged), nullptr: slot = token
    const int* aux;      // [B][4] reload split (paged)
    long long list_ld;
    long long tok_bytes; // 2*H*row bytes
    long long seq_bytes; // Ncap * tok_bytes (host tier)
    long long dev_seq_bytes;  // pcap * tok_bytes (device side)
    int which;           // 0 offload (device -> host), 2 reload (host -> device),
                         // -1 both at once (blockIdx.z 0 / 1): the two PCIe directions overlap
    int second;          // paged: 0 = offloads + reloads before the split, 1 = reloads from the split on
    int poison;          // offload: overwrite the device row with 0xFF (NaN) afterwards
};

}  // namespace skvd
