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
};

// apply_actions data movement (engine.hpp:686-716) for one layer: the rows of
// the tokens in one action list move between the device cache and the pinned,
// device-mapped host tier (same [B][Ncap][2][H][row] layout in both).
struct MoveParams {
    uint8_t* dev;        // layer base of the device cache
    uint8_t* host;       // layer base of the host tier (mapped pinned memory)
    const int* lists;    // [B][4][list_ld]
    const int* counts;   // [B][4]
    long long list_ld;
    long long tok_bytes; // 2*H*row bytes
    long long seq_bytes; // Ncap * tok_bytes
    int which;           // 0 offload (device -> host), 2 reload (host -> device),
                         // -1 both at once (blockIdx.z 0 / 1): the two PCIe directions overlap
    int poison;          // offload: overwrite the device row with 0xFF (NaN) afterwards
};

}  // namespace skvd
