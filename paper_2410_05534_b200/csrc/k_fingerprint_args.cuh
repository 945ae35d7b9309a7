// Launch arguments of k_fingerprint (K12, EGraph.fingerprint).
#pragma once
#include <cstdint>

namespace esat {



struct FArgs {
    const uint32_t* krank;       // [n_syms] rank of symbol.key() among all keys (Python tuple order)
    const uint32_t* key_off;     // [n_syms+1] offsets of repr(symbol.key()) in key_bytes
    const uint8_t* key_bytes;
    unsigned long long *lab0, *lab1;   // [node rows] labels by class position (double buffer)
    uint32_t *rep0, *rep1;       // [node rows] partition representative (double buffer)
    uint32_t* nord;              // [node rows] nodes of each class in description order
    uint8_t* lchg;               // [node rows] class label changed in the last round
    unsigned long long *dec0, *dec1;   // [4 x node rows] decimal repr of each label (3 words + length; double buffer)
    unsigned long long* tkey;    // [table rows] label -> smallest class position
    uint32_t *tval, *cord;       // [table rows]
    unsigned long long* fp;      // [L]
    uint32_t* status;            // [L] 0 ok
};

template <int T> __global__ void k_fingerprint(Dev, FArgs);

}  // namespace esat
