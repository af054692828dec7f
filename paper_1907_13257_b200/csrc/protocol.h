// protocol.h — the cross-GPU argmin of one search round (SURVEY.md §8(e), row
// a8).  Rank r of R holds the lexicographic (makespan, index)
// argmin of its contiguous candidate slice [⌊r·n/R⌋, ⌊(r+1)·n/R⌋).  Two u64
// min all-reduces make every rank agree on the global argmin:
//
//   key_r   = (min(makespan, 2^61 − 1) << 3) | r      (UINT64_MAX: empty slice)
//   key     = min_r key_r                           → the winning makespan
//   idx_r   = local index if key_r has the winning makespan, else UINT64_MAX
//   idx     = min_r idx_r
//
// Every rank whose local argmin reaches the winning makespan contributes its
// index, so idx is the smallest global index with the minimum makespan: the
// result equals the single-GPU argmin for any rank count (R9), whatever the
// order of the slices' indices (the symmetry-reduced GRAY search reports
// Gray indices that are not ordered by rank).  Feasible makespans are < 2^61
// (pp_load_dfg), so the clamp only maps the infeasible sentinel to 2^61 − 1.
//
// The functions below are the protocol's only definition: the device kernels
// (projection.cu, search_kernel.cuh round_update_kernel), the NCCL driver
// (capi.cpp) and the host entry points exported for multi-process tests
// (pp_round_exchange_host, pp_round_key, …) all call them, and the exchange
// sequence itself is the template `exchange`, instantiated once with an NCCL
// executor (device scalars, stream-ordered) and once with a host executor
// (a caller-supplied all-reduce callback, e.g. torch.distributed over gloo).
#pragma once
#include <stdint.h>

#ifdef __CUDACC__
#define PP_HD __host__ __device__ __forceinline__
#else
#define PP_HD inline
#endif

namespace pp {
namespace proto {

constexpr uint64_t kNone = ~0ull;                    // no candidate / empty slice
constexpr uint64_t kKeyCap = (1ull << 61) - 1;       // clamp of the infeasible sentinel

PP_HD uint64_t key(uint64_t makespan, uint64_t index, int rank) {
    if (index == kNone) return kNone;                 // an empty slice never wins
    return ((makespan < kKeyCap ? makespan : kKeyCap) << 3) | (uint64_t)(rank & 7);
}
PP_HD int key_rank(uint64_t key) { return (int)(key & 7); }
PP_HD uint64_t key_makespan(uint64_t key) {
    if (key == kNone) return kNone;
    const uint64_t m = key >> 3;
    return m == kKeyCap ? kNone : m;
}
// this rank's contribution to the index all-reduce: its local argmin index
// iff its key carries the winning (clamped) makespan
PP_HD uint64_t contrib(uint64_t key_global, uint64_t key_local, uint64_t local_index) {
    return (key_global != kNone && key_local != kNone && (key_local >> 3) == (key_global >> 3)) ? local_index
                                                                                                : kNone;
}
// the PERTURB base moves to the round winner iff the winner is strictly better
// than the base: candidate 0 is the base, so (lexicographic argmin) the winner
// is strictly better exactly when its index is not 0 (O7)
PP_HD bool moves_base(uint64_t win_index) { return win_index != 0 && win_index != kNone; }

// Scalar slots the exchange reads and writes (internal.h ScalarSlot order).
enum : int { LOCAL_MK = 0, LOCAL_IDX = 1, KEY_LOCAL = 2, KEY_GLOBAL = 3, IDX_LOCAL = 4, IDX_GLOBAL = 5 };

// The exchange sequence.  Ex provides pack() (KEY_LOCAL ← key(LOCAL_MK,
// LOCAL_IDX, rank)), contrib() (IDX_LOCAL ← contrib(KEY_GLOBAL, KEY_LOCAL,
// LOCAL_IDX)) and allreduce_min(src, dst) (dst ← min over ranks of src); each
// returns 0 or a PP_E_* code.
template <class Ex>
int exchange(Ex &ex) {
    int rc;
    if ((rc = ex.pack())) return rc;
    if ((rc = ex.allreduce_min(KEY_LOCAL, KEY_GLOBAL))) return rc;
    if ((rc = ex.contrib())) return rc;
    return ex.allreduce_min(IDX_LOCAL, IDX_GLOBAL);
}

}  // namespace proto
}  // namespace pp
