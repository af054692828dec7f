// search_inst.cu — instantiates the search/eval kernels for one device count
// M (compiled once per M ∈ [1,8] with -DPP_M=M, in parallel).
#include "search_kernel.cuh"

#ifndef PP_M
#error "compile with -DPP_M=<1..8>"
#endif

#define PP_CAT2(a, b) a##b
#define PP_CAT(a, b) PP_CAT2(a, b)

namespace pp {

template <int GEN, bool MEM, bool WA>
static KernelInfo info() {
    return KernelInfo{&launch_search<PP_M, GEN, MEM, WA>,
                      reinterpret_cast<const void *>(&search_kernel<PP_M, GEN, MEM, WA>)};
}

KernelInfo PP_CAT(kernel_for_m, PP_M)(int gen, bool mem, bool wa) {
    switch (gen) {
        case GEN_GRAY:
            return mem ? (wa ? info<GEN_GRAY, true, true>() : info<GEN_GRAY, true, false>())
                       : (wa ? info<GEN_GRAY, false, true>() : info<GEN_GRAY, false, false>());
        case GEN_RANDOM:
            return mem ? (wa ? info<GEN_RANDOM, true, true>() : info<GEN_RANDOM, true, false>())
                       : (wa ? info<GEN_RANDOM, false, true>() : info<GEN_RANDOM, false, false>());
        case GEN_PERTURB:
            return mem ? (wa ? info<GEN_PERTURB, true, true>() : info<GEN_PERTURB, true, false>())
                       : (wa ? info<GEN_PERTURB, false, true>() : info<GEN_PERTURB, false, false>());
        default:
            return mem ? info<GEN_EXPLICIT, true, true>() : info<GEN_EXPLICIT, false, true>();
    }
}

UpdateFn PP_CAT(update_for_m, PP_M)(int gen) {
    switch (gen) {
        case GEN_GRAY: return &launch_update<PP_M, GEN_GRAY>;
        case GEN_RANDOM: return &launch_update<PP_M, GEN_RANDOM>;
        default: return &launch_update<PP_M, GEN_PERTURB>;
    }
}

}  // namespace pp
