// search_inst.cu — instantiates the search/eval kernels for one device count
// M (compiled once per M ∈ [1,8] with -DPP_M=M, in parallel).
#include "search_kernel.cuh"

#ifndef PP_M
#error "compile with -DPP_M=<1..8>"
#endif

#define PP_CAT2(a, b) a##b
#define PP_CAT(a, b) PP_CAT2(a, b)

namespace pp {

template <int GEN, bool MEM, bool WA, bool F64, int NP>
static KernelInfo info1() {
    return KernelInfo{&launch_search<PP_M, GEN, MEM, WA, F64, NP>,
                      reinterpret_cast<const void *>(&search_kernel<PP_M, GEN, MEM, WA, F64, NP>)};
}

// placements per lane: 1, 2 or 4 for the argmin (search) kernels; the
// write-all (per-candidate output) kernels are built for NP = 2 only
template <int GEN, bool MEM, bool WA, bool F64>
static KernelInfo info_np(int np) {
    if (WA) return info1<GEN, MEM, WA, F64, 2>();
    if (np >= 4) return info1<GEN, MEM, WA, F64, 4>();
    if (np == 2) return info1<GEN, MEM, WA, F64, 2>();
    return info1<GEN, MEM, WA, F64, 1>();
}

template <int GEN, bool MEM, bool WA>
static KernelInfo info_f(bool f64, int np) {
    return f64 ? info_np<GEN, MEM, WA, true>(np) : info_np<GEN, MEM, WA, false>(np);
}

KernelInfo PP_CAT(kernel_for_m, PP_M)(int gen, bool mem, bool wa, bool f64, int np) {
    switch (gen) {
        case GEN_GRAY:
            return mem ? (wa ? info_f<GEN_GRAY, true, true>(f64, np) : info_f<GEN_GRAY, true, false>(f64, np))
                       : (wa ? info_f<GEN_GRAY, false, true>(f64, np) : info_f<GEN_GRAY, false, false>(f64, np));
        case GEN_RANDOM:
            return mem ? (wa ? info_f<GEN_RANDOM, true, true>(f64, np) : info_f<GEN_RANDOM, true, false>(f64, np))
                       : (wa ? info_f<GEN_RANDOM, false, true>(f64, np) : info_f<GEN_RANDOM, false, false>(f64, np));
        case GEN_PERTURB:
            return mem ? (wa ? info_f<GEN_PERTURB, true, true>(f64, np) : info_f<GEN_PERTURB, true, false>(f64, np))
                       : (wa ? info_f<GEN_PERTURB, false, true>(f64, np) : info_f<GEN_PERTURB, false, false>(f64, np));
        default:
            return mem ? info_f<GEN_EXPLICIT, true, true>(f64, np) : info_f<GEN_EXPLICIT, false, true>(f64, np);
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
