// search_inst.cu — instantiates the search/eval kernels for one device count
// M (compiled once per M ∈ [1,8] with -DPP_M=M, in parallel).
#include "exact_kernel.cuh"
#include "search_kernel.cuh"

#ifndef PP_M
#error "compile with -DPP_M=<1..8>"
#endif

#define PP_CAT2(a, b) a##b
#define PP_CAT(a, b) PP_CAT2(a, b)

namespace pp {

template <int GEN, bool MEM, bool WA, bool F64, int NP, bool HW>
static KernelInfo info2() {
    return KernelInfo{&launch_search<PP_M, GEN, MEM, WA, F64, NP, HW>,
                      reinterpret_cast<const void *>(&search_kernel<PP_M, GEN, MEM, WA, F64, NP, HW>)};
}

// the hardware-graph variant exists for the tagged-f64 arithmetic and M ≥ 2
template <int GEN, bool MEM, bool WA, bool F64, int NP>
static KernelInfo info1(bool hw) {
    constexpr bool kHw = F64 && PP_M >= 2;
    if (kHw && hw) return info2<GEN, MEM, WA, F64, NP, kHw>();
    return info2<GEN, MEM, WA, F64, NP, false>();
}

// placements per lane: 1, 2 or 4 for the argmin (search) kernels; the
// write-all (per-candidate output) kernels are built for NP = 2 only
template <int GEN, bool MEM, bool WA, bool F64>
static KernelInfo info_np(int np, bool hw) {
    if (WA) return info1<GEN, MEM, WA, F64, 2>(hw);
    if (np >= 4) return info1<GEN, MEM, WA, F64, 4>(hw);
    if (np == 2) return info1<GEN, MEM, WA, F64, 2>(hw);
    return info1<GEN, MEM, WA, F64, 1>(hw);
}

// The shared-memory tier runs the tagged-f64 arithmetic only: a DFG whose
// time bound needs tagged u64 (≥ 2^49 ps) is placed on the global-state tier
// at load time (loader.cpp), so f64 is always true here.
template <int GEN, bool MEM, bool WA>
static KernelInfo info_f(bool, int np, bool hw) {
    return info_np<GEN, MEM, WA, true>(np, hw);
}

template <int GEN>
static KernelInfo info_gen(bool mem, bool wa, bool f64, int np, bool hw) {
    if (mem) return wa ? info_f<GEN, true, true>(f64, np, hw) : info_f<GEN, true, false>(f64, np, hw);
    return wa ? info_f<GEN, false, true>(f64, np, hw) : info_f<GEN, false, false>(f64, np, hw);
}

// GEN_SYM (the symmetry-reduced exhaustive GRAY search) runs only as an
// argmin on the uniform link model
template <bool MEM, bool F64>
static KernelInfo info_sym_np(int np) {
    if constexpr (PP_M == 3) {   // M = 3: a lane takes the 3 values of the last position
        if (np == 3) return info2<GEN_SYM, MEM, false, F64, 3, false>();
    }
    if (np >= 4) return info2<GEN_SYM, MEM, false, F64, 4, false>();
    if (np == 2) return info2<GEN_SYM, MEM, false, F64, 2, false>();
    return info2<GEN_SYM, MEM, false, F64, 1, false>();
}
template <bool MEM>
static KernelInfo info_sym(bool, int np) {
    return info_sym_np<MEM, true>(np);
}

// the record-prefetch variants of the PERTURB argmin kernels (M = 2: the
// cut-word schedule, M = 4, 8: the device-word schedule; RP)
template <bool MEM, int NP>
static KernelInfo info_rp() {
    return KernelInfo{&launch_search<PP_M, GEN_PERTURB, MEM, false, true, NP, false, true>,
                      reinterpret_cast<const void *>(&search_kernel<PP_M, GEN_PERTURB, MEM, false, true, NP, false, true>)};
}
KernelInfo PP_CAT(rp_kernel_for_m, PP_M)(bool mem, int np) {
    if constexpr (PP_M == 2 || PP_M == 4 || PP_M == 8) {
        if (np >= 4) return mem ? info_rp<true, 4>() : info_rp<false, 4>();
        if (np == 2) return mem ? info_rp<true, 2>() : info_rp<false, 2>();
        return mem ? info_rp<true, 1>() : info_rp<false, 1>();
    }
    return KernelInfo{nullptr, nullptr};
}

KernelInfo PP_CAT(kernel_for_m, PP_M)(int gen, bool mem, bool wa, bool f64, int np, bool hw) {
    switch (gen) {
        case GEN_SYM: return mem ? info_sym<true>(f64, np) : info_sym<false>(f64, np);
        case GEN_GRAY: return info_gen<GEN_GRAY>(mem, wa, f64, np, hw);
        case GEN_RANDOM: return info_gen<GEN_RANDOM>(mem, wa, f64, np, hw);
        case GEN_PERTURB: return info_gen<GEN_PERTURB>(mem, wa, f64, np, hw);
        default:
            return mem ? info_f<GEN_EXPLICIT, true, true>(f64, np, hw) : info_f<GEN_EXPLICIT, false, true>(f64, np, hw);
    }
}

template <int GEN, bool F64>
static KernelInfo big_info() {
    return KernelInfo{&launch_search_big<PP_M, GEN, F64>,
                      reinterpret_cast<const void *>(&search_big_kernel<PP_M, GEN, F64>)};
}
template <bool F64>
static KernelInfo big_gen(int gen) {
    switch (gen) {
        case GEN_GRAY: return big_info<GEN_GRAY, F64>();
        case GEN_RANDOM: return big_info<GEN_RANDOM, F64>();
        case GEN_PERTURB: return big_info<GEN_PERTURB, F64>();
        default: return big_info<GEN_EXPLICIT, F64>();
    }
}
KernelInfo PP_CAT(big_for_m, PP_M)(int gen, bool f64) { return f64 ? big_gen<true>(gen) : big_gen<false>(gen); }

UpdateFn PP_CAT(update_for_m, PP_M)(int gen) {
    switch (gen) {
        case GEN_GRAY: return &launch_update<PP_M, GEN_GRAY>;
        case GEN_RANDOM: return &launch_update<PP_M, GEN_RANDOM>;
        default: return &launch_update<PP_M, GEN_PERTURB>;
    }
}

template <int GEN>
static XKernelInfo xinfo() {
    return XKernelInfo{&launch_exact<PP_M, GEN>, reinterpret_cast<const void *>(&exact_kernel<PP_M, GEN>)};
}

XKernelInfo PP_CAT(exact_for_m, PP_M)(int gen) {
    switch (gen) {
        case GEN_GRAY: return xinfo<GEN_GRAY>();
        case GEN_SYM: return xinfo<GEN_SYM>();
        case GEN_RANDOM: return xinfo<GEN_RANDOM>();
        case GEN_PERTURB: return xinfo<GEN_PERTURB>();
        default: return xinfo<GEN_EXPLICIT>();
    }
}

}  // namespace pp
