// eft.cu — SURVEY.md §8(f) f4: the earliest-finish-time greedy placement used
// as a PERTURB base seed (SPEC.md:245–253 heuristic_place; reading R23 in
// DESIGN.md §13).  Forward ops in π order; lane m < M prices device m (data
// ready over the op's in-arcs with this placement's delays, then the device's
// free time, then Δf), the warp takes the smallest finish (ties → smaller m).
// A device whose memory would exceed the cap is skipped.
// Sequential in K by construction: one warp, state in shared memory; the EFT
// image is first copied into shared memory when it fits (the op loop then
// reads no global memory: 245 → ~40 µs for the Inception-shaped DFG).
#include <cuda_runtime.h>

#include <cstdint>

#include "internal.h"

namespace pp {

struct EftParams {
    const uint8_t *g_gimage;
    uint8_t *g_out;          // [K] placement by π position
    int *g_status;           // 0 ok, 1 no memory-feasible device
    uint64_t cap;
    uint32_t K, off_arc, off_rows, off_cls, gcls;
    uint32_t g_bytes;        // image bytes (multiple of 16) staged into shared memory, 0 = read from global
    int M;
};

__global__ void __launch_bounds__(32) eft_kernel(const EftParams P) {
    extern __shared__ __align__(16) uint8_t smem[];
    const uint32_t m = threadIdx.x;
    const uint8_t *img = P.g_gimage;
    if (P.g_bytes) {   // stage the image (16-B words, one warp)
        for (uint32_t o = 16 * m; o < P.g_bytes; o += 16 * 32)
            *reinterpret_cast<uint4 *>(smem + o) = __ldg(reinterpret_cast<const uint4 *>(P.g_gimage + o));
        __syncwarp();
        img = smem;
    }
    uint64_t *fin = reinterpret_cast<uint64_t *>(smem + P.g_bytes);
    uint8_t *dev = smem + P.g_bytes + 8ull * P.K;
    const GOp *ops = reinterpret_cast<const GOp *>(img);
    const GArc *arcs = reinterpret_cast<const GArc *>(img + P.off_arc);
    const uint64_t *rows = reinterpret_cast<const uint64_t *>(img + P.off_rows);
    const uint8_t *cls = img + P.off_cls;
    constexpr uint64_t kNone = ~0ull;
    uint64_t free_t = 0, used = 0;
    int status = 0;
    for (uint32_t p = 0; p < P.K; p++) {
        const GOp op = ops[p];
        uint64_t f = kNone;
        if ((int)m < P.M && !(P.cap > 0 && used + op.mem > P.cap)) {
            uint64_t r = 0;
            for (uint32_t a = 0; a < op.in_cnt; a++) {
                const GArc arc = arcs[op.in_begin + a];
                const uint64_t t = fin[arc.u] + rows[(uint64_t)arc.row * P.gcls + cls[dev[arc.u] * 8 + m]];
                r = t > r ? t : r;
            }
            f = (r > free_t ? r : free_t) + op.fwd;
        }
        uint64_t bf = f;
        uint32_t bm = m;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const uint64_t of = __shfl_xor_sync(0xffffffffu, bf, o);
            const uint32_t om = __shfl_xor_sync(0xffffffffu, bm, o);
            if (of < bf || (of == bf && om < bm)) { bf = of; bm = om; }
        }
        if (bf == kNone) { status = 1; break; }
        if (m == 0) {
            dev[p] = (uint8_t)bm;
            fin[p] = bf;
        }
        if (m == bm) {
            free_t = bf;
            used += op.mem;
        }
        __syncwarp();
    }
    __syncwarp();
    if (status == 0)
        for (uint32_t p = m; p < P.K; p += 32) P.g_out[p] = dev[p];
    if (m == 0) *P.g_status = status;
}

int launch_eft(const pp_dfg *g, int M, uint8_t *d_out, int *d_status, void *stream) {
    EftParams p{};
    p.g_gimage = g->d_gimage;
    p.g_out = d_out;
    p.g_status = d_status;
    p.cap = g->cap;
    p.K = (uint32_t)g->K;
    p.off_arc = g->g_off_arc;
    p.off_rows = g->g_off_rows;
    p.off_cls = g->g_off_cls;
    p.gcls = g->gcls;
    p.M = M;
    const size_t state = 9ull * g->K + 16;
    p.g_bytes = ((size_t)g->g_bytes + 15) / 16 * 16 + state <= 200 * 1024 ? ((g->g_bytes + 15) / 16 * 16) : 0;
    const size_t smem = p.g_bytes + state;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(eft_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return (int)e;
    }
    eft_kernel<<<1, 32, smem, (cudaStream_t)stream>>>(p);
    return (int)cudaGetLastError();
}

}  // namespace pp
