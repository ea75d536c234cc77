// common.cuh -- shared definitions for the sm_100a sFFT-DT kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "cx.cuh"
#include "../../include/sfdt.h"

namespace sfdt {

constexpr double TINY = 2.2250738585072014e-308;   // np.finfo(float).tiny
constexpr double SINGULARITY_RTOL = 1e-10;         // syndrome.py:23
constexpr double CONSISTENCY_RTOL = 1e-6;          // exact.py:26
constexpr double SNAP_TOL = 0.25;                  // exact.py:27
constexpr double UNIT_MODULUS_TOL = 1e-6;          // exact.py:28
constexpr double TWO_PI = 6.283185307179586;       // 2.0 * np.pi
constexpr int MAX_SHIFTS = 8;                      // 2 * a_max, a_max <= 4
constexpr int FFT_SMEM_MAX = 8192;                 // complex128 points per CTA in smem

__device__ __forceinline__ cx ldcx(const cx *p) {
    double2 v = __ldg(reinterpret_cast<const double2 *>(p));
    return mk(v.x, v.y);
}
__device__ __forceinline__ void stcx(cx *p, cx v) {
    *reinterpret_cast<double2 *>(p) = make_double2(v.re, v.im);
}

__host__ __device__ __forceinline__ int ilog2_64(int64_t v) {
    int r = 0;
    while ((int64_t(1) << (r + 1)) <= v) r++;
    return r;
}

// Grid of a grid-stride worklist kernel: `cap` CTAs fill the GPU, but a
// small batch (config 1: 256 bins) must not launch a thousand idle CTAs --
// the worklist never exceeds max_items, so no more CTAs than it needs.
static inline unsigned wl_grid(int64_t max_items, int items_per_cta, int64_t cap) {
    int64_t g = (max_items + items_per_cta - 1) / items_per_cta;
    if (g > cap) g = cap;
    return (unsigned)(g < 1 ? 1 : g);
}

// CTAs of `kernel` resident on the whole GPU at once.  Grid-stride kernels
// whose items are a few long serial chains (the multi-collision decodes and
// pursuits) must not be launched in several waves: a later wave's chains
// would only start when the earlier wave's longest chain ends.
template <typename K>
static inline int64_t one_wave(K kernel, int threads, size_t smem = 0) {
    int dev = 0, sms = 148, per = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kernel, threads, smem) != cudaSuccess || per < 1)
        per = 1;
    return (int64_t)sms * per;
}

// python-style non-negative modulo for power-of-two n
__host__ __device__ __forceinline__ int64_t pmod(int64_t a, int64_t n) { return a & (n - 1); }

// Programmatic dependent launch: a kernel launched with launch_pdl may be
// scheduled while its predecessor in the stream is still running; it must
// call pdl_wait() before touching memory the predecessor writes (every
// kernel of a PDL chain calls it first thing, so the semantics stay those of
// stream order -- only the launch latency between kernels overlaps).  A
// no-op when the kernel was launched normally.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }

template <typename... KArgs, typename... Args>
static inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                                     cudaStream_t stream, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, args...);
}

// the measured-best design decisions (sfdt_tuning, include/sfdt.h)
static inline sfdt_tuning default_tuning() {
    sfdt_tuning t;
    t.fft_split = 0;
    t.gen_dedup = 1;
    t.gen_svd_closed = 1;
    t.gen_mf_small = 1;
    t.gen_mf_list = 0;
    t.gen_warp = -1;
    t.gen_split_a = 3;
    t.gen_prune_lanes = 0;
    t.gen_deal = 8;
    t.decode_coop = -1;
    t.latency_path = -1;
    t.gen_window = -1;
    return t;
}
static inline sfdt_tuning tuning_or_default(const sfdt_tuning *t) { return t ? *t : default_tuning(); }

}  // namespace sfdt

#define SFDT_CHECK_LAUNCH()                                   \
    do {                                                      \
        if (cudaPeekAtLastError() != cudaSuccess) return SFDT_ECUDA; \
    } while (0)
