// Event-timed launches of the real multi-collision decode kernels
// (k_decode_multi / k_decode_coop of csrc/exact.cu) on a synthetic worklist:
// `nb` bins with a = `acol` collisions each, one signal of L = 256 bins.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -std=c++17 \
//        -o tools/decode_kernels tools/decode_kernels.cu && tools/decode_kernels
#include <cstdio>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>

__device__ long long g_clk[64];
#define SFDT_COOP_CLK(i) do { if ((threadIdx.x & 31) == 0 && blockIdx.x == 0) g_clk[(threadIdx.x >> 5) * 8 + i] = clock64(); } while (0)
#include "../paper_1407_8315_b200/csrc/exact.cu"

static void fill_bin(std::vector<double> &V, int64_t L, int64_t k, int a, int64_t n) {
    for (int j = 0; j < a; j++) {
        const int64_t loc = k + L * (int64_t)(17 + 211 * j);
        const double mag = 1.0 + 2.0 * j, ph = 0.3 + j;
        for (int l = 0; l < 8; l++) {
            const double th = 2 * M_PI * (double)((loc * l) % n) / (double)n;
            V[2 * (l * L + k)] += mag * cos(th + ph);
            V[2 * (l * L + k) + 1] += mag * sin(th + ph);
        }
    }
}

int main() {
    const int64_t n = 1 << 16, L = 256;
    for (int acol = 2; acol <= 5; acol++)
        for (int nb : {1, 8}) {
            std::vector<double> V(2 * 8 * L, 0.0);
            std::vector<int64_t> wl(L, 0);
            // one bin with acol collisions (first in the list), the rest a = 2
            for (int i = 0; i < nb; i++) { wl[i] = 5 + 7 * i; fill_bin(V, L, wl[i], i == 0 ? acol : 2, n); }
            cx *dV; int64_t *dwl, *dwl2, *bloc; cx *bval; uint8_t *st; unsigned long long *cnt;
            cudaMalloc(&dV, V.size() * 8); cudaMalloc(&dwl, L * 8); cudaMalloc(&dwl2, L * 8);
            cudaMalloc(&bloc, L * 4 * 8); cudaMalloc(&bval, L * 4 * 16); cudaMalloc(&st, L); cudaMalloc(&cnt, 64);
            cudaMemcpy(dV, V.data(), V.size() * 8, cudaMemcpyHostToDevice);
            cudaMemcpy(dwl, wl.data(), L * 8, cudaMemcpyHostToDevice);
            unsigned long long c[2] = {(unsigned long long)nb, 0};
            cudaMemcpy(cnt, c, 16, cudaMemcpyHostToDevice);
            cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
            float ms;
            for (int variant = 0; variant < 4; variant++) {
                float best = 1e9f;
                for (int rep = 0; rep < 5; rep++) {
                    cudaMemset(cnt + 1, 0, 8);
                    cudaEventRecord(e0);
                    if (variant == 0)
                        k_decode_multi<8><<<2, 128>>>(dV, L, 4, 4, n, st, bloc, bval, dwl, cnt, dwl2, cnt + 1);
                    else
                        k_decode_coop<8><<<64, 32 * variant>>>(dV, L, 4, 2, n, st, bloc, bval, dwl, cnt);
                    cudaEventRecord(e1);
                    cudaEventSynchronize(e1);
                    cudaEventElapsedTime(&ms, e0, e1);
                    if (ms < best) best = ms;
                }
                uint8_t hs[256];
                cudaMemcpy(hs, st, L, cudaMemcpyDeviceToHost);
                printf("a=%d bins=%d %-22s best %6.1f us  status[first]=%d\n", acol, nb,
                       variant == 0 ? "k_decode_multi" : (variant == 1 ? "k_decode_coop nw=1" : (variant == 2 ? "k_decode_coop nw=2" : "k_decode_coop nw=3")),
                       best * 1e3, hs[wl[0]]);
                if (variant) {
                    long long h[64];
                    cudaMemcpyFromSymbol(h, g_clk, sizeof(h));
                    for (int w = 0; w < variant; w++)
                        printf("      warp %d last trial: scale %lld hankel %lld roots %lld resid %lld vand %lld snap %lld cons %lld\n", w,
                               0LL, h[w * 8 + 2] - h[w * 8 + 1], h[w * 8 + 3] - h[w * 8 + 2], h[w * 8 + 4] - h[w * 8 + 3],
                               h[w * 8 + 5] - h[w * 8 + 4], h[w * 8 + 6] - h[w * 8 + 5], h[w * 8 + 7] - h[w * 8 + 6]);
                }
            }
            printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
        }
    return 0;
}
