// Micro-experiments for the K1 histogram/CRC kernel (not part of the product).
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>
#include "../../paper_2505_09810_b200/csrc/lmc_common.cuh"
using namespace lmcg;

template <int V>
__global__ void __launch_bounds__(256) kexp(const uint8_t* src, uint64_t n /*elements*/, uint32_t B, const CrcTables* ct,
                                           uint32_t* hist_out, uint32_t* sink) {
    __shared__ uint32_t sh_hist[8][256];
    __shared__ uint32_t sh_slice[1024];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // slot -> (plane g, block j): interleaved
    const uint32_t g = blockIdx.x & 1, j = blockIdx.x >> 1;
    for (int i = tid; i < 8 * 256; i += 256) (&sh_hist[0][0])[i] = 0;
    if (V >= 2) for (int i = tid; i < 1024; i += 256) sh_slice[i] = ct->slice[i >> 8][i & 255];
    __syncthreads();
    uint32_t* hist = sh_hist[warp];
    const uint64_t e0 = (uint64_t)j * B;           // first element
    const uint64_t T = 1024;                       // positions per warp tile (w = 2)
    uint32_t x = 0, crcacc = 0;
    for (uint64_t t = warp; t * T < B; t += 8) {
        const uint64_t base = (e0 + t * T) * 2 + 16ull * lane;
        uint4 a[4];
#pragma unroll
        for (int q = 0; q < 4; q++) a[q] = __ldg(reinterpret_cast<const uint4*>(src + base + 512ull * q));
        if (V == 0) {
#pragma unroll
            for (int q = 0; q < 4; q++) x ^= a[q].x ^ a[q].y ^ a[q].z ^ a[q].w;
        }
        if (V == 1 || V == 3) {
#pragma unroll
            for (int q = 0; q < 4; q++) {
                uint32_t sy[4];
                piece_symbols(a[q], 2, g, sy);
#pragma unroll
                for (int i = 0; i < 8; i++) atomicAdd(&hist[(sy[i >> 2] >> (8 * (i & 3))) & 0xFF], 1u);
            }
        }
        if (V == 4) {  // match_any aggregation
#pragma unroll
            for (int q = 0; q < 4; q++) {
                uint32_t sy[4];
                piece_symbols(a[q], 2, g, sy);
#pragma unroll
                for (int i = 0; i < 8; i++) {
                    const uint32_t s = (sy[i >> 2] >> (8 * (i & 3))) & 0xFF;
                    const uint32_t m = __match_any_sync(0xFFFFFFFFu, s);
                    if (lane == __ffs(m) - 1) atomicAdd(&hist[s], __popc(m));
                }
            }
        }
        if (V == 5) {  // 4 sub-histograms per warp by lane % 4, padded banks
#pragma unroll
            for (int q = 0; q < 4; q++) {
                uint32_t sy[4];
                piece_symbols(a[q], 2, g, sy);
#pragma unroll
                for (int i = 0; i < 8; i++) {
                    const uint32_t s = (sy[i >> 2] >> (8 * (i & 3))) & 0xFF;
                    atomicAdd(&(&sh_hist[0][0])[(((lane & 3) * 2 + (warp & 1)) * 257) % 1792 + s], 1u);
                }
            }
        }
        if (V == 2 || V == 3) {
            if (g == 0) {
                uint32_t acc = 0;
#pragma unroll
                for (int q = 0; q < 4; q++) {
                    const uint32_t part = crc_warp_tree(ct, crc16(sh_slice, a[q]), lane, kShift16);
                    acc = crc_shift_tab(&ct->shift[kShift512][0][0], acc) ^ part;
                }
                crcacc ^= acc;
            }
        }
        if (V == 6 || V == 7) {  // Horner over rows per lane, one lane tree per tile
            if (g == 0) {
                uint32_t v = crc16(sh_slice, a[0]);
#pragma unroll
                for (int q = 1; q < 4; q++) v = crc_shift_tab(&ct->shift[kShift512][0][0], v) ^ crc16(sh_slice, a[q]);
                crcacc ^= crc_warp_tree(ct, v, lane, kShift16);
            }
        }
        if (V == 7) {
#pragma unroll
            for (int q = 0; q < 4; q++) {
                uint32_t sy[4];
                piece_symbols(a[q], 2, g, sy);
#pragma unroll
                for (int i = 0; i < 8; i++) atomicAdd(&hist[(sy[i >> 2] >> (8 * (i & 3))) & 0xFF], 1u);
            }
        }
    }
    __syncthreads();
    uint32_t sum = 0;
    for (int q = 0; q < 8; q++) sum += sh_hist[q][tid];
    hist_out[blockIdx.x * 256 + tid] = sum;
    if (x == 0x12345678u || crcacc == 0x9abcdef0u) sink[0] = x ^ crcacc;
}

int main() {
    const uint64_t n = 64ull << 20;  // elements (128 MiB)
    const uint32_t B = 65536;
    std::vector<uint16_t> h(n);
    uint64_t st = 88172645463325252ull;
    for (uint64_t i = 0; i < n; i++) {
        // cheap normal-ish bf16: sum of uniforms * 0.02
        st ^= st << 13; st ^= st >> 7; st ^= st << 17;
        float u = ((st & 0xFFFF) + ((st >> 16) & 0xFFFF) + ((st >> 32) & 0xFFFF) - 3 * 32768.f) / 32768.f * 0.02f;
        uint32_t b; memcpy(&b, &u, 4);
        h[i] = (uint16_t)((b + 0x7FFF + ((b >> 16) & 1)) >> 16);
    }
    uint8_t* d; cudaMalloc(&d, n * 2);
    cudaMemcpy(d, h.data(), n * 2, cudaMemcpyHostToDevice);
    CrcTables* ct; cudaMalloc(&ct, sizeof(CrcTables)); cudaMemset(ct, 0, sizeof(CrcTables));
    uint32_t *hist, *sink; cudaMalloc(&hist, 4096ull * 256 * 4); cudaMalloc(&sink, 4);
    const int grid = (int)(2 * n / B);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    auto run = [&](auto kern, const char* name) {
        for (int i = 0; i < 3; i++) kern<<<grid, 256>>>(d, n, B, ct, hist, sink);
        cudaEventRecord(a);
        for (int i = 0; i < 10; i++) kern<<<grid, 256>>>(d, n, B, ct, hist, sink);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b); ms /= 10;
        printf("%-28s %8.1f us  %7.1f GB/s (source read x1)\n", name, ms * 1e3, 2.0 * n / (ms * 1e-3) / 1e9);
    };
    run(kexp<0>, "V0 loads only");
    run(kexp<1>, "V1 loads+hist atomics");
    run(kexp<2>, "V2 loads+crc");
    run(kexp<3>, "V3 loads+hist+crc");
    run(kexp<4>, "V4 hist match_any");
    run(kexp<5>, "V5 hist 4-way sub-hists");
    run(kexp<6>, "V6 loads+crc horner");
    run(kexp<7>, "V7 loads+hist+crc horner");
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
