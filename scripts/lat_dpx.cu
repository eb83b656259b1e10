// Throughput / SASS probe of the packed 16x2 DPX instructions on sm_100a (would a
// two-units-per-thread thread tier pay?).  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdint>
#include <cstdio>
#define N 2048
template <int OP>
__global__ void thr(unsigned* out, unsigned a0, unsigned b, unsigned c, long long* cyc) {
    unsigned a[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) a[q] = a0 + threadIdx.x * (q + 1);
    long long t0 = clock64();
    for (int i = 0; i < N; ++i) {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            if (OP == 0) a[q] = __vimax3_s16x2(a[q], b, c);
            if (OP == 1) a[q] = __viaddmax_s16x2(a[q], b, c);
            if (OP == 2) a[q] = __vimax3_s32(int(a[q]), int(b), int(c));
            if (OP == 3) a[q] = __viaddmax_s32(int(a[q]), int(b), int(c));
            if (OP == 4) { bool ph, pl; a[q] = __vibmax_s16x2(a[q], b, &ph, &pl); a[q] += (ph ? 1u : 0u) + (pl ? 65536u : 0u); }
            if (OP == 5) a[q] = __vimax_s16x2_relu(a[q], b);
            if (OP == 6) a[q] = __vadd2(a[q], b);
            if (OP == 7) a[q] = __vcmpges2(a[q], b) & c;
        }
    }
    long long t1 = clock64();
    unsigned s = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) s ^= a[q];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
int main() {
    unsigned* out; long long* cyc; cudaMalloc(&out, 1 << 20); cudaMallocManaged(&cyc, 8);
    const char* names[] = {"vimax3_s16x2", "viaddmax_s16x2", "vimax3_s32", "viaddmax_s32", "vibmax_s16x2+use", "vimax_s16x2_relu", "vadd2", "vcmpges2&c"};
#define RUN(OP) thr<OP><<<148, 512>>>(out, 3, 5, 7, cyc); cudaDeviceSynchronize(); thr<OP><<<148, 512>>>(out, 3, 5, 7, cyc); cudaDeviceSynchronize(); printf("%-18s %.2f cycles per 8 ops per warp (16 warps/SM: %.1f lane-ops/clk/SM)\n", names[OP], double(*cyc) / N, 16.0 * 32 * 8 / (double(*cyc) / N));
    RUN(0) RUN(1) RUN(2) RUN(3) RUN(4) RUN(5) RUN(6) RUN(7)
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
