// Which pipe runs the packed fp16 min/max/compare/add on sm_100a, and at what rate?
// Alone, and interleaved with VIADDMNMX (ALU pipe) / IMAD (FMA pipe): a pair that runs on
// different pipes approaches the issue ceiling (~126 lane-ops/clk/SM), the same pipe stays at 64.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o lat_half2 scripts/lat_half2.cu
#include <cuda_fp16.h>
#include <cstdint>
#include <cstdio>
#define N 2048
template <int OP, int MIX>
__global__ void thr(unsigned* out, unsigned a0, unsigned b, unsigned c, long long* cyc) {
    __half2 h[8];
    int x[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        unsigned v = a0 + threadIdx.x * (q + 1);
        h[q] = *reinterpret_cast<__half2*>(&v);
        x[q] = int(v);
    }
    const __half2 hb = *reinterpret_cast<const __half2*>(&b), hc = *reinterpret_cast<const __half2*>(&c);
    long long t0 = clock64();
    for (int i = 0; i < N; ++i) {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            if (OP == 0) h[q] = __hmax2(h[q], hb);
            if (OP == 1) h[q] = __hadd2(h[q], hb);
            if (OP == 2) h[q] = __hge2(h[q], hb);
            if (OP == 3) { unsigned m = __hge2_mask(h[q], hb); h[q] = *reinterpret_cast<__half2*>(&m); }
            if (OP == 4) h[q] = __hfma2(h[q], hb, hc);
            if (MIX == 1) x[q] = __viaddmax_s32(x[q], int(b), int(c));
            if (MIX == 2) asm volatile("mad.lo.s32 %0, %0, %1, %2;" : "+r"(x[q]) : "r"(int(b)), "r"(int(c)));
        }
    }
    long long t1 = clock64();
    unsigned s = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) s ^= *reinterpret_cast<unsigned*>(&h[q]) ^ unsigned(x[q]);
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
int main() {
    unsigned* out; long long* cyc; cudaMalloc(&out, 1 << 20); cudaMallocManaged(&cyc, 8);
    const char* names[] = {"HMNMX2 (hmax2)", "HADD2", "HSET2 (hge2)", "HSET2.BM (hge2_mask)", "HFMA2"};
    const char* mix[] = {"alone", "+VIADDMNMX", "+IMAD"};
#define RUN(OP, MIX) thr<OP, MIX><<<148, 512>>>(out, 0x3c003c00u, 0x3c003c00u, 7, cyc); cudaDeviceSynchronize(); thr<OP, MIX><<<148, 512>>>(out, 0x3c003c00u, 0x3c003c00u, 7, cyc); cudaDeviceSynchronize(); printf("%-22s %-12s %.1f lane-instr/clk/SM\n", names[OP], mix[MIX], 16.0 * 32 * 8 * (MIX ? 2 : 1) / (double(*cyc) / N));
    RUN(0, 0) RUN(0, 1) RUN(0, 2) RUN(1, 0) RUN(1, 1) RUN(1, 2) RUN(2, 0) RUN(2, 1) RUN(2, 2) RUN(3, 0) RUN(3, 1) RUN(3, 2) RUN(4, 0) RUN(4, 1) RUN(4, 2)
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
