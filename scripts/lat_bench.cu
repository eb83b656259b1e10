// Dependent-chain latency and independent-chain throughput of the integer
// instructions the thread tier uses (sm_100a).  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cstdint>
#define N 4096
template <int OP>
__global__ void lat(int* out, int a0, int b, int c, long long* cyc) {
    int a = a0 + threadIdx.x;
    long long t0 = clock64();
#pragma unroll 64
    for (int i = 0; i < N; ++i) {
        if (OP == 0) a = __viaddmax_s32(a, b, c);
        if (OP == 1) a = __vimax3_s32(a, b, c);
        if (OP == 2) asm volatile("mad.lo.s32 %0, %0, %1, %2;" : "+r"(a) : "r"(b), "r"(c));
        if (OP == 3) a = int(__umulhi(unsigned(a), 1u << 28)) + a;  // LEA.HI
        if (OP == 4) a = (a & c) | b;                                 // LOP3
        if (OP == 5) { int p = a < c; a = p ? a + b : c; }            // ISETP+SEL
        if (OP == 6) asm volatile("{.reg .pred p; setp.lt.s32 p, %0, %2; @p mad.lo.s32 %0, %0, %1, %2;}" : "+r"(a) : "r"(b), "r"(c));
        if (OP == 7) a = __funnelshift_l(a, b, 2);
    }
    long long t1 = clock64();
    out[threadIdx.x] = a;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}
int main() {
    int* out; long long* cyc; cudaMalloc(&out, 4096); cudaMallocManaged(&cyc, 8);
    const char* names[] = {"VIADDMNMX", "VIMNMX3", "IMAD", "LEA.HI", "LOP3", "ISETP+SEL", "ISETP+@p IMAD", "SHF.funnel"};
#define RUN(OP) lat<OP><<<1, 32>>>(out, 3, 5, 7, cyc); cudaDeviceSynchronize(); lat<OP><<<1, 32>>>(out, 3, 5, 7, cyc); cudaDeviceSynchronize(); printf("%-16s %.2f cycles/dependent op\n", names[OP], double(*cyc) / N);
    RUN(0) RUN(1) RUN(2) RUN(3) RUN(4) RUN(5) RUN(6) RUN(7)
    return 0;
}
