// Latency probes for the lane tier (one band slot per lane): primitive
// latencies (SHFL, VOTE, REDUX, FLO) and two prototypes of the DNA step.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o lat_lane scripts/lat_lane.cu
#include <cstdint>
#include <cstdio>
#define N 4096
constexpr int kDead = -(1 << 24);

template <int OP>
__global__ void prim(int* out, int a0, int b, long long* cyc) {
    int a = a0 + threadIdx.x;
    long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; ++i) {
        if (OP == 0) a = __shfl_down_sync(0xFFFFFFFFu, a, 1) + b;
        if (OP == 1) a = int(__ballot_sync(0xFFFFFFFFu, a > b)) + b;
        if (OP == 2) a = __reduce_max_sync(0xFFFFFFFFu, a) + b;
        if (OP == 3) a = (31 - __clz(a)) + b;
        if (OP == 4) a = __vimax3_s32(a, b, i);
        if (OP == 5) { unsigned m = __ballot_sync(0xFFFFFFFFu, a > b); a = ((m >> (threadIdx.x & 31)) != 0) + a; }
        if (OP == 6) a = __shfl_sync(0xFFFFFFFFu, a, (threadIdx.x + 1) & 31) + b;
        if (OP == 7) { unsigned m = __match_any_sync(0xFFFFFFFFu, a & 3); a = int(m) + b; }
    }
    long long t1 = clock64();
    out[threadIdx.x] = a;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}

// One slot per lane, DNA +1/-1/-1.  V = 0: kill, then shuffle the killed value
// to the neighbour.  V = 1: shuffle the raw candidate at once, each lane kills
// its copy of the neighbour's value with the neighbour's threshold.
template <int V>
__global__ void step(int* out, const uint32_t* seqv, const uint32_t* seqh, int X, int steps, long long* cyc,
                     long long* cells_out) {
    const int lane = threadIdx.x & 31;
    int e = lane == 16 ? X + 1 : kDead, o = kDead;  // rows d-2 / d-1 by parity
    int nbk = kDead;                                 // neighbour's killed value for the coming step
    int Tv = 1;
    uint32_t vs = seqv[lane] & 3u, hs = seqh[lane] & 3u;
    uint32_t rv = seqv[32], rh = seqh[32];
    int hs1 = 16, ls1 = 16, hs2 = -1, ls2 = 64;
    long long cells = 1;
    int delta_w = 1, best_d = 0, best_u = 0;
    int stop = 0;
    long long t0 = clock64();
    for (int it = 0; it < steps; ++it) {
#pragma unroll
        for (int par = 1; par >= 0; --par) {  // odd then even
            const int d = 2 * it + 2 - par;
            int& cur = par ? o : e;
            int& prv = par ? e : o;
            Tv += 1;
            // window (uniform)
            const int lo = par ? min(ls1 - 1, ls2) : min(ls1, ls2);
            const int hi = par ? max(hs1, hs2) : max(hs1 + 1, hs2);
            const int w = hi - lo + 1;
            if ((lo < 0 || hi > 31 || w > 256 || w <= 0) && !stop) { stop = 1; out[64] = d; }
            cells += w;
            delta_w = max(delta_w, w);
            const int sc = vs == hs ? 3 : 1;
            const int cand = __vimax3_s32(cur + sc, prv, nbk);
            const unsigned bal = __ballot_sync(0xFFFFFFFFu, cand > Tv + X);
            int nraw;
            if (V == 1) nraw = par ? __shfl_up_sync(0xFFFFFFFFu, cand, 1) : __shfl_down_sync(0xFFFFFFFFu, cand, 1);
            const int thr = Tv + ((bal >> lane) != 0);
            const bool live = cand >= thr;
            const int kept = live ? cand : kDead;
            cur = kept;
            if (V == 1) {
                const int nl = par ? lane - 1 : lane + 1;  // next step's source lane
                const int nthr = Tv + (nl >= 0 && nl < 32 && (bal >> nl) != 0);
                nbk = (nraw >= nthr && nl >= 0 && nl < 32) ? nraw : kDead;
            } else {
                nbk = par ? __shfl_up_sync(0xFFFFFFFFu, kept, 1) : __shfl_down_sync(0xFFFFFFFFu, kept, 1);
                if (par ? lane == 0 : lane == 31) nbk = kDead;
            }
            if (bal) {
                Tv += 1;
                best_d = d;
                best_u = 31 - __clz(bal);
            }
            const unsigned lm = __ballot_sync(0xFFFFFFFFu, live);
            hs2 = hs1;
            ls2 = ls1;
            hs1 = lm ? 31 - __clz(lm) : -1;
            ls1 = lm ? __ffs(lm) - 1 : 64;
            // feed
            if (par) {
                uint32_t in = __shfl_up_sync(0xFFFFFFFFu, vs, 1);
                if (lane == 0) { in = rv >> 30; }
                rv = (rv << 2) | (rv >> 30);
                vs = in;
            } else {
                uint32_t in = __shfl_down_sync(0xFFFFFFFFu, hs, 1);
                if (lane == 31) { in = rh & 3u; }
                rh = (rh >> 2) | (rh << 30);
                hs = in;
            }
        }
    }
    long long t1 = clock64();
    out[lane] = e + o + best_d + best_u + delta_w;
    if (lane == 0) { *cyc = t1 - t0; *cells_out = cells; }
}

int main() {
    int* out; long long* cyc; uint32_t *sv, *sh;
    cudaMalloc(&out, 4096); cudaMallocManaged(&cyc, 16); cudaMallocManaged(&sv, 256); cudaMallocManaged(&sh, 256);
    for (int i = 0; i < 33; ++i) { sv[i] = 0x1B1B1B1Bu * (i + 1); sh[i] = 0x1B1B1B1Bu * (i + 1); }
    const char* names[] = {"SHFL.DOWN+IADD", "ISETP+VOTE+IADD", "REDUX.MAX+IADD", "FLO+IADD", "VIMNMX3", "VOTE+SHF+ISETP+IADD", "SHFL.IDX+IADD", "MATCH.ANY"};
#define RUN(OP) prim<OP><<<1, 32>>>(out, 3, 5, cyc); cudaDeviceSynchronize(); prim<OP><<<1, 32>>>(out, 3, 5, cyc); cudaDeviceSynchronize(); printf("%-22s %.2f cycles/dependent round\n", names[OP], double(*cyc) / N);
    RUN(0) RUN(1) RUN(2) RUN(3) RUN(4) RUN(5) RUN(6) RUN(7)
    for (int rep = 0; rep < 2; ++rep) {
        step<0><<<1, 32>>>(out, sv, sh, 15, 20000, cyc, cyc + 1); cudaDeviceSynchronize();
        printf("step V0 (kill then shuffle): %.1f cycles/antidiagonal (cells %lld)\n", double(cyc[0]) / 40000, cyc[1]);
        step<1><<<1, 32>>>(out, sv, sh, 15, 20000, cyc, cyc + 1); cudaDeviceSynchronize();
        printf("step V1 (raw shuffle, local kill): %.1f cycles/antidiagonal (cells %lld)\n", double(cyc[0]) / 40000, cyc[1]);
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
