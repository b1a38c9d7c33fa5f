// Inner-loop variants of the split sweep's cross product (experiment, not
// part of the library): pairs/s for each formulation at 2 CTAs x 256 thr/SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
constexpr int TY = 1024;

template <int V, int CPS, int NR>
__global__ void __launch_bounds__(256, CPS) k(int iters, uint64_t* sink) {
    __shared__ __align__(16) double ys[TY];
    __shared__ __align__(16) double yq[2 * TY];      // V5: (y, lo word + 2^42) per element
    __shared__ __align__(16) uint32_t yh[TY];         // V5: hi word
    for (int i = threadIdx.x; i < TY; i += blockDim.x) {
        ys[i] = 1.0 + 1e-3 * ((i * 37) % 101);
        yq[2 * i] = ys[i];
        yq[2 * i + 1] = (double)(uint32_t)__double2loint(ys[i]) + 4398046511104.0;
        yh[i] = (uint32_t)__double2hiint(ys[i]);
    }
    __syncthreads();
    double xv[NR]; uint64_t cs[NR]; uint32_t c32[NR]; double L[NR];
#pragma unroll
    for (int u = 0; u < NR; ++u) { xv[u] = 1.0 + 1e-3 * ((threadIdx.x + 13 * u) % 101); cs[u] = 0; c32[u] = 0; L[u] = 0; }
    const double4* y4 = reinterpret_cast<const double4*>(yq);
    const uint2* h2 = reinterpret_cast<const uint2*>(yh);
    const double2* y2 = reinterpret_cast<const double2*>(ys);
    for (int it = 0; it < iters; ++it) {
#pragma unroll 2
        for (int y = 0; y < TY / 2; ++y) {
            const double2 yy = y2[y];
            if (V == 5) {
                // count-encoded lo sum on the FP64 pipe: L += (x > y) * (lo + 2^42) via SEL + DFMA,
                // hi words mod 2^32 with a predicated IADD (FMA pipe)
                const double4 q = y4[y];
                const uint2 h = h2[y];
#pragma unroll
                for (int u = 0; u < NR; ++u) {
                    asm("{\n\t.reg .pred p;\n\t.reg .b32 t;\n\t.reg .f64 d;\n\t"
                        "setp.gt.f64 p, %2, %3;\n\tselp.b32 t, 1072693248, 0, p;\n\tmov.b64 d, {0, t};\n\t"
                        "fma.rn.f64 %0, d, %4, %0;\n\t@p add.u32 %1, %1, %5;\n\t}"
                        : "+d"(L[u]), "+r"(c32[u]) : "d"(xv[u]), "d"(q.x), "d"(q.y), "r"(h.x));
                    asm("{\n\t.reg .pred p;\n\t.reg .b32 t;\n\t.reg .f64 d;\n\t"
                        "setp.gt.f64 p, %2, %3;\n\tselp.b32 t, 1072693248, 0, p;\n\tmov.b64 d, {0, t};\n\t"
                        "fma.rn.f64 %0, d, %4, %0;\n\t@p add.u32 %1, %1, %5;\n\t}"
                        : "+d"(L[u]), "+r"(c32[u]) : "d"(xv[u]), "d"(q.z), "d"(q.w), "r"(h.y));
                }
                continue;
            }
#pragma unroll
            for (int u = 0; u < NR; ++u) {
                if (V == 0) {
                    const double a = xv[u] > yy.x ? xv[u] : yy.x;
                    const double b = xv[u] > yy.y ? xv[u] : yy.y;
                    cs[u] += (uint64_t)__double_as_longlong(a) + (uint64_t)__double_as_longlong(b);
                } else if (V == 1) {
                    const uint64_t xa = __double_as_longlong(xv[u]);
                    const uint64_t a = xa > (uint64_t)__double_as_longlong(yy.x) ? xa : (uint64_t)__double_as_longlong(yy.x);
                    const uint64_t b = xa > (uint64_t)__double_as_longlong(yy.y) ? xa : (uint64_t)__double_as_longlong(yy.y);
                    cs[u] += a + b;
                } else if (V == 2) {
                    const int xh = __double2hiint(xv[u]);
                    c32[u] += max(xh, __double2hiint(yy.x)) + max(xh, __double2hiint(yy.y));
                } else if (V == 4) {           // lo words into a 64-bit sum (IMAD.WIDE, FMA pipe), hi words mod 2^32
                    const double a = xv[u] > yy.x ? xv[u] : yy.x;
                    const double b = xv[u] > yy.y ? xv[u] : yy.y;
                    cs[u] += (uint64_t)(uint32_t)__double2loint(a);
                    cs[u] += (uint64_t)(uint32_t)__double2loint(b);
                    c32[u] += (uint32_t)__double2hiint(a) + (uint32_t)__double2hiint(b);
                } else if (V == 3) {
                    const double a = fmax(xv[u], yy.x);
                    const double b = fmax(xv[u], yy.y);
                    cs[u] += (uint64_t)__double_as_longlong(a) + (uint64_t)__double_as_longlong(b);
                }
            }
        }
    }
    uint64_t c = 0;
#pragma unroll
    for (int u = 0; u < NR; ++u) c += cs[u] + c32[u] + (uint64_t)L[u];
    if (c == 42) sink[0] = c;
}

template <int V, int CPS, int NR = 8>
void run(const char* name) {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    uint64_t* sink; cudaMalloc(&sink, 8);
    int grid = sms * CPS, iters = 200;
    k<V, CPS, NR><<<grid, 256>>>(4, sink);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    k<V, CPS, NR><<<grid, 256>>>(iters, sink);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double pairs = (double)grid * 256 * NR * TY * iters;
    printf("%-28s CPS=%d NR=%d %.3e pairs/s\n", name, CPS, NR, pairs / (ms / 1e3));
}

int main(int argc, char**) {
    if (argc > 1) {   // slot-count sweep of the production formulation
        run<0, 2, 1>("ns sweep"); run<0, 2, 2>("ns sweep"); run<0, 2, 3>("ns sweep");
        run<0, 2, 4>("ns sweep"); run<0, 2, 5>("ns sweep"); run<0, 2, 6>("ns sweep");
        run<0, 2, 8>("ns sweep"); run<0, 2, 12>("ns sweep"); run<0, 2, 16>("ns sweep");
        return 0;
    }
    run<0, 2>("dsetp+fsel+sel+iadd3");
    run<5, 2>("dsetp+sel+dfma+iadd (V5)");
    run<5, 2, 4>("dsetp+sel+dfma+iadd (V5)");
    run<5, 2, 6>("dsetp+sel+dfma+iadd (V5)");
    run<4, 2>("lo imad.wide + hi iadd3");
    run<4, 2, 16>("lo imad.wide + hi iadd3");
    run<0, 4>("dsetp+fsel+sel+iadd3");
    run<0, 3, 4>("dsetp+fsel+sel+iadd3");
    run<0, 4, 4>("dsetp+fsel+sel+iadd3");
    run<0, 2, 16>("dsetp+fsel+sel+iadd3");
    run<1, 2>("u64 isetp+sel+iadd3");
    run<1, 4>("u64 isetp+sel+iadd3");
    run<2, 2>("hi32 imnmx+iadd3");
    run<3, 2>("fmax (dsetp.max)");
    return 0;
}
