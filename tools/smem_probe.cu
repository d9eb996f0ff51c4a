// Shared-memory / shuffle throughput probe (B200): SM cycles per warp-level
// LDS.64 / LDS.128 / SHFL for the access patterns a per-lane coefficient
// table or a broadcast source would produce.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/smem_probe tools/smem_probe.cu
// Output: one line per pattern, cycles per warp instruction per SM.
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 4096;
constexpr int kWarps = 16;  // per block, one block per SM

// pattern -> element index (in units of the access width) for lane l, slot s
__device__ __forceinline__ int pat(int p, int l, int s) {
    switch (p) {
        case 0: return 0;                                  // all lanes one address (broadcast)
        case 1: return ((l * 7 + s * 3) ^ (l >> 2)) & 15;  // 16 random-ish slots (LDS.64: one 128-B row)
        case 2: return l;                                  // 32 distinct consecutive
        case 3: return ((l * 5 + s * 3) ^ (l >> 3)) & 7;   // 8 random-ish slots
        case 4: return l >> 4;                             // two addresses (half warps)
        case 5: return (l * 13 + s * 5) & 31;              // 32 slots permuted
        default: return (l >> 3);                          // 4 addresses (quarter warps)
    }
}

template <int W>  // access width in bytes: 8 or 16
__global__ void lds_kernel(int p, unsigned long long *cyc, int *sink) {
    __shared__ __align__(16) double tab[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) tab[i] = i;
    __syncthreads();
    const int l = threadIdx.x & 31;
    int off[8];
#pragma unroll
    for (int s = 0; s < 8; ++s) off[s] = pat(p, l, s) * (W / 8) + s * 64;
    unsigned acc = 0;
    const unsigned long long t0 = clock64();
    for (int it = 0; it < kIters; ++it) {
#pragma unroll
        for (int s = 0; s < 8; ++s) {
            if (W == 8) {
                double v;
                asm volatile("ld.volatile.shared.f64 %0, [%1];" : "=d"(v) : "r"((unsigned)__cvta_generic_to_shared(tab + off[s] + (it & 1) * 256)));
                acc ^= __double2loint(v) ^ __double2hiint(v);
            } else {
                double a, b;
                asm volatile("ld.volatile.shared.v2.f64 {%0, %1}, [%2];"
                             : "=d"(a), "=d"(b)
                             : "r"((unsigned)__cvta_generic_to_shared(tab + off[s] + (it & 1) * 256)));
                acc ^= __double2loint(a) ^ __double2hiint(a) ^ __double2loint(b) ^ __double2hiint(b);
            }
        }
    }
    const unsigned long long t1 = clock64();
    if (threadIdx.x == 0) atomicAdd(cyc, t1 - t0);
    if (acc == 0x12345) sink[0] = acc;
}

__global__ void shfl_kernel(int p, unsigned long long *cyc, int *sink) {
    const int l = threadIdx.x & 31;
    int src[8];
#pragma unroll
    for (int s = 0; s < 8; ++s) src[s] = pat(p, l, s) & 31;
    unsigned acc = l, v[8];
#pragma unroll
    for (int s = 0; s < 8; ++s) v[s] = l * 3 + s;
    const unsigned long long t0 = clock64();
    for (int it = 0; it < kIters; ++it) {
#pragma unroll
        for (int s = 0; s < 8; ++s) v[s] = __shfl_sync(0xffffffffu, v[s], src[s]) + it;
    }
#pragma unroll
    for (int s = 0; s < 8; ++s) acc ^= v[s];
    const unsigned long long t1 = clock64();
    if (threadIdx.x == 0) atomicAdd(cyc, t1 - t0);
    if (acc == 0x12345) sink[0] = acc;
}

int main() {
    unsigned long long *cyc;
    int *sink;
    cudaMalloc(&cyc, 8);
    cudaMalloc(&sink, 4);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const char *names[] = {"broadcast", "16 slots", "32 consecutive", "8 slots", "2 addresses", "32 permuted",
                           "4 addresses"};
    for (int w = 0; w < 3; ++w) {
        for (int p = 0; p < 7; ++p) {
            unsigned long long h = 0;
            for (int rep = 0; rep < 2; ++rep) {
                cudaMemset(cyc, 0, 8);
                if (w == 0) lds_kernel<8><<<sms, 32 * kWarps>>>(p, cyc, sink);
                if (w == 1) lds_kernel<16><<<sms, 32 * kWarps>>>(p, cyc, sink);
                if (w == 2) shfl_kernel<<<sms, 32 * kWarps>>>(p, cyc, sink);
                cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
            }
            // per SM: kWarps warps issue kIters * 8 instructions each in (h / sms) cycles
            const double per_block = (double)h / sms;
            const double c = per_block / ((double)kIters * 8 * kWarps);
            printf("%-6s %-16s %.3f cycles per warp instruction per SM\n", w == 0 ? "LDS.64" : (w == 1 ? "LDS.128" : "SHFL"),
                   names[p], c);
        }
    }
    cudaError_t e = cudaDeviceSynchronize();
    printf("status %s\n", cudaGetErrorString(e));
    return 0;
}
