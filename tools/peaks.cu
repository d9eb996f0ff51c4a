// Micro-benchmarks for the roofline denominators MEASURED_PEAKS.json lacks:
// fp64 FMA throughput, fp64 tensor-core MMA (DMMA) throughput,
// shared-memory bandwidth (64-bit LDS/STS), native
// fp64 global reductions (REDG.E.ADD.F64) into an L2-resident array, and an
// fp64 copy (HBM) as a cross-check.  Prints one JSON object.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o peaks tools/peaks.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#define CK(x)                                                                  \
    do {                                                                       \
        cudaError_t e = (x);                                                   \
        if (e != cudaSuccess) {                                                \
            fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); \
            return 1;                                                          \
        }                                                                      \
    } while (0)

__global__ void dfma_kernel(double *out, int iters, double a, double b) {
    double x[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = threadIdx.x * 1e-9 + j;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = fma(x[j], a, b);
    }
    double s = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += x[j];
    if (s == 12345.678) out[0] = s;
}

// fp64 tensor-core MMA (mma.sync.m8n8k4.f64, DMMA): 4 independent
// accumulator tiles per warp, 2 * 8 * 8 * 4 = 512 flop per instruction
__global__ void dmma_kernel(double *out, int iters, double a0, double b0) {
    double a = a0 + threadIdx.x * 1e-12, b = b0;
    double c[4][2] = {{0, 0}, {0, 0}, {0, 0}, {0, 0}};
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 4; ++j)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                         : "+d"(c[j][0]), "+d"(c[j][1])
                         : "d"(a), "d"(b));
    }
    double s = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) s += c[j][0] + c[j][1];
    if (s == 12345.678) out[0] = s;
}

__global__ void smem_kernel(double *out, int iters) {
    __shared__ double buf[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) buf[i] = i;
    __syncthreads();
    double acc = 0;
    int idx = threadIdx.x;
    for (int i = 0; i < iters; ++i) {
        double v = buf[idx];
        buf[(idx + 32 * 7) & 4095] = v + 1.0;
        acc += v;
        idx = (idx + 32) & 4095;
    }
    if (acc == 12345.678) out[0] = acc;
}

__global__ void red_kernel(double *arr, size_t n, int iters) {
    size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    size_t stride = (size_t)gridDim.x * blockDim.x;
    for (int i = 0; i < iters; ++i) {
        size_t k = (tid + (size_t)i * stride * 7) % n;
        atomicAdd(arr + k, 1.0);
    }
}

__global__ void copy_kernel(const double2 *__restrict__ a, double2 *__restrict__ b, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}

template <class F>
float time_ms(F f, int reps) {
    cudaEvent_t s, e;
    cudaEventCreate(&s);
    cudaEventCreate(&e);
    f();
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < reps; ++r) {
        cudaEventRecord(s);
        f();
        cudaEventRecord(e);
        cudaEventSynchronize(e);
        float ms;
        cudaEventElapsedTime(&ms, s, e);
        if (ms < best) best = ms;
    }
    return best;
}

int main() {
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    double *out;
    CK(cudaMalloc(&out, 64));
    // fp64 FMA: blocks = 8 per SM x 256 threads, 8 independent chains
    int iters = 4096;
    int blocks = sms * 8, threads = 256;
    float ms = time_ms([&] { dfma_kernel<<<blocks, threads>>>(out, iters, 0.999999, 1e-7); }, 5);
    double flops = 2.0 * 8 * iters * (double)blocks * threads;
    double fp64_tflops = flops / (ms * 1e-3) / 1e12;
    // fp64 tensor-core MMA
    int diters = 4096;
    ms = time_ms([&] { dmma_kernel<<<sms * 8, 256>>>(out, diters, 1e-3, 1e-3); }, 5);
    double dmma_tflops = 512.0 * 4 * diters * (sms * 8 * 256 / 32.0) / (ms * 1e-3) / 1e12;
    // shared memory: one LDS.64 + one STS.64 per thread-iteration
    int siters = 1 << 14;
    ms = time_ms([&] { smem_kernel<<<sms * 4, 512>>>(out, siters); }, 5);
    double smem_bytes = 16.0 * siters * (double)sms * 4 * 512;
    double smem_tbs = smem_bytes / (ms * 1e-3) / 1e12;
    // fp64 REDG into a 16 MB (L2-resident) array
    size_t n = (16u << 20) / 8;
    double *arr;
    CK(cudaMalloc(&arr, n * 8));
    CK(cudaMemset(arr, 0, n * 8));
    int riters = 64;
    ms = time_ms([&] { red_kernel<<<sms * 8, 256>>>(arr, n, riters); }, 5);
    double reds = (double)riters * sms * 8 * 256;
    double red_g = reds / (ms * 1e-3) / 1e9;
    // HBM copy, 2 x 1 GiB
    size_t cn = (1ull << 30) / 16;
    double2 *a, *b;
    CK(cudaMalloc(&a, cn * 16));
    CK(cudaMalloc(&b, cn * 16));
    CK(cudaMemset(a, 0, cn * 16));
    ms = time_ms([&] { copy_kernel<<<sms * 16, 256>>>(a, b, cn); }, 5);
    double hbm = 2.0 * cn * 16 / (ms * 1e-3) / 1e9;
    cudaDeviceProp prop;
    cudaGetDeviceProperties(&prop, 0);
    printf("{\"gpu\": \"%s\", \"sms\": %d, \"fp64_fma_tflops\": %.2f, \"fp64_dmma_tflops\": %.2f, \"smem_tbs\": %.2f, "
           "\"redg_f64_gops\": %.2f, \"copy_hbm_gbs\": %.1f, "
           "\"how\": \"dfma 8 chains x %d iters x %d blocks x 256; smem LDS.64+STS.64 per iter; "
           "REDG.F64 to a 16 MB array, 8 x 256 thr per SM; float2x2 copy of 1 GiB; best of 5, CUDA events\"}\n",
           prop.name, sms, fp64_tflops, dmma_tflops, smem_tbs, red_g, hbm, iters, blocks);
    return 0;
}
