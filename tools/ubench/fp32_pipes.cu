// fp32_pipes.cu -- FP32 pipe microbenchmark on sm_100a (K1 design input).
// Measures sustained FFMA (scalar), FFMA2 (fma.rn.f32x2) and MUFU.EX2 rates
// with 8 independent chains per thread, full occupancy, CUDA-event timing.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp32_pipes fp32_pipes.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;

__global__ void k_ffma(float* out, float a, float b) {
    float x[8];
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3f + i;
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = fmaf(x[i], a, b);
    }
    float s = 0;
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 1234.5f) out[threadIdx.x] = s;
}

__global__ void k_ffma_reg(float* out, const float* ab) {
    // all-register operands (a, b per thread, not constant-bank)
    float a = ab[threadIdx.x & 31], b = ab[32 + (threadIdx.x & 31)];
    float x[8];
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3f + i;
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = fmaf(x[i], a, b);
    }
    float s = 0;
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 1234.5f) out[threadIdx.x] = s;
}

__global__ void k_ffma2(float* out, float a, float b) {
    unsigned long long x[8];
    float2 av = make_float2(a, a), bv = make_float2(b, b);
    unsigned long long A = *reinterpret_cast<unsigned long long*>(&av);
    unsigned long long B = *reinterpret_cast<unsigned long long*>(&bv);
    for (int i = 0; i < 8; ++i) {
        float2 v = make_float2(threadIdx.x * 1e-3f + i, i * 0.5f);
        x[i] = *reinterpret_cast<unsigned long long*>(&v);
    }
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x[i]) : "l"(A), "l"(B));
    }
    float s = 0;
    for (int i = 0; i < 8; ++i) {
        float2 v = *reinterpret_cast<float2*>(&x[i]);
        s += v.x + v.y;
    }
    if (s == 1234.5f) out[threadIdx.x] = s;
}

__global__ void k_ex2(float* out, float a) {
    float x[8];
    for (int i = 0; i < 8; ++i) x[i] = -(threadIdx.x * 1e-3f + i) * 1e-3f;
    for (int it = 0; it < ITERS / 4; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x[i]));
    }
    float s = 0;
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 1234.5f) out[threadIdx.x] = s;
}

template <typename F>
float time_it(F f) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    f();
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) f();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms / 5;
}

// Sustained FFMA: back-to-back launches for `seconds` (power/thermal steady
// state, like MEASURED_PEAKS.json's sustained bf16 figure); returns TF/s of
// the last second.
double sustained_ffma(int sms, float* out, float* ab, double seconds) {
    const int blocks = sms * 8, threads = 256;
    const double fl = double(blocks) * threads * ITERS * 8 * 2;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    double elapsed = 0, last = 0;
    while (elapsed < seconds) {
        cudaEventRecord(e0);
        for (int r = 0; r < 50; ++r) k_ffma_reg<<<blocks, threads>>>(out, ab);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        elapsed += ms * 1e-3;
        last = 50 * fl / (ms * 1e-3) / 1e12;
    }
    return last;
}

int main(int argc, char** argv) {
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, 0);
    int sms = p.multiProcessorCount;
    float* out;
    cudaMalloc(&out, 1 << 20);
    const int blocks = sms * 8, threads = 256;
    const double lanes = double(blocks) * threads;
    float t = time_it([&] { k_ffma<<<blocks, threads>>>(out, 0.999f, 1e-3f); });
    double fl = lanes * ITERS * 8 * 2;
    printf("{\"sms\": %d, \"ffma_tflops\": %.2f, ", sms, fl / t / 1e9);
    float* ab;
    cudaMalloc(&ab, 256);
    cudaMemset(ab, 0, 256);
    t = time_it([&] { k_ffma_reg<<<blocks, threads>>>(out, ab); });
    printf("\"ffma_reg_tflops\": %.2f, ", fl / t / 1e9);
    t = time_it([&] { k_ffma2<<<blocks, threads>>>(out, 0.999f, 1e-3f); });
    fl = lanes * ITERS * 8 * 4;
    printf("\"ffma2_tflops\": %.2f, ", fl / t / 1e9);
    t = time_it([&] { k_ex2<<<blocks, threads>>>(out, 0.999f); });
    double ops = lanes * (ITERS / 4) * 8;
    printf("\"ex2_gops\": %.1f, \"ex2_per_clk_per_sm_at_max\": %.2f", ops / t / 1e6,
           ops / (t * 1e-3) / sms / (p.clockRate * 1e3));
    if (argc > 1) printf(", \"ffma_sustained_tflops\": %.2f, \"sustained_s\": %s",
                         sustained_ffma(sms, out, ab, atof(argv[1])), argv[1]);
    printf("}\n");
    return 0;
}
