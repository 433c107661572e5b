// Microbenchmark: per-SMSP issue cost of the softmax's instruction mix, W warps per CTA,
// one CTA per SM, 8 independent chains per thread.  Usage: ubench_alu <op> <warps>
//   op 0: ex2.approx.ftz.f32    op 1: fma.rn.f32x2    op 2: cvt.rn.bf16x2.f32 (F2FP)
//   op 3: max3 (fmaxf(fmaxf))   op 4: softmax-like mix per element (FFMA2/2, EX2, F2FP/2, FADD2/2)
#include "../paper_2603_29494_b200/csrc/common.cuh"
#include <cstdio>
#include <cstdlib>

using namespace va;
constexpr int REPS = 2048;

__global__ void __launch_bounds__(1024, 1) kern(int op, unsigned long long* out, float* sink) {
    float x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = -0.001f * (threadIdx.x + i);
    uint32_t u = 0;
    float2 acc = make_float2(0.f, 0.f);
    __syncthreads();
    const unsigned long long t0 = clock64();
    for (int r = 0; r < REPS; ++r) {
        if (op == 0) {
#pragma unroll
            for (int i = 0; i < 8; ++i) x[i] = ex2(x[i]) - 1.0f;
        } else if (op == 1) {
#pragma unroll
            for (int i = 0; i < 8; i += 2) {
                const float2 y = unpack_f32x2(ffma2(pack_f32x2(x[i], x[i + 1]), pack_f32x2(0.999f, 0.999f),
                                                    pack_f32x2(0.001f, 0.001f)));
                x[i] = y.x;
                x[i + 1] = y.y;
            }
        } else if (op == 2) {
#pragma unroll
            for (int i = 0; i < 8; i += 2) {
                u ^= pack_bf16x2(x[i], x[i + 1]);
                x[i] += 1e-7f;
            }
        } else if (op == 3) {
#pragma unroll
            for (int i = 0; i < 8; i += 2) x[i] = fmaxf(fmaxf(x[i], x[i + 1]), x[(i + 2) & 7] * 0.5f);
        } else {
#pragma unroll
            for (int i = 0; i < 8; i += 2) {
                const float2 y = unpack_f32x2(ffma2(pack_f32x2(x[i], x[i + 1]), pack_f32x2(0.5f, 0.5f),
                                                    pack_f32x2(-0.25f, -0.25f)));
                const float p0 = ex2(y.x), p1 = ex2(y.y);
                acc = fadd2(acc, make_float2(p0, p1));
                u ^= pack_bf16x2(p0, p1);
                x[i] = p0 - 1.0f;
                x[i + 1] = p1 - 1.0f;
            }
        }
    }
    const unsigned long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    float s = acc.x + acc.y + (float)u;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 1234.5f) sink[threadIdx.x] = s;
}

int main(int argc, char** argv) {
    const int op = atoi(argv[1]), W = atoi(argv[2]);
    unsigned long long* d;
    float* sink;
    cudaMalloc(&d, 148 * 8);
    cudaMalloc(&sink, 4096 * 4);
    kern<<<148, 32 * W>>>(op, d, sink);
    kern<<<148, 32 * W>>>(op, d, sink);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h[148];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double m = 0;
    for (int i = 0; i < 148; ++i) m += h[i];
    m /= 148;
    const double elems = (double)REPS * 8 * 32 * W;  // element-ops per SM
    printf("op=%d warps=%d: %.2f clk per warp-iteration, %.2f element-ops/clk/SM  %s\n", op, W, m / REPS,
           elems / m, cudaGetErrorString(e));
    return 0;
}
