// Dependent-chain latency of DADD / DSETP on the device (one thread), cycles per operation.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/probes/fp64_latency.cu -o /tmp/fp64_latency
#include <cstdio>
__global__ void k(double* out, long long* cyc, double a, double b, int iters) {
    double x = a, y = b, t = 0.0;
    int nm = 0;
    long long c0 = clock64();
    for (int i = 0; i < iters; ++i) {  // the reference's per-position chain: total += el + x
        x = x + b;
    }
    long long c1 = clock64();
    for (int i = 0; i < iters; ++i) {  // compare chained into an integer count, el advancing
        nm += y <= a;
        y = y + b;
    }
    long long c2 = clock64();
    for (int i = 0; i < iters; ++i) {  // two DADDs per step, one dependent on the other chain
        t += y + a;
        y = y + b;
    }
    long long c3 = clock64();
    out[0] = x + y + t + nm;
    cyc[0] = c1 - c0, cyc[1] = c2 - c1, cyc[2] = c3 - c2;
}
int main() {
    double* o; long long* c;
    cudaMalloc(&o, 8); cudaMalloc(&c, 24);
    const int it = 1 << 16;
    k<<<1, 1>>>(o, c, 1.0, 1e-9, it);
    k<<<1, 1>>>(o, c, 1.0, 1e-9, it);
    long long h[3];
    cudaMemcpy(h, c, 24, cudaMemcpyDeviceToHost);
    printf("DADD chain: %.2f cycles/op; compare+advance: %.2f cycles/step; total+=el+x with el chain: %.2f cycles/step\n",
           (double)h[0] / it, (double)h[1] / it, (double)h[2] / it);
    return 0;
}
