// Cycles per position of K2's sequential score loop (one active lane; operands in shared memory),
// in several formulations -- where the replay kernel's time per proposal goes.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/probes/chain_loop.cu -o tools/probes/chain_loop
#include <cstdio>
constexpr int N = 1024;
__global__ void k(const double2* gx, const double* gd, double* out, long long* cyc) {
    __shared__ double2 xa[N];
    __shared__ double dl[N];
    for (int i = threadIdx.x; i < N; i += blockDim.x) xa[i] = gx[i], dl[i] = gd[i];
    __syncthreads();
    if (threadIdx.x != 0) return;
    const double2* dl2 = reinterpret_cast<const double2*>(dl);
    double acc = 0.0;
    long long c[6];
    // V0: plain loop, no unroll hints
    c[0] = clock64();
    {
        double total = 0.0, el = 0.0;
        int nm = 0;
        for (int q = 0; q < N; ++q) {
            const double2 v = xa[q];
            nm += el <= dl[q];
            total += el + v.x;
            el += v.y;
        }
        acc += total + nm + el;
    }
    c[1] = clock64();
    // V1: unroll 16, loads inside
    {
        double total = 0.0, el = 0.0;
        int nm = 0;
#pragma unroll 16
        for (int q = 0; q < N; ++q) {
            const double2 v = xa[q];
            nm += el <= dl[q];
            total += el + v.x;
            el += v.y;
        }
        acc += total + nm + el;
    }
    c[2] = clock64();
    // V2: total chain only (el from the array: what the DADD floor allows)
    {
        double total = 0.0;
#pragma unroll 16
        for (int q = 0; q < N; ++q) total += xa[q].y + xa[q].x;
        acc += total;
    }
    c[3] = clock64();
    // V3: K2's 16-wide double-buffered blocks
    {
        double total = 0.0, el = 0.0;
        int nm = 0;
        auto load16 = [&](double2 (&u)[16], double2 (&d)[8], int q0) {
#pragma unroll
            for (int j = 0; j < 16; ++j) u[j] = xa[q0 + j];
#pragma unroll
            for (int j = 0; j < 8; ++j) d[j] = dl2[(q0 >> 1) + j];
        };
        auto run16 = [&](const double2 (&u)[16], const double2 (&d)[8]) {
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                nm += el <= ((j & 1) ? d[j >> 1].y : d[j >> 1].x);
                total += el + u[j].x;
                el += u[j].y;
            }
        };
        double2 A[16], B[16], DA[8], DB[8];
        load16(A, DA, 0);
        for (int q = 0; q < N; q += 32) {
            load16(B, DB, q + 16);
            run16(A, DA);
            if (q + 32 < N) load16(A, DA, q + 32);
            run16(B, DB);
        }
        acc += total + nm + el;
    }
    c[4] = clock64();
    // V4: el advanced only at batch ends (branch), the rest as V1
    {
        double total = 0.0, el = 0.0;
        int nm = 0;
#pragma unroll 16
        for (int q = 0; q < N; ++q) {
            const double2 v = xa[q];
            nm += el <= dl[q];
            total += el + v.x;
            if (v.y != 0.0) el += v.y;
        }
        acc += total + nm + el;
    }
    c[5] = clock64();
    out[0] = acc;
    for (int i = 0; i < 5; ++i) cyc[i] = c[i + 1] - c[i];
}
int main() {
    double2 hx[N];
    double hd[N];
    for (int i = 0; i < N; ++i) hx[i] = make_double2(100.0 + i, (i % 4 == 3) ? 400.0 + i : 0.0), hd[i] = 1e5 + 7.0 * i;
    double2* gx; double* gd; double* o; long long* c;
    cudaMalloc(&gx, sizeof hx); cudaMalloc(&gd, sizeof hd); cudaMalloc(&o, 8); cudaMalloc(&c, 5 * 8);
    cudaMemcpy(gx, hx, sizeof hx, cudaMemcpyHostToDevice);
    cudaMemcpy(gd, hd, sizeof hd, cudaMemcpyHostToDevice);
    for (int r = 0; r < 3; ++r) k<<<1, 32>>>(gx, gd, o, c);
    long long h[5];
    cudaMemcpy(h, c, sizeof h, cudaMemcpyDeviceToHost);
    const char* names[5] = {"plain loop", "unroll 16", "total chain only", "K2 16-wide double-buffered", "el at batch ends only"};
    for (int i = 0; i < 5; ++i) printf("%-28s %.2f cycles/position\n", names[i], (double)h[i] / N);
    return 0;
}
