// Ceiling micro-benchmark for the CSC scalar-block update (sparse_async.cuh), not part of
// the library.  A synthetic CSC matrix with the configs[4] shape (m = 1e5 rows, n = 1e6
// columns, `nnz` nonzeros per column at uniform random rows, int32 rowidx + fp64 vals)
// and an interleaved [r_i, y_i] residual array (1.6 MB, L2-resident).  Each kernel does one
// sweep of exactly the memory traffic of the update's data path, with NO dependency chain
// (no guards, no schedule, no solve, no completion):
//   gather   : colptr, the column's rowidx/vals, one 16-byte [r, y] gather per nonzero, x_j store
//   scatter  : gather + one f64 red.add into r per nonzero (the A_j dx_j push)
//   atomics  : only the red.adds (random rows), to separate the atomic rate
// in two layouts: a lane per column ("lane") and an 8-lane group per column ("group8").
// The best "scatter" rate is the ceiling the async kernel is measured against.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mb_sparse tools/mb_sparse.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double2 ld_relaxed_f64x2(const double* p) {
    double2 v;
    asm volatile("ld.relaxed.gpu.global.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint32_t hash32(uint32_t h) {
    h ^= h >> 16; h *= 0x85EBCA6Bu; h ^= h >> 13; h *= 0xC2B2AE35u; h ^= h >> 16;
    return h;
}

__global__ void gen_kernel(long long n, int nnz, int m, long long* colptr, int* rowidx, double* vals) {
    for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < n; j += (long long)gridDim.x * blockDim.x) {
        colptr[j] = j * nnz;
        if (j == n - 1) colptr[n] = n * nnz;
        for (int q = 0; q < nnz; ++q) {
            rowidx[j * nnz + q] = (int)(hash32((uint32_t)(j * 977 + q * 131071 + 7)) % (uint32_t)m);
            vals[j * nnz + q] = 1e-6 * (double)((int)(hash32((uint32_t)(j * 31 + q)) & 1023) - 512);
        }
    }
}

template <int MODE>  // 0 gather, 1 scatter, 2 atomics only
__global__ void __launch_bounds__(128) lane_kernel(const long long* __restrict__ colptr, const int* __restrict__ rowidx,
                                                   const double* __restrict__ vals, long long n, double* ry, double* x) {
    for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < n; j += (long long)gridDim.x * blockDim.x) {
        const long long s = __ldg(&colptr[j]), e = __ldg(&colptr[j + 1]);
        double acc = 0.0;
        if (MODE != 2) {
            for (long long q = s; q < e; ++q) {
                const int row = __ldg(&rowidx[q]);
                const double2 p = ld_relaxed_f64x2(&ry[2 * (long long)row]);
                acc = fma(__ldg(&vals[q]), p.x * p.y, acc);
            }
            x[j] = acc;
        }
        if (MODE != 0) {
            const double d = MODE == 2 ? 1e-9 : acc * 1e-12;
            for (long long q = s; q < e; ++q) atomicAdd(&ry[2 * (long long)__ldg(&rowidx[q])], __ldg(&vals[q]) * d);
        }
    }
}

template <int MODE>
__global__ void __launch_bounds__(128) group_kernel(const long long* __restrict__ colptr, const int* __restrict__ rowidx,
                                                    const double* __restrict__ vals, long long n, double* ry, double* x) {
    const int gl = threadIdx.x & 7;
    const unsigned gmask = 0xFFu << (threadIdx.x & 24);
    const long long g0 = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 3;
    const long long ng = ((long long)gridDim.x * blockDim.x) >> 3;
    for (long long j = g0; j < n; j += ng) {
        const long long s = __ldg(&colptr[j]), e = __ldg(&colptr[j + 1]);
        double acc = 0.0;
        if (MODE != 2) {
            for (long long q = s + gl; q < e; q += 8) {
                const int row = __ldg(&rowidx[q]);
                const double2 p = ld_relaxed_f64x2(&ry[2 * (long long)row]);
                acc = fma(__ldg(&vals[q]), p.x * p.y, acc);
            }
            acc += __shfl_xor_sync(gmask, acc, 4);
            acc += __shfl_xor_sync(gmask, acc, 2);
            acc += __shfl_xor_sync(gmask, acc, 1);
            if (gl == 0) x[j] = acc;
        }
        if (MODE != 0) {
            const double d = MODE == 2 ? 1e-9 : acc * 1e-12;
            for (long long q = s + gl; q < e; q += 8) atomicAdd(&ry[2 * (long long)__ldg(&rowidx[q])], __ldg(&vals[q]) * d);
        }
    }
}

int main(int argc, char** argv) {
    const int m = 100000, nnz = argc > 1 ? atoi(argv[1]) : 10;
    const long long n = 1000000;
    long long* colptr;
    int* rowidx;
    double *vals, *ry, *x;
    cudaMalloc(&colptr, sizeof(long long) * (n + 1));
    cudaMalloc(&rowidx, sizeof(int) * n * nnz);
    cudaMalloc(&vals, sizeof(double) * n * nnz);
    cudaMalloc(&ry, sizeof(double) * 2 * m);
    cudaMalloc(&x, sizeof(double) * n);
    cudaMemset(ry, 0, sizeof(double) * 2 * m);
    gen_kernel<<<1184, 256>>>(n, nnz, m, colptr, rowidx, vals);
    cudaDeviceSynchronize();
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const char* names[3] = {"gather", "scatter", "atomics"};
    for (int layout = 0; layout < 2; ++layout)
        for (int mode = 0; mode < 3; ++mode)
            for (int occ : {4, 8, 16}) {
                const int grid = sms * occ;
                auto launch = [&]() {
                    if (layout == 0) {
                        if (mode == 0) lane_kernel<0><<<grid, 128>>>(colptr, rowidx, vals, n, ry, x);
                        if (mode == 1) lane_kernel<1><<<grid, 128>>>(colptr, rowidx, vals, n, ry, x);
                        if (mode == 2) lane_kernel<2><<<grid, 128>>>(colptr, rowidx, vals, n, ry, x);
                    } else {
                        if (mode == 0) group_kernel<0><<<grid, 128>>>(colptr, rowidx, vals, n, ry, x);
                        if (mode == 1) group_kernel<1><<<grid, 128>>>(colptr, rowidx, vals, n, ry, x);
                        if (mode == 2) group_kernel<2><<<grid, 128>>>(colptr, rowidx, vals, n, ry, x);
                    }
                };
                for (int w = 0; w < 3; ++w) launch();
                cudaEventRecord(a);
                const int reps = 20;
                for (int r = 0; r < reps; ++r) launch();
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms = 0;
                cudaEventElapsedTime(&ms, a, b);
                const double per = ms / reps;
                printf("{\"layout\": \"%s\", \"mode\": \"%s\", \"ctas_per_sm\": %d, \"nnz_per_col\": %d, "
                       "\"ms_per_sweep\": %.4f, \"G_updates_per_s\": %.3f, \"G_nnz_per_s\": %.2f}\n",
                       layout ? "group8" : "lane", names[mode], occ, nnz, per, n / per / 1e6, n * (double)nnz / per / 1e6);
            }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
    return 0;
}
