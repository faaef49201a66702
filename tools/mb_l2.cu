// Micro-benchmarks for the row-slab design decisions (not part of the library):
//   1. L2-resident read bandwidth (TMA bulk copies into smem, all SMs)
//   2. HBM read bandwidth with the same loop
//   3. grid-wide all-reduce round latency: every CTA red.adds B doubles + a release
//      arrival, then waits for all arrivals and reads the sums (one round per "sequence")
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_l2 tools/mb_l2.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, int n) {
    asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t tx) {
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(tx) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
    asm volatile(
        "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n @!p bra W;\n}" ::"r"(smem_u32(b)),
        "r"(ph)
        : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// each CTA streams chunks [blockIdx.x + i*grid] of a buffer of nchunk chunks, `reps` times
__global__ void __launch_bounds__(32) stream_kernel(const char* buf, long long nchunk, int chunk, int reps, double* sink) {
    extern __shared__ __align__(128) char sm[];
    __shared__ uint64_t bar[8];
    const int NS = 6;
    if (threadIdx.x == 0) {
        for (int i = 0; i < NS; ++i) mbar_init(&bar[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    long long it = 0;
    double acc = 0;
    const long long per = (nchunk - blockIdx.x + gridDim.x - 1) / gridDim.x;
    const long long total = per * reps;
    // prologue
    if (threadIdx.x == 0)
        for (int s = 0; s < NS && s < total; ++s) {
            const long long c = blockIdx.x + (s % per) * gridDim.x;
            mbar_expect(&bar[s], chunk);
            bulk(sm + (size_t)s * chunk, buf + c * (long long)chunk, chunk, &bar[s]);
        }
    for (it = 0; it < total; ++it) {
        const int s = (int)(it % NS);
        mbar_wait(&bar[s], (uint32_t)((it / NS) & 1));
        acc += ((const double*)(sm + (size_t)s * chunk))[threadIdx.x];
        __syncwarp();
        const long long nx = it + NS;
        if (threadIdx.x == 0 && nx < total) {
            const long long c = blockIdx.x + (nx % per) * gridDim.x;
            mbar_expect(&bar[s], chunk);
            bulk(sm + (size_t)s * chunk, buf + c * (long long)chunk, chunk, &bar[s]);
        }
    }
    if (acc == 12345.0) sink[0] = acc;
}

__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
// all-reduce rounds: K rounds; round k uses slot k % S and is handled by warp k % W of every CTA:
// lanes < B red.add into gacc[slot][sub][lane], then a release arrival; the same warp later waits
// for round k - depth*W... (its own round k - W*depth) and reads the sums
__global__ void __launch_bounds__(256) allreduce_kernel(double* gacc, unsigned* arrive, int K, int S, int B, int SUB,
                                                       int depth, int rel, double* out) {
    double tot = 0;
    const int sub = blockIdx.x % SUB;
    const int W = blockDim.x / 32, w = threadIdx.x / 32, lane = threadIdx.x & 31;
    for (int kk = 0; kk < K / W + depth; ++kk) {
        const int k = kk * W + w;
        if (kk < K / W) {
            const int slot = k % S;
            for (int c = lane; c < B; c += 32) atomicAdd(&gacc[((size_t)slot * SUB + sub) * B + c], 1.0 + blockIdx.x);
            __syncwarp();
            if (lane == 0) {
                if (rel) {
                    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(arrive + slot) : "memory");
                } else {
                    asm volatile("fence.acq_rel.gpu;" ::: "memory");
                    asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(arrive + slot) : "memory");
                }
            }
        }
        const int jj = kk - depth;
        if (jj >= 0) {
            const int j = jj * W + w;
            const int slot = j % S;
            const unsigned need = (unsigned)(j / S + 1) * gridDim.x;
            if (lane == 0)
                while (ld_acq(&arrive[slot]) < need) { }
            __syncwarp();
            double g = 0;
            for (int c = lane; c < B; c += 32)
                for (int s = 0; s < SUB; ++s) g += *(volatile double*)&gacc[((size_t)slot * SUB + s) * B + c];
            tot += g;
        }
    }
    if (tot == 1.0) out[0] = tot;
}

int main() {
    int nsm;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    const size_t big = 4ull << 30;
    char* buf;
    cudaMalloc(&buf, big);
    cudaMemset(buf, 0, big);
    double* sink;
    cudaMalloc(&sink, 64);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int chunk = 32768;
    cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 6 * chunk);
    for (int ctas_per_sm = 1; ctas_per_sm <= 1; ++ctas_per_sm)
        for (size_t foot : {48ull << 20, 4ull << 30}) {
            const long long nchunk = foot / chunk;
            const int reps = foot >= (1ull << 30) ? 1 : (int)((4ull << 30) / foot);
            stream_kernel<<<nsm * ctas_per_sm, 32, 6 * chunk>>>(buf, nchunk, chunk, 1, sink);
            cudaEventRecord(a);
            stream_kernel<<<nsm * ctas_per_sm, 32, 6 * chunk>>>(buf, nchunk, chunk, reps, sink);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            printf("stream footprint %6.1f MB reps %4d: %.2f TB/s\n", foot / 1e6, reps, (double)foot * reps / ms / 1e9);
        }
    // all-reduce rounds
    double* gacc;
    unsigned* arr;
    cudaMalloc(&gacc, 1 << 24);
    cudaMalloc(&arr, 1 << 16);
    for (int B : {32, 128})
        for (int SUB : {1, 8})
            for (int W : {1, 4, 8})
                for (int depth : {0, 2, 8})
                    for (int rel : {0, 1}) {
                        const int S = 256, K = 24000;
                        if (depth * W * 2 > S) continue;
                        cudaMemset(gacc, 0, 1 << 24);
                        cudaMemset(arr, 0, 1 << 16);
                        cudaEventRecord(a);
                        allreduce_kernel<<<nsm, 32 * W>>>(gacc, arr, K, S, B, SUB, depth, rel, sink);
                        cudaEventRecord(b);
                        cudaEventSynchronize(b);
                        float ms;
                        cudaEventElapsedTime(&ms, a, b);
                        printf("allreduce B %3d SUB %d W %d depth %2d rel %d: %.3f us/round  err=%s\n", B, SUB, W, depth,
                               rel, ms * 1e3 / K, cudaGetErrorString(cudaGetLastError()));
                    }
    return 0;
}
