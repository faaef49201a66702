// Microbenchmark: HBM streaming rate of 2-D TMA boxes (R rows x C fp64 columns) from a
// column-major matrix, in the row-slab pattern (CTA s reads rows [s*Rs, s*Rs+Rs) of every
// column block) or the panel pattern (CTAs take consecutive R-row panels of a block).
// One CTA per SM; one issuing thread per ring (NR rings per CTA, NS stages each); the
// consumer only waits and frees.  Prints GB/s.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_tma mb_tma.cu -lcuda
// ./mb_tma m n R C NS NR pattern(0 slab,1 panel)
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(128, 1) k_stream(const __grid_constant__ CUtensorMap tm, int64_t m, int64_t n, int R,
                                                   int C, int NS, int pattern, unsigned long long* sink, int NL) {
    extern __shared__ __align__(1024) unsigned char sm[];
    const int NR0 = blockDim.x / 32;
    const int NR = NR0 * NL;  // issuing threads per CTA
    const int warp = (threadIdx.x >> 5) * NL + (threadIdx.x & 31), lane = (threadIdx.x & 31) < NL ? 0 : 1;
    const uint32_t box = (uint32_t)R * C * 8;
    unsigned char* base = sm + (size_t)(lane == 0 ? warp : 0) * NS * box;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + (size_t)NR * NS * box) + (lane == 0 ? warp : 0) * NS;
    if (lane == 0)
        for (int s = 0; s < NS; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bars[s])));
    asm volatile("fence.mbarrier_init.release.cluster;");
    __syncthreads();
    asm volatile("fence.mbarrier_init.release.cluster;");
    __syncthreads();
    const int64_t G = gridDim.x;
    const int64_t Rs = ((m + G - 1) / G + 1) & ~1ll;
    const int64_t nb = (n + C - 1) / C;
    // task list of this warp: (row, col) boxes
    int64_t ntask;
    if (pattern == 0) {
        const int64_t nr = (Rs + R - 1) / R;  // boxes per slab column block
        ntask = nb * nr;                      // split over the NR warps
    } else {
        ntask = ((m + R - 1) / R) * nb;
    }
    unsigned long long acc = 0;
    if (lane == 0) {
        int64_t it = 0;
        auto coords = [&](int64_t t, int& r, int& c) {
            if (pattern == 0) {
                const int64_t nr = (Rs + R - 1) / R;
                const int64_t b = t / nr, q = t - b * nr;
                r = (int)(blockIdx.x * Rs + q * R);
                c = (int)(b * C);
            } else {
                const int64_t G0 = (m + R - 1) / R;
                const int64_t b = t / G0, q = t - b * G0;
                r = (int)(q * R);
                c = (int)(b * C);
            }
        };
        // my tasks: pattern 0: t = warp, warp + NR, ... ; pattern 1: t = blockIdx * NR + warp + k * G * NR
        const int64_t t0 = pattern == 0 ? warp : blockIdx.x * NR + warp;
        const int64_t dt = pattern == 0 ? NR : G * NR;
        int64_t issued = 0, done = 0;
        int64_t tq = t0;
        for (; issued < NS && tq < ntask; ++issued, tq += dt) {
            int r, c;
            coords(tq, r, c);
            const int s = (int)(issued % NS);
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bars[s])), "r"(box));
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                    su(base + (size_t)s * box)),
                "l"(&tm), "r"(r), "r"(c), "r"(su(&bars[s]))
                : "memory");
        }
        while (done < issued) {
            const int s = (int)(done % NS);
            const uint32_t ph = (uint32_t)((done / NS) & 1);
            uint32_t ok = 0;
            while (!ok)
                asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                             : "=r"(ok)
                             : "r"(su(&bars[s])), "r"(ph)
                             : "memory");
            acc += *reinterpret_cast<volatile unsigned long long*>(base + (size_t)s * box);
            ++done;
            if (tq < ntask) {
                int r, c;
                coords(tq, r, c);
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bars[s])), "r"(box));
                asm volatile(
                    "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
                    "[%4];" ::"r"(su(base + (size_t)s * box)),
                    "l"(&tm), "r"(r), "r"(c), "r"(su(&bars[s]))
                    : "memory");
                ++issued;
                tq += dt;
            }
        }
    }
    if (acc == 0x1234567ull) *sink = acc;
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
    const int64_t m = atoll(argv[1]), n = atoll(argv[2]);
    const int R = atoi(argv[3]), C = atoi(argv[4]), NS = atoi(argv[5]), NR = atoi(argv[6]), pattern = atoi(argv[7]);
    const int NL = argc > 8 ? atoi(argv[8]) : 1;
    double* A;
    cudaMalloc(&A, sizeof(double) * m * n);
    cudaMemset(A, 0, sizeof(double) * m * n);
    unsigned long long* sink;
    cudaMalloc(&sink, 8);
    EncFn enc;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
    CUtensorMap tm;
    cuuint64_t dims[2] = {(cuuint64_t)m, (cuuint64_t)n};
    cuuint64_t str[1] = {(cuuint64_t)(m * 8)};
    cuuint32_t box[2] = {(cuuint32_t)R, (cuuint32_t)C};
    cuuint32_t es[2] = {1, 1};
    CUresult cr = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, A, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr) { printf("encode failed %d\n", cr); return 1; }
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const size_t smem = (size_t)NR * NL * NS * R * C * 8 + NR * NL * NS * 8;
    cudaFuncSetAttribute(k_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int rep = 0; rep < 4; ++rep) {
        cudaEventRecord(e0);
        k_stream<<<sms, 32 * NR, smem>>>(tm, m, n, R, C, NS, pattern, sink, NL);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep > 0 && ms < best) best = ms;
    }
    cudaError_t err = cudaGetLastError();
    printf("NL %d m %lld n %lld box %dx%d NS %d NR %d pattern %s smem %zu KB: %.3f ms  %.1f GB/s  %s\n", NL, (long long)m,
           (long long)n, R, C, NS, NR, pattern ? "panel" : "slab", smem / 1024, best,
           8.0 * m * n / (best * 1e-3) / 1e9, cudaGetErrorString(err));
    return 0;
}
