// sparse_async.cuh -- asynchronous scalar-block updates on a CSC matrix.
//
// Algorithm 1 [PAPER.md:246-260] with N = n scalar blocks (the paper's own
// setting, "always setting N=n" [PAPER.md:382]).  Persistent warps claim
// chunks of sequence numbers from one global atomic counter; each 8-lane
// group of a warp performs one block update at a time: gather the column's
// nonzeros, read the shared residual at those rows (inconsistent read),
// phi'(r) . a_j with a shuffle reduction, closed-form best response (Eq. 2),
// (S.4) on x_j, and scatter a_j * dx_j back into r with atomicAdd.
// Guards: D4 freshness (ver[j] = number of applied updates of column j) and
// the bounded-delay window D1 (done[] ring), both pointing to older sequences.
#pragma once
#include "common.cuh"

namespace asy {

struct SparseAsyncParams {
    const int64_t* __restrict__ colptr;
    const int32_t* __restrict__ rowidx;
    const double* __restrict__ vals;
    int64_t m, n;
    double* r;
    const double* aux;
    double* x;
    const double* tau;
    Scalars S;
    double gamma;
    int sched;
    uint64_t seed;
    int64_t epoch0;
    int64_t K;        // block updates in this launch
    int64_t delay;
    unsigned long long* counter;
    unsigned* ver;    // [n]
    long long* done;  // [slots]
    int64_t slots;
    int chunk;
};

__global__ void sparse_async_init(SparseAsyncParams P) {
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    if (tid == 0) *P.counter = 0ull;
    for (int64_t s = tid; s < P.slots; s += nth) P.done[s] = (long long)s - (long long)P.slots;
    for (int64_t j = tid; j < P.n; j += nth) P.ver[j] = 0u;
}

__global__ void __launch_bounds__(256) sparse_async_kernel(SparseAsyncParams P) {
    const int lane = threadIdx.x & 31;
    const int grp = lane >> 3, gl = lane & 7;
    const unsigned gmask = 0xFFu << (grp * 8);
    for (;;) {
        long long base = 0;
        if (lane == 0) base = (long long)atomicAdd(P.counter, (unsigned long long)P.chunk);
        base = __shfl_sync(0xffffffffu, base, 0);
        if (base >= P.K) break;
        const long long kend = (base + P.chunk) < P.K ? (base + P.chunk) : P.K;
        for (long long k = base + grp; k < kend; k += 4) {
            const long long j = schedule_block(P.sched, P.seed, P.n, P.epoch0 * P.n + k);
            if (gl == 0) {
                spin_until_ge_u32(&P.ver[j], (unsigned)(k / P.n));                 // D4
                const long long kd = k - P.delay - 1;
                if (kd >= 0) spin_until_ge(&P.done[kd & (P.slots - 1)], kd);      // D1 window
            }
            __syncwarp(gmask);
            const int64_t s = P.colptr[j], e = P.colptr[j + 1];
            double acc = 0.0;
            for (int64_t q = s + gl; q < e; q += 8) {
                const int32_t row = P.rowidx[q];
                acc = fma(P.vals[q], loss_prime(P.S, ld_relaxed_f64(&P.r[row]), P.aux[row]), acc);
            }
            acc += __shfl_xor_sync(gmask, acc, 4);
            acc += __shfl_xor_sync(gmask, acc, 2);
            acc += __shfl_xor_sync(gmask, acc, 1);
            double d = 0.0;
            if (gl == 0) {
                const double y = ld_relaxed_f64(&P.x[j]);
                const double xh = best_response(P.S, acc, y, P.tau[j], j);
                const double xn = y + P.gamma * (xh - y);
                P.x[j] = xn;
                d = xn - y;
            }
            d = __shfl_sync(gmask, d, grp * 8);
            if (d != 0.0) {
                for (int64_t q = s + gl; q < e; q += 8) atomicAdd(&P.r[P.rowidx[q]], P.vals[q] * d);
                __threadfence();
            }
            __syncwarp(gmask);
            if (gl == 0) {
                __threadfence();
                st_release_u32(&P.ver[j], (unsigned)(k / P.n) + 1u);
                atomicMax(&P.done[k & (P.slots - 1)], k);  // monotone: a late older seq never regresses it
            }
        }
        __syncwarp();
    }
}

}  // namespace asy
