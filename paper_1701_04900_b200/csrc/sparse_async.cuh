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
    double* r;         // the residual's pair buffer [r_i, aux_i] (2 m doubles; r_i at 2 i)
    const double* aux; // (unused by the kernel: aux_i is at r[2 i + 1])
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

__device__ __forceinline__ unsigned ld_relaxed_u32_g(const unsigned* p) {
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ long long ld_relaxed_s64_g(const long long* p) {
    long long v;
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void red_relaxed_max_s64_g(long long* p, long long v) {
    asm volatile("red.relaxed.gpu.global.max.s64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void red_relaxed_u32_g(unsigned* p, unsigned v) {
    asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// relaxed polls (an acquire per poll would invalidate the SM's L1); the caller fences once
__device__ __forceinline__ void spin_relaxed_u32_g(const unsigned* p, unsigned v) {
    unsigned ns = 32;
    while (ld_relaxed_u32_g(p) < v) {
        __nanosleep(ns);
        if (ns < 256) ns <<= 1;
    }
}
__device__ __forceinline__ void spin_relaxed_s64_g(const long long* p, long long v) {
    unsigned ns = 32;
    while (ld_relaxed_s64_g(p) < v) {
        __nanosleep(ns);
        if (ns < 256) ns <<= 1;
    }
}

// residual and b / y interleaved for the launch (one 16-byte gather per nonzero), and back
__global__ void sparse_pair_pack(const double* r, const double* aux, double* ry, int64_t m) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        ry[2 * i] = r[i];
        ry[2 * i + 1] = aux[i];
    }
}
__global__ void sparse_pair_unpack(const double* ry, double* r, int64_t m) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
        r[i] = ry[2 * i];
}
__device__ __forceinline__ double2 ld_relaxed_f64x2(const double* p) {
    double2 v;
    asm volatile("ld.relaxed.gpu.global.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p) : "memory");
    return v;
}

__global__ void sparse_async_init(SparseAsyncParams P) {
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    if (tid == 0) *P.counter = 0ull;
    for (int64_t s = tid; s < P.slots; s += nth) P.done[s] = (long long)s - (long long)P.slots;
    for (int64_t j = tid; j < P.n; j += nth) P.ver[j] = 0u;
}

// One block update's dependency chain is a few L2 round trips, so the kernel is arranged
// to issue independent loads together: the guard loads, colptr, and (after colptr) the
// column's row indices / values and x_j, tau_j are in flight at once; the residual is
// gathered only after the guards passed.  No 64-bit division per update (the epoch and
// position advance incrementally), one fence per update (after the scatter, before the
// version / window counters; deferred to overlap the next update's loads), no returning
// atomics on the path, the loss fixed at compile time.
#ifndef ASY_SPARSE_MINB
#define ASY_SPARSE_MINB 1
#endif
#ifndef ASY_SPARSE_THREADS
#define ASY_SPARSE_THREADS 128  // small CTAs: finer occupancy granularity at ~87 registers
#endif
constexpr int kSparseThreads = ASY_SPARSE_THREADS;
template <int LOSS>
__global__ void __launch_bounds__(kSparseThreads, ASY_SPARSE_MINB) sparse_async_kernel(SparseAsyncParams P) {
    const int lane = threadIdx.x & 31;
    const int grp = lane >> 3, gl = lane & 7;
    const unsigned gmask = 0xFFu << (grp * 8);
    const int64_t N = P.n;
    const int half = perm_half_bits(N);
    PermKeys pk{};
    int64_t pkE = -1;
    // completion of the group's previous update (fence, then its version and window counters),
    // issued once the next update's first loads are in flight; never deferred across a wait
    bool pend = false;
    int64_t pj = 0;
    long long pkk = 0;
    auto flush = [&]() {
        if (pend && gl == 0) {
            asm volatile("fence.acq_rel.gpu;" ::: "memory");  // its scatter and x_j first
            red_relaxed_u32_g(&P.ver[pj], 1u);
            red_relaxed_max_s64_g(&P.done[pkk & (P.slots - 1)], pkk);  // monotone window counter
        }
        pend = false;
    };
    for (;;) {
        long long base = 0;
        if (lane == 0) base = (long long)atomicAdd(P.counter, (unsigned long long)P.chunk);
        base = __shfl_sync(0xffffffffu, base, 0);
        if (base >= P.K) break;
        const long long kend = (base + P.chunk) < P.K ? (base + P.chunk) : P.K;
        // local epoch u and position i of this group's first sequence (one division per chunk)
        long long k = base + grp;
        int64_t u = k / N, i = k - u * N;
        // the head of an update: its column (S.1), guard counters and column extent; the
        // next update's head is loaded while the current one runs (counters are monotone, so an
        // early read can only be stale-low: the guard then re-polls)
        struct Head { int64_t j, s, e; unsigned vj; long long dn; };
        auto head = [&](long long kk, int64_t ii, int64_t uu) {
            Head hd;
            hd.j = ii;
            if (P.sched == SCHED_RANDOM) {
                const int64_t E = P.epoch0 + uu;
                if (E != pkE) { pk = perm_keys(P.seed, E); pkE = E; }
                uint64_t v = (uint64_t)ii;
                do { v = feistel(v, half, pk); } while (v >= (uint64_t)N);
                hd.j = (int64_t)v;
            }
            const long long kd = kk - P.delay - 1;
            hd.vj = 0;
            hd.dn = 0;
            if (gl == 0) {
                hd.vj = ld_relaxed_u32_g(&P.ver[hd.j]);
                if (kd >= 0) hd.dn = ld_relaxed_s64_g(&P.done[kd & (P.slots - 1)]);
            }
            hd.s = __ldg(&P.colptr[hd.j]);
            hd.e = __ldg(&P.colptr[hd.j + 1]);
            return hd;
        };
        Head nx{};
        if (k < kend) nx = head(k, i, u);
        for (; k < kend; k += 4) {
            const Head cur = nx;
            const int64_t j = cur.j, s = cur.s, e = cur.e;
            const long long kd = k - P.delay - 1;
            const unsigned vj = cur.vj;
            const long long dn = cur.dn;
            // this lane's first two nonzeros (columns of up to 16 in one round trip; ~10 on
            // average in configs[4]) and the block's x / tau (x_j final once ver[j] == u)
            int32_t row0 = 0, row1 = 0;
            double val0 = 0.0, val1 = 0.0;
            if (s + gl < e) {
                row0 = __ldg(&P.rowidx[s + gl]);
                val0 = __ldg(&P.vals[s + gl]);
            }
            if (s + gl + 8 < e) {
                row1 = __ldg(&P.rowidx[s + gl + 8]);
                val1 = __ldg(&P.vals[s + gl + 8]);
            }
            const int64_t ucur = u;
            i += 4;
            while (i >= N) { i -= N; ++u; }
            if (k + 4 < kend) nx = head(k + 4, i, u);
            double tj = 0.0;
            if (gl == 0) {
                tj = __ldg(&P.tau[j]);
                const bool ok4 = vj >= (unsigned)ucur, ok1 = kd < 0 || dn >= kd;
                if (!ok4 || !ok1) {
                    flush();  // (the awaited update may be this group's pending one)
                    if (!ok4) spin_relaxed_u32_g(&P.ver[j], (unsigned)ucur);                   // D4
                    if (!ok1) spin_relaxed_s64_g(&P.done[kd & (P.slots - 1)], kd);             // D1
                    asm volatile("fence.acq_rel.gpu;" ::: "memory");
                }
            }
            flush();
            __syncwarp(gmask);
            double xj = 0.0;
            if (gl == 0) xj = ld_relaxed_f64(&P.x[j]);
            // gradient: sum_q a_qj phi'(r_q) over the column (inconsistent read of r)
            double acc = 0.0;
            {
                double2 ra0 = make_double2(0.0, 0.0), ra1 = make_double2(0.0, 0.0);
                if (s + gl < e) ra0 = ld_relaxed_f64x2(&P.r[2 * (int64_t)row0]);
                if (s + gl + 8 < e) ra1 = ld_relaxed_f64x2(&P.r[2 * (int64_t)row1]);
                if (s + gl < e) acc = val0 * loss_prime_t<LOSS>(P.S, ra0.x, ra0.y);
                if (s + gl + 8 < e) acc = fma(val1, loss_prime_t<LOSS>(P.S, ra1.x, ra1.y), acc);
            }
            for (int64_t q = s + gl + 16; q < e; q += 8) {
                const int32_t row = __ldg(&P.rowidx[q]);
                const double2 ra = ld_relaxed_f64x2(&P.r[2 * (int64_t)row]);
                acc = fma(__ldg(&P.vals[q]), loss_prime_t<LOSS>(P.S, ra.x, ra.y), acc);
            }
            acc += __shfl_xor_sync(gmask, acc, 4);
            acc += __shfl_xor_sync(gmask, acc, 2);
            acc += __shfl_xor_sync(gmask, acc, 1);
            double d = 0.0;
            if (gl == 0) {
                const double xh = best_response(P.S, acc, xj, tj, j);
                const double xn = xj + P.gamma * (xh - xj);
                P.x[j] = xn;
                d = xn - xj;
            }
            d = __shfl_sync(gmask, d, grp * 8);
            if (d != 0.0) {
                if (s + gl < e) atomicAdd(&P.r[2 * (int64_t)row0], val0 * d);
                if (s + gl + 8 < e) atomicAdd(&P.r[2 * (int64_t)row1], val1 * d);
                for (int64_t q = s + gl + 16; q < e; q += 8)
                    atomicAdd(&P.r[2 * (int64_t)__ldg(&P.rowidx[q])], __ldg(&P.vals[q]) * d);
            }
            __syncwarp(gmask);  // (orders the group's atomics before lane 0's later fence)
            pend = true;
            pj = j;
            pkk = k;
        }
        // before the warp-wide claim: another group of this warp may be waiting for it
        flush();
        __syncwarp();
    }
}

}  // namespace asy
