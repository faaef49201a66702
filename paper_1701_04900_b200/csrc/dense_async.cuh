// dense_async.cuh -- the fused asynchronous block-update kernel (dense A).
//
// Algorithm 1 [PAPER.md:246-260] on one B200.  Persistent CTAs are the
// asynchronous workers.  Work is handed out from ONE global atomic counter in
// units of "panel subtasks": subtask t = (sequence k = t / G, panel p = t % G),
// where sequence k updates block b = schedule(k) (S.1) and panel p covers
// rows [p*R, p*R+R) of that block's columns A_b: an R x B tile loaded by one
// 2-D TMA (cp.async.bulk.tensor, OOB rows/columns zero-filled) into a stage of
// an NS-deep shared-memory ring.  A panel is read from HBM exactly once and
// used for both the dot and the axpy.
//
// Warp roles (every role is per-warp, so 4 panels can be in each phase):
//   warp 0 (lane 0)  producer: claim t, arm the stage mbarrier, issue the TMA;
//   warps 1-4        dot: stage `it` is taken by dot warp it%4.  Guards, then
//                    w = phi'(r) on the panel rows (inconsistent read of the
//                    shared residual), A_{b,p}^T w (lane = rows, 32 column
//                    accumulators, butterfly transpose-reduction), publish;
//                    the LAST of the G panels of sequence k solves the block
//                    subproblem (Eq. 2, closed form) and applies (S.4) to x_b;
//   warps 5-8        axpy: stage `it` is taken by axpy warp it%4.  Wait for
//                    dx_b, push A_{b,p} dx_b into r (red.add), free the stage,
//                    then publish completion.
// Guards (all point to strictly older sequences -> deadlock free with
// co-resident CTAs):
//   * D4 freshness [PAPER.md:233]: the panel of block b is not read before the
//     previous update of b has been applied to those rows (ver[] counters);
//   * bounded delay D1 [PAPER.md:224]: sequence k does not read before
//     sequence k - delay - 1 is fully applied (done[] ring);
//   * slot reuse of the per-sequence accumulators.
// delay == 0 makes the kernel the sequential (d^k = 0) scheme and, with the
// fixed-order partial reduction (deterministic = 1), bit-reproducible.
#pragma once
#include <cuda.h>

#include "common.cuh"

namespace asy {

constexpr int kDotWarps = 4;
constexpr int kAxpyWarps = 4;
constexpr int kDenseThreads = 32 * (1 + kDotWarps + kAxpyWarps);
constexpr int kMaxRowsPerLane = 8;  // R <= 256 (one TMA box per panel)

struct DenseAsyncParams {
    int64_t m, n;
    int64_t B;      // block size
    int64_t nblk;   // number of blocks
    int64_t R;      // panel rows (multiple of 32, <= 256) = TMA box rows
    int64_t G;      // panels per block
    double* r;      // shared residual (LS: Ax-b, logistic: Ax)
    const double* aux;  // b (LS) or y (logistic)
    double* x;
    const double* tau;
    Scalars S;
    double gamma;
    int sched;
    uint64_t seed;
    int64_t epoch0;   // schedule epoch of sequence 0 of this launch
    int64_t T;        // subtasks in this launch = K*G
    int64_t delay;    // bounded delay window (>= 0)
    int deterministic;
    // synchronisation state (initialised by dense_async_init)
    unsigned long long* counter;
    double* gacc;        // [S][Bmax]
    double* dxr;         // [S][Bmax]
    double* part;        // [G][Bmax] (deterministic mode)
    unsigned* arrive;    // [S]
    unsigned* consumed;  // [S]
    long long* ready;    // [S]
    long long* done;     // [S]
    unsigned* ver;       // [nblk*G]
    int64_t slots;       // power of two
    int32_t Bmax;
    int32_t stages;
};

struct StageMeta {
    long long t, k, b, p;
};

__global__ void dense_async_init(DenseAsyncParams P) {
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    if (tid == 0) *P.counter = 0ull;
    for (int64_t s = tid; s < P.slots; s += nth) {
        P.arrive[s] = 0u;
        P.consumed[s] = (unsigned)P.G;
        P.ready[s] = (long long)s - (long long)P.slots;
        P.done[s] = (long long)s - (long long)P.slots;
    }
    for (int64_t i = tid; i < P.slots * P.Bmax; i += nth) P.gacc[i] = 0.0;
    for (int64_t i = tid; i < P.nblk * P.G; i += nth) P.ver[i] = 0u;
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar,
                                            uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
        "[%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}

__device__ __forceinline__ unsigned atom_add_acqrel_u32(unsigned* p, unsigned v) {
    unsigned old;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}
__device__ __forceinline__ void fence_acqrel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ long long ld_relaxed_s64(const long long* p) {
    long long v;
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned ld_relaxed_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Butterfly reduce-scatter: in: v[c] = this lane's partial of column c (32 columns);
// out: the returned value on lane l is the warp total of column l.  31 shuffles.
__device__ __forceinline__ double transpose_reduce32(double (&v)[32], int lane) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        const bool up = (lane & o) != 0;
#pragma unroll
        for (int i = 0; i < o; ++i) {
            const double send = up ? v[i] : v[i + o];
            const double keep = up ? v[i + o] : v[i];
            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
    }
    return v[0];
}

__global__ void __launch_bounds__(kDenseThreads, 1)
    dense_async_kernel(const __grid_constant__ CUtensorMap tmap, const DenseAsyncParams P) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    const int NS = P.stages;
    const int R = (int)P.R;
    const int Bmax = P.Bmax;
    const size_t PANEL = (size_t)R * Bmax;  // doubles per stage
    double* panels = reinterpret_cast<double*>(smem_raw);             // NS * PANEL
    double* wbuf = panels + NS * PANEL;                               // kDotWarps * R
    double* dxs = wbuf + kDotWarps * R;                               // kAxpyWarps * Bmax
    StageMeta* meta = reinterpret_cast<StageMeta*>(dxs + kAxpyWarps * Bmax);
    uint64_t* full = reinterpret_cast<uint64_t*>(meta + NS);
    uint64_t* empty = full + NS;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
        mbar_fence_init();
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmap) : "memory");
    }
    __syncthreads();
    const int rows_per_lane = R / 32;

    if (warp == 0) {
        // ------------------------------------------------------------------ producer
        if (lane != 0) return;
        const uint64_t pol = policy_evict_first();
        const uint32_t box_bytes = (uint32_t)(PANEL * 8);
        int ends = 0;
        for (long long it = 0;; ++it) {
            const int st = (int)(it % NS);
            if (it >= NS) mbar_wait(&empty[st], (uint32_t)(((it / NS) - 1) & 1));
            StageMeta& md = meta[st];
            long long t = -1;
            if (ends == 0) {
                t = (long long)atomicAdd(P.counter, 1ull);
                if (t >= P.T) t = -1;
            }
            if (t < 0) {  // one end marker for each of the 4 dot / 4 axpy warps
                md.t = -1;
                mbar_arrive(&full[st]);
                if (++ends == 4) break;
                continue;
            }
            const long long k = t / P.G, p = t - k * P.G;
            const long long b = schedule_block(P.sched, P.seed, P.nblk, P.epoch0 * P.nblk + k);
            md.t = t; md.k = k; md.b = b; md.p = p;
            mbar_arrive_expect_tx(&full[st], box_bytes);
            tma_load_2d(panels + st * PANEL, &tmap, (int)(p * R), (int)(b * P.B), &full[st], pol);
        }
        return;
    }

    if (warp <= kDotWarps) {
        // ------------------------------------------------------------------ dot warps
        const int dw = warp - 1;
        double* wv = wbuf + dw * R;
        for (long long it = dw;; it += kDotWarps) {
            const int st = (int)(it % NS);
            mbar_wait(&full[st], (uint32_t)((it / NS) & 1));
            const StageMeta md = meta[st];
            if (md.t < 0) break;
            const long long k = md.k, b = md.b, p = md.p;
            const long long slot = k & (P.slots - 1);
            const long long c0 = b * P.B;
            const int nc = (int)((P.n - c0) < P.B ? (P.n - c0) : P.B);
            const double* pan = panels + st * PANEL;
            // guards: three independent relaxed loads, one acquire fence
            if (lane == 0) {
                const unsigned u = (unsigned)(k / P.nblk);
                const long long kd = k - P.delay - 1;
                long long* donep = &P.done[kd & (P.slots - 1)];
                const long long rdy = ld_relaxed_s64(&P.ready[slot]);
                const unsigned ver = ld_relaxed_u32(&P.ver[b * P.G + p]);
                const long long dn = kd >= 0 ? ld_relaxed_s64(donep) : kd;
                if (rdy < k - P.slots) spin_until_ge(&P.ready[slot], k - P.slots);
                if (ver < u) spin_until_ge_u32(&P.ver[b * P.G + p], u);
                if (dn < kd) spin_until_ge(donep, kd);
                fence_acqrel_gpu();
            }
            __syncwarp();
            // w = phi'(r) on the panel rows: issue all loads first, then compute
            const long long r0 = p * R;
            double rv[kMaxRowsPerLane];
#pragma unroll
            for (int q = 0; q < kMaxRowsPerLane; ++q) {
                const long long row = r0 + lane + 32 * q;
                rv[q] = (q < rows_per_lane && row < P.m) ? ld_relaxed_f64(&P.r[row]) : 0.0;
            }
#pragma unroll
            for (int q = 0; q < kMaxRowsPerLane; ++q) {
                if (q < rows_per_lane) {
                    const long long row = r0 + lane + 32 * q;
                    wv[lane + 32 * q] = row < P.m ? loss_prime(P.S, rv[q], P.aux[row]) : 0.0;
                }
            }
            __syncwarp();
            // A_{b,p}^T w, 32 columns at a time
            for (int g0 = 0; g0 < nc; g0 += 32) {
                const int ncg = (nc - g0) < 32 ? (nc - g0) : 32;
                double acc[32];
#pragma unroll
                for (int c = 0; c < 32; ++c) acc[c] = 0.0;
                for (int q = 0; q < rows_per_lane; ++q) {
                    const int i = lane + 32 * q;
                    const double w = wv[i];
                    const double* a = pan + (size_t)g0 * R + i;
#pragma unroll
                    for (int c = 0; c < 32; ++c)
                        if (c < ncg) acc[c] = fma(a[(size_t)c * R], w, acc[c]);
                }
                const double colsum = transpose_reduce32(acc, lane);
                if (lane < ncg) {
                    if (P.deterministic) P.part[p * Bmax + g0 + lane] = colsum;
                    else atomicAdd(&P.gacc[slot * Bmax + g0 + lane], colsum);
                }
            }
            __syncwarp();
            unsigned last = 0;
            if (lane == 0) last = atom_add_acqrel_u32(&P.arrive[slot], 1u) == (unsigned)(P.G - 1);
            last = __shfl_sync(0xffffffffu, last, 0);
            if (last) {
                // last panel of sequence k: solve the block subproblem (Eq. 2) and apply (S.4)
                if (lane == 0) {
                    P.arrive[slot] = 0u;
                    spin_until_ge_u32(&P.consumed[slot], (unsigned)P.G);  // seq k-S fully applied
                    P.consumed[slot] = 0u;
                }
                __syncwarp();
                for (int c = lane; c < nc; c += 32) {
                    double g;
                    if (P.deterministic) {
                        g = 0.0;
                        for (long long q = 0; q < P.G; ++q) g += ld_relaxed_f64(&P.part[q * Bmax + c]);
                    } else {
                        g = ld_relaxed_f64(&P.gacc[slot * Bmax + c]);
                        P.gacc[slot * Bmax + c] = 0.0;
                    }
                    const long long j = c0 + c;
                    const double y = ld_relaxed_f64(&P.x[j]);
                    const double xh = best_response(P.S, g, y, P.tau[j], j);
                    const double xn = y + P.gamma * (xh - y);
                    P.x[j] = xn;
                    P.dxr[slot * Bmax + c] = xn - y;
                }
                __syncwarp();
                if (lane == 0) st_release_s64(&P.ready[slot], k);
            }
        }
        return;
    }

    // ---------------------------------------------------------------------- axpy warps
    const int aw = warp - 1 - kDotWarps;
    double* dv = dxs + aw * Bmax;
    for (long long it = aw;; it += kAxpyWarps) {
        const int st = (int)(it % NS);
        mbar_wait(&full[st], (uint32_t)((it / NS) & 1));
        const StageMeta md = meta[st];
        if (md.t < 0) break;
        const long long k = md.k, b = md.b, p = md.p;
        const long long slot = k & (P.slots - 1);
        const long long c0 = b * P.B;
        const int nc = (int)((P.n - c0) < P.B ? (P.n - c0) : P.B);
        const double* pan = panels + st * PANEL;
        if (lane == 0) spin_until_ge(&P.ready[slot], k);
        __syncwarp();
        bool nz = false;
        for (int c = lane; c < Bmax; c += 32) {
            const double d = c < nc ? ld_relaxed_f64(&P.dxr[slot * Bmax + c]) : 0.0;
            dv[c] = d;
            nz |= d != 0.0;
        }
        nz = __any_sync(0xffffffffu, nz);
        __syncwarp();
        const long long r0 = p * R;
        if (nz) {
            // rows_per_lane independent FMA chains (one per row), dx broadcast from smem
            double d[kMaxRowsPerLane];
#pragma unroll
            for (int q = 0; q < kMaxRowsPerLane; ++q) d[q] = 0.0;
            for (int c = 0; c < nc; ++c) {
                const double dc = dv[c];
                const double* a = pan + (size_t)c * R + lane;
#pragma unroll
                for (int q = 0; q < kMaxRowsPerLane; ++q)
                    if (q < rows_per_lane) d[q] = fma(a[32 * q], dc, d[q]);
            }
#pragma unroll
            for (int q = 0; q < kMaxRowsPerLane; ++q) {
                const long long row = r0 + lane + 32 * q;
                if (q < rows_per_lane && row < P.m && d[q] != 0.0) atomicAdd(&P.r[row], d[q]);
            }
        }
        __syncwarp();
        if (lane == 0) {
            mbar_arrive(&empty[st]);  // smem stage free; the red.adds may still be in flight
            fence_acqrel_gpu();       // ... and are performed before the completion counters move
            atomicAdd(&P.ver[b * P.G + p], 1u);
            const unsigned old = atomicAdd(&P.consumed[slot], 1u);
            if (old == (unsigned)(P.G - 1)) st_release_s64(&P.done[slot], k);
        }
    }
}

}  // namespace asy
