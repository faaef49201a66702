// dense_async.cuh -- the fused asynchronous block-update kernel (dense A).
//
// Algorithm 1 [PAPER.md:246-260] on one B200.  Persistent CTAs are the
// asynchronous workers.  Work is handed out from ONE global atomic counter in
// units of "panel subtasks": subtask t = (sequence k = t / G, panel p = t % G),
// where sequence k updates block b = schedule(k) (S.1) and panel p covers
// rows [p*R, p*R+R) of that block's columns A_b (R x |b| doubles, one
// contiguous bulk copy per column, staged in shared memory by the TMA engine).
//
// Each CTA runs three warp roles over an NS-stage shared-memory ring:
//   producer (1 warp):  claim t -> cp.async.bulk the panel into a free stage;
//   dot warps (4):      w = phi'(r) on the panel rows (inconsistent read of the
//                       shared residual), partial A_{b,p}^T w per column
//                       (warp-shuffle reductions), publish; the LAST of the G
//                       panels of sequence k solves the block subproblem
//                       (Eq. 2 closed form) and applies (S.4) to x_b;
//   axpy warps (4):     wait for dx_b, push A_{b,p} dx_b into r (atomicAdd),
//                       release the stage.
// A panel is read from HBM exactly once and used for both the dot and the
// axpy.  Guards (all point to strictly older sequences -> deadlock free with
// co-resident CTAs):
//   * D4 freshness [PAPER.md:233]: the panel of block b is not read before the
//     previous update of b has been applied to those rows (ver[] counters);
//   * bounded delay D1 [PAPER.md:224]: sequence k does not read before
//     sequence k - delay - 1 is fully applied (done[] ring);
//   * slot reuse of the per-sequence accumulators.
// delay == 0 makes the kernel the sequential (d^k = 0) scheme and, with the
// fixed-order partial reduction (deterministic = 1), bit-reproducible.
#pragma once
#include "common.cuh"

namespace asy {

constexpr int kDotWarps = 4;
constexpr int kAxpyWarps = 4;
constexpr int kDenseThreads = 32 * (1 + kDotWarps + kAxpyWarps);

struct DenseAsyncParams {
    const double* __restrict__ A;
    int64_t lda, m, n;
    int64_t B;      // block size
    int64_t nblk;   // number of blocks
    int64_t R;      // panel rows (even)
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
    // synchronisation state (zeroed / initialised by dense_async_init)
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
    long long t, k, b, p, nr, nc;
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

__global__ void __launch_bounds__(kDenseThreads, 1) dense_async_kernel(DenseAsyncParams P) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int NS = P.stages;
    const int64_t R = P.R;
    const int Bmax = P.Bmax;
    // carve shared memory
    double* panels = reinterpret_cast<double*>(smem_raw);                 // NS * R * Bmax
    double* wbuf = panels + (size_t)NS * R * Bmax;                          // R
    double* dxs = wbuf + R;                                                 // Bmax
    StageMeta* meta = reinterpret_cast<StageMeta*>(dxs + Bmax);             // NS
    uint64_t* full = reinterpret_cast<uint64_t*>(meta + NS);                // NS
    uint64_t* empty = full + NS;                                            // NS
    __shared__ int s_flag;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
        mbar_fence_init();
    }
    __syncthreads();

    if (warp == 0) {
        // ------------------------------------------------------------ producer
        if (lane == 0) {
            const uint64_t pol = policy_evict_first();
            for (long long it = 0;; ++it) {
                const int st = (int)(it % NS);
                if (it >= NS) mbar_wait(&empty[st], (uint32_t)(((it / NS) - 1) & 1));
                const long long t = (long long)atomicAdd(P.counter, 1ull);
                StageMeta& md = meta[st];
                if (t >= P.T) {
                    md.t = -1;
                    mbar_arrive(&full[st]);
                    break;
                }
                const long long k = t / P.G, p = t - k * P.G;
                const long long b = schedule_block(P.sched, P.seed, P.nblk, P.epoch0 * P.nblk + k);
                const long long r0 = p * R;
                const long long nr = (P.m - r0) < R ? (P.m - r0) : R;
                const long long c0 = b * P.B;
                const long long nc = (P.n - c0) < P.B ? (P.n - c0) : P.B;
                const long long nrc = (nr + 1) & ~1ll;  // 16-byte multiple (lda even)
                md.t = t; md.k = k; md.b = b; md.p = p; md.nr = nr; md.nc = nc;
                mbar_arrive_expect_tx(&full[st], (uint32_t)(nrc * nc * 8));
                double* dst = panels + (size_t)st * R * Bmax;
                const double* src = P.A + c0 * P.lda + r0;
                for (long long c = 0; c < nc; ++c)
                    bulk_g2s(dst + c * R, src + c * P.lda, (uint32_t)(nrc * 8), &full[st], pol);
            }
        }
    } else if (warp <= kDotWarps) {
        // ------------------------------------------------------------ dot warps
        const int dw = warp - 1;
        const int dtid = threadIdx.x - 32;
        const int nthr = 32 * kDotWarps;
        for (long long it = 0;; ++it) {
            const int st = (int)(it % NS);
            mbar_wait(&full[st], (uint32_t)((it / NS) & 1));
            const StageMeta md = meta[st];
            if (md.t < 0) break;
            const long long k = md.k, b = md.b, p = md.p, nr = md.nr, nc = md.nc;
            const long long slot = k & (P.slots - 1);
            const double* pan = panels + (size_t)st * R * Bmax;
            if (dtid == 0) {
                spin_until_ge(&P.ready[slot], k - P.slots);                     // slot free
                const unsigned u = (unsigned)(k / P.nblk);
                spin_until_ge_u32(&P.ver[b * P.G + p], u);                       // D4
                const long long kd = k - P.delay - 1;
                if (kd >= 0) spin_until_ge(&P.done[kd & (P.slots - 1)], kd);     // D1 window
            }
            named_bar_sync(1, nthr);
            const long long r0 = p * R;
            for (long long i = dtid; i < nr; i += nthr)
                wbuf[i] = loss_prime(P.S, ld_relaxed_f64(&P.r[r0 + i]), P.aux[r0 + i]);
            named_bar_sync(1, nthr);
            for (long long c = dw; c < nc; c += kDotWarps) {
                const double* col = pan + c * R;
                double acc = 0.0;
                for (long long i = lane; i < nr; i += 32) acc = fma(col[i], wbuf[i], acc);
                acc = warp_sum(acc);
                if (lane == 0) {
                    if (P.deterministic) P.part[p * Bmax + c] = acc;
                    else atomicAdd(&P.gacc[slot * Bmax + c], acc);
                    __threadfence();
                }
            }
            named_bar_sync(1, nthr);
            if (dtid == 0) {
                __threadfence();
                const unsigned old = atomicAdd(&P.arrive[slot], 1u);
                s_flag = (old == (unsigned)(P.G - 1));
            }
            named_bar_sync(1, nthr);
            if (s_flag) {
                // last panel of sequence k: solve the block subproblem (Eq. 2)
                if (dtid == 0) {
                    __threadfence();
                    P.arrive[slot] = 0u;
                    spin_until_ge_u32(&P.consumed[slot], (unsigned)P.G);  // seq k-S fully applied
                    P.consumed[slot] = 0u;
                }
                named_bar_sync(1, nthr);
                for (long long c = dtid; c < nc; c += nthr) {
                    double g;
                    if (P.deterministic) {
                        g = 0.0;
                        for (long long q = 0; q < P.G; ++q) g += ld_relaxed_f64(&P.part[q * Bmax + c]);
                    } else {
                        g = ld_relaxed_f64(&P.gacc[slot * Bmax + c]);
                        P.gacc[slot * Bmax + c] = 0.0;
                    }
                    const long long j = b * P.B + c;
                    const double y = ld_relaxed_f64(&P.x[j]);
                    const double xh = best_response(P.S, g, y, P.tau[j], j);
                    const double xn = y + P.gamma * (xh - y);
                    P.x[j] = xn;
                    P.dxr[slot * Bmax + c] = xn - y;
                }
                named_bar_sync(1, nthr);
                if (dtid == 0) {
                    __threadfence();
                    st_release_s64(&P.ready[slot], k);
                }
            }
        }
    } else {
        // ------------------------------------------------------------ axpy warps
        const int atid = threadIdx.x - 32 * (1 + kDotWarps);
        const int nthr = 32 * kAxpyWarps;
        for (long long it = 0;; ++it) {
            const int st = (int)(it % NS);
            mbar_wait(&full[st], (uint32_t)((it / NS) & 1));
            const StageMeta md = meta[st];
            if (md.t < 0) break;
            const long long k = md.k, b = md.b, p = md.p, nr = md.nr, nc = md.nc;
            const long long slot = k & (P.slots - 1);
            const double* pan = panels + (size_t)st * R * Bmax;
            if (atid == 0) spin_until_ge(&P.ready[slot], k);
            named_bar_sync(2, nthr);
            for (long long c = atid; c < nc; c += nthr) dxs[c] = ld_relaxed_f64(&P.dxr[slot * Bmax + c]);
            named_bar_sync(2, nthr);
            const long long r0 = p * R;
            for (long long i = atid; i < nr; i += nthr) {
                double d = 0.0;
                for (long long c = 0; c < nc; ++c) d = fma(pan[c * R + i], dxs[c], d);
                if (d != 0.0) atomicAdd(&P.r[r0 + i], d);
            }
            named_bar_sync(2, nthr);
            if (atid == 0) {
                __threadfence();
                atomicAdd(&P.ver[b * P.G + p], 1u);
                const unsigned old = atomicAdd(&P.consumed[slot], 1u);
                if (old == (unsigned)(P.G - 1)) {
                    __threadfence();
                    st_release_s64(&P.done[slot], k);
                }
                mbar_arrive(&empty[st]);
            }
        }
    }
}

}  // namespace asy
