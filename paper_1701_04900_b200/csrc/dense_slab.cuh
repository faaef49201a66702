// dense_slab.cuh -- the asynchronous block-update kernel for dense A, row-slab form.
//
// Algorithm 1 [PAPER.md:246-260] on one B200.  One persistent CTA per SM owns a
// fixed slab of rows [row0, row0 + rows) of A, of the shared residual r and of
// b / y; the slab of r lives in shared memory for the whole launch (no other SM
// ever touches it, so the residual needs no atomics at all).  Every block
// update ("sequence" k, block b = schedule(k), (S.1)) is computed by all CTAs
// together:
//   dot    (S.2 gradient)  g_b += A[slab, b]^T phi'(r_slab)   -- the CTA's partial
//   publish               red.add of the partial into gacc[k] + release arrival
//   solve  (S.2 / S.3)    once all CTAs arrived: hat x_b (Eq. 2 closed form),
//                          (S.4) x_b += gamma (hat x_b - x_b), dx_b -- every CTA
//                          computes the same numbers; CTA k mod grid stores x_b
//   axpy   (S.4 pushed)   r_slab += A[slab, b] dx_b
// Sequences are pipelined: the dot of sequence k may run while the all-reduces
// of up to `delay` older sequences are in flight -- exactly the inconsistent
// read of Algorithm 1 (r_slab then lacks their contributions), with the
// bounded delay of Assumption D1 [PAPER.md:224] enforced per CTA:
//     dot(k) starts only after axpy(k - delay - 1) was applied to r_slab;
// and D4 [PAPER.md:233] (own block read fresh):
//     dot(k) starts only after axpy(kprev) was applied, kprev = previous update
//     of the same block (schedule_prev).
// delay == 0 is the sequential (d^k = 0) scheme; with the fixed-order partial
// reduction (deterministic = 1) it is bit-reproducible.
//
// The slab tile of sequence k is loaded as nch chunks of Rc rows (TMA boxes
// Rc x B).  Chunks are numbered c = k * nch + ch across the launch.
// Warp roles (512 threads):
//   warp 0       dot producer and the only evaluator of the schedule: writes the
//                sequence's metadata, TMA-loads chunk c into dot warp (c mod 4)'s
//                sub-ring of stages;
//   warp 1       axpy producer (hold == 0): re-loads the chunks (L2 hits: the dot
//                pass brought them in shortly before) into the axpy ring; idle when
//                hold == 1 (the axpy reads the dot stage);
//   warps 2-5    dot: warp w takes the chunks c = w mod 4 (all columns; lanes run
//                over the chunk rows, butterfly transpose-reduction) and writes its
//                partial of sequence k to its own slot (fixed-order sum later);
//   warps 6-9    axpy: warp a owns the slab rows of the (chunk, 32-row group) items
//                = a mod 4 and applies every sequence to them in order;
//                progress[a] = sequences applied by it;
//   warps 10-15  sequence warps: warp 10 + (k mod 6) sums the CTA's partial of
//                sequence k, publishes it, waits for all CTAs, reads the reduced
//                gradient and x_b, solves, hands dx_b to the axpy warps.  Six of
//                them keep six global all-reduces in flight per CTA.
// Every mbarrier stage has a single consumer warp (or all four of a role in the
// same order), so parity waits never alias across phases.
// Slot reuse: sequence k uses gacc slot k mod S, double-buffered per use; the
// half of the slot's next user is zeroed by the solves of sequence k.  S >=
// 2*delay + 2 makes both safe (a CTA publishing k+S has seen arrival(k+S-delay-1),
// so every CTA has finished the solve of k).
#pragma once
#include <cuda.h>

#include "common.cuh"

namespace asy {

constexpr int kSlabDot = 4;
constexpr int kSlabAx = 4;
constexpr int kSlabSeq = 6;
constexpr int kSlabDot0 = 2;
constexpr int kSlabAx0 = kSlabDot0 + kSlabDot;
constexpr int kSlabSeq0 = kSlabAx0 + kSlabAx;
constexpr int kSlabWarps = kSlabSeq0 + kSlabSeq;
constexpr int kSlabThreads = 32 * kSlabWarps;
constexpr int kSlabNP = kSlabSeq;   // partial ring: slot k mod 6 <-> sequence warp k mod 6
constexpr int kSlabNDX = kSlabSeq;  // dx ring
// All-reduce layout: CTA c adds its partial into replica c mod kGaccRep of the slot (148 CTAs
// adding into one copy serialise ~150 fp64 atomics per address on a few L2 slices); readers
// sum the replicas.  Arrival counters sit one per 128-byte line (hundreds of warps poll them).
#ifndef ASY_GACC_REP
#define ASY_GACC_REP 8
#endif
constexpr int kGaccRep = ASY_GACC_REP;
constexpr int kArrivePad = 32;
constexpr int kSlabMaxStages = 24;
constexpr int kSlabPad = 32;        // zero doubles after each stage (reads past the last column)

struct SlabParams {
    int64_t m, n, B, nblk;
    int64_t Rs;        // rows per CTA slab (last CTA: fewer)
    int Rc;            // chunk rows (TMA box rows, even, <= 256)
    int nch;           // chunks per sequence: nch * Rc >= Rs
    int hold;          // 1: the axpy reads the dot stage; 0: re-loaded into the axpy ring
    int nst, nsa;      // dot / axpy ring stages
    int64_t stage_dbl; // doubles per stage (>= Rc * BMAX + kSlabPad)
    double* r;         // global residual (LS: Ax-b, logistic: Ax), loaded / stored per slab
    const double* aux; // b (LS) or y (logistic)
    double* x0;        // x read in even local epochs (written in odd ones)
    double* x1;
    const double* tau;
    Scalars S;
    double gamma;
    int sched;
    uint64_t seed;
    int64_t epoch0;    // schedule epoch of sequence 0 of this launch
    int64_t K;         // sequences in this launch
    int64_t delay;     // bounded delay (effective)
    int deterministic;
    double* gacc;      // [S][2][kGaccRep][B]
    double* part;      // [S][grid][B]   (deterministic)
    unsigned* arrive;  // [S * kArrivePad] monotonic (slot s at s * kArrivePad)
    int64_t slots;     // S, power of two, >= 2*delay + 2
    unsigned long long* prof;  // optional [grid][kSlabWarps][8] clock64 segment sums
    // TMEM-parking form only (dense_slabt.cuh)
    const double* A;   // column-major, for the 1-D bulk copies of a slab's ragged last row group
    int64_t lda;
    int npark[4];      // park ring per dot warp d: TMEM slots (256 / BMAX) + its smem hold slots
    int hoff[4];       // first smem hold slot of dot warp d
    int rotate;        // the slab's last, partial round of row groups rotates over the warps per sequence
    unsigned* dobs;    // max observed delay (earlier sequences missing from a read), atomicMax; may be null
};

__global__ void slab_init(SlabParams P) {
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    for (int64_t s = tid; s < P.slots; s += nth) P.arrive[s * kArrivePad] = 0u;
    for (int64_t i = tid; i < 2 * P.slots * kGaccRep * P.B; i += nth) P.gacc[i] = 0.0;
}

__device__ __forceinline__ void slab_tma_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar,
                                            uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
        "[%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ unsigned ld_relaxed_gpu_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long ld_acquire_cta_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.cta.shared.b64 %0, [%1];" : "=l"(v) : "r"(smem_u32(p)) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_cta_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.cta.shared.b64 [%0], %1;" ::"r"(smem_u32(p)), "l"(v) : "memory");
}
__device__ __forceinline__ void red_release_gpu_u32(unsigned* p, unsigned v) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// Poll a counter other SMs increment with release semantics.  A strong relaxed load
// (L2) instead of ld.acquire: acquire would invalidate this SM's whole L1 on every
// poll (CCTL.IVALL), which stalls the shared-memory pipe of all warps.  Everything
// read after it that other SMs wrote is read with strong (.relaxed.gpu, L2) loads,
// so no stale L1 line can be observed.
__device__ __forceinline__ void spin_until_ge_relaxed_u32(const unsigned* p, unsigned v) {
    unsigned ns = 32;
    while (ld_relaxed_gpu_u32(p) < v) {
        __nanosleep(ns);
        if (ns < 256) ns <<= 1;
    }
}
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

// Butterfly reduce-scatter over 16 columns: lanes l and l ^ 16 return column (l & 15)'s total.
__device__ __forceinline__ double slab_reduce16(double* v, int lane) {
#pragma unroll
    for (int o = 8; o >= 1; o >>= 1) {
        const bool up = (lane & o) != 0;
#pragma unroll
        for (int i = 0; i < o; ++i) {
            const double send = up ? v[i] : v[i + o];
            const double keep = up ? v[i + o] : v[i];
            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
    }
    return v[0] + __shfl_xor_sync(0xffffffffu, v[0], 16);
}

// Butterfly reduce-scatter over 8 columns: lanes with l & 7 == c return column c's total.
__device__ __forceinline__ double slab_reduce8(double* v, int lane) {
#pragma unroll
    for (int o = 4; o >= 1; o >>= 1) {
        const bool up = (lane & o) != 0;
#pragma unroll
        for (int i = 0; i < o; ++i) {
            const double send = up ? v[i] : v[i + o];
            const double keep = up ? v[i + o] : v[i];
            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
    }
    const double t = v[0] + __shfl_xor_sync(0xffffffffu, v[0], 8);
    return t + __shfl_xor_sync(0xffffffffu, t, 16);
}

// (compiled in only with -DASY_SEGPROF -- a profiling build, `build.py --variant prof
// ASY_SEGPROF`, loaded with ASY_LIB_VARIANT=prof; otherwise every call is empty)
struct SlabProf {
#ifdef ASY_SEGPROF
    unsigned long long seg[8];
    long long last;
    __device__ void start() {
        for (int i = 0; i < 8; ++i) seg[i] = 0;
        last = clock64();
    }
    __device__ void mark(int i) {
        const long long t = clock64();
        seg[i] += (unsigned long long)(t - last);
        last = t;
    }
    __device__ void flush(unsigned long long* out, int lane) {
        if (out && lane == 0)
            for (int i = 0; i < 8; ++i) out[i] = seg[i];
    }
#else
    __device__ void start() {}
    __device__ void mark(int) {}
    __device__ void flush(unsigned long long*, int) {}
#endif
};

// Per-sequence metadata, written once by the dot producer (the only thread that
// evaluates the schedule), read by the dot and sequence warps.
struct SeqMeta {
    int64_t need;  // dot(k) may start once applied >= need  (D1: k - delay, D4: kprev + 1)
    int32_t b;     // block (S.1)
    int32_t flags; // bit 0: local epoch parity (x double buffer), bit 1: this CTA stores x_b
};
constexpr int kSlabNM = 256;  // metadata ring (power of two, > delay + stages + sequence warps)

// ring position: slot index and mbarrier phase advanced without divisions
struct RingPos {
    int i, n;
    uint32_t ph;
    __device__ void init(int n_) { i = 0; n = n_; ph = 0; }
    __device__ void next() {
        if (++i == n) { i = 0; ph ^= 1u; }
    }
};

// The schedule walk of one CTA's producer (S.1): block b of sequence k, the index of
// the previous update of b (D4, via the inverse permutation: schedule_prev) and the
// sequence's guard need = max(k - delay, kprev + 1).  Sequences are visited in order.
struct SlabSchedule {
    PermKeys pk, pkp;
    int half;
    int64_t e, i;  // local epoch, position in it
    int kmod;      // k mod grid
    __device__ void init(int64_t N) {
        half = perm_half_bits(N);
        e = 0; i = 0; kmod = 0;
    }
    __device__ SeqMeta next(const SlabParams& P, int64_t k) {
        const int64_t N = P.nblk;
        if (i == 0 && P.sched == SCHED_RANDOM) {
            pk = perm_keys(P.seed, P.epoch0 + e);
            if (P.epoch0 + e > 0) pkp = perm_keys(P.seed, P.epoch0 + e - 1);
        }
        int64_t b = i, kprev = -1;
        if (P.sched == SCHED_RANDOM) {
            uint64_t v = (uint64_t)i;
            do { v = feistel(v, half, pk); } while (v >= (uint64_t)N);
            b = (int64_t)v;
        }
        if (P.epoch0 + e > 0) {
            int64_t pos = b;
            if (P.sched == SCHED_RANDOM) {
                uint64_t v = (uint64_t)b;
                do { v = feistel_inv(v, half, pkp); } while (v >= (uint64_t)N);
                pos = (int64_t)v;
            }
            kprev = (e - 1) * N + pos;  // local index (negative: an earlier launch)
        }
        SeqMeta md;
        md.need = k - P.delay;
        if (kprev + 1 > md.need) md.need = kprev + 1;
        md.b = (int32_t)b;
        md.flags = (int32_t)(e & 1) | (kmod == (int)blockIdx.x ? 2 : 0);
        if (++i == N) { i = 0; ++e; }
        if (++kmod == (int)gridDim.x) kmod = 0;
        return md;
    }
};

// Sequence warp q (of kSlabSeq): for its sequences k = q, q + 6, ... sums the CTA's
// kSlabDot partials (fixed order), publishes them into the grid-wide accumulator,
// waits for all CTAs, solves the block subproblem (Eq. 2 closed form) + (S.4) and
// hands dx_b to the axpy warps; CTA k mod grid stores x_b.  Shared by both slab kernels.
template <int BMAX, int NSPLIT = 1>
__device__ __forceinline__ void slab_sequence_warp(const SlabParams& P, int q, int lane, const double* pring,
                                                   double* dxring, const SeqMeta* meta, uint64_t* pfull,
                                                   uint64_t* pempty, uint64_t* dxfull, uint64_t* dxempty,
                                                   SlabProf& sp, uint64_t* arrived = nullptr,
                                                   const long long* meta_k = nullptr) {
    const int64_t K = P.K;
    const int B = (int)P.B;
    const int64_t S = P.slots;
    int lgS = 0;
    while (((int64_t)1 << lgS) < S) ++lgS;
    const unsigned grid = gridDim.x;
    constexpr int CS = BMAX / NSPLIT;  // columns of a sub-sequence
    constexpr int PER = CS / 32;        // block columns per lane
    // this warp's sub-sequences s = q + 6 t (s = k * NSPLIT + h: columns [h CS, h CS + CS) of
    // sequence k's block) use ring slot q, phase t & 1
    uint32_t ph = 0;
    for (int64_t s = q; s < K * NSPLIT; s += kSlabSeq, ph ^= 1u) {
        const int64_t k = s / NSPLIT;
        const int h = (int)(s - k * NSPLIT);
        double tpre[PER];
        bool have_tau = false;
        if (meta_k) {
            // metadata ready (flag): prefetch tau_b while the CTA's partial is computed
            if (lane == 0) {
                long long v;
                for (;;) {
                    asm volatile("ld.acquire.cta.shared.b64 %0, [%1];"
                                 : "=l"(v)
                                 : "r"(smem_u32(&meta_k[k & (kSlabNM - 1)]))
                                 : "memory");
                    if (v == k) break;
                    __nanosleep(32);
                }
            }
            __syncwarp();
            const int64_t cb = (int64_t)meta[k & (kSlabNM - 1)].b * P.B + h * CS;
            const int ncb = (int)max((int64_t)0, min(min((int64_t)CS, P.B - h * CS), P.n - cb));
#pragma unroll
            for (int e = 0; e < PER; ++e) {
                const int cc = lane + 32 * e;
                tpre[e] = cc < ncb ? __ldg(&P.tau[cb + cc]) : 1.0;
            }
            have_tau = true;
        }
        // the CTA's partial (the dot warps' arrivals also publish the sequence's metadata)
        mbar_wait(&pfull[q], ph);
        sp.mark(1);
        const SeqMeta md = meta[k & (kSlabNM - 1)];
        const int64_t c0 = (int64_t)md.b * P.B + h * CS;
        const int nc = (int)max((int64_t)0, min(min((int64_t)CS, P.B - h * CS), P.n - c0));
        const int64_t slot = s & (S - 1), use = s >> lgS;
        const int half = (int)(use & 1);
        const double* xr = (md.flags & 1) ? P.x1 : P.x0;
        double* xw = (md.flags & 1) ? P.x0 : P.x1;
        double pv[PER];
#pragma unroll
        for (int e = 0; e < PER; ++e) {
            const int cc = lane + 32 * e;
            const double* pw = pring + (size_t)q * kSlabDot * CS + cc;
            pv[e] = ((pw[0] + pw[CS]) + pw[2 * CS]) + pw[3 * CS];  // fixed order
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&pempty[q]);
        // publish
        const int rep = (int)(blockIdx.x % kGaccRep);
        double* gk = P.gacc + (slot * 2 + half) * kGaccRep * P.B;  // replica 0 of the slot half
        double* gmine = gk + rep * P.B;
#pragma unroll
        for (int e = 0; e < PER; ++e) {
            const int cc = lane + 32 * e;
            if (cc < nc) {
                if (P.deterministic) P.part[(slot * grid + blockIdx.x) * P.B + cc] = pv[e];
                else atomicAdd(&gmine[cc], pv[e]);
            }
        }
        __syncwarp();
        if (lane == 0) red_release_gpu_u32(&P.arrive[slot * kArrivePad], 1u);
        if (!have_tau) {  // (after the release: it would wait for this load as well)
#pragma unroll
            for (int e = 0; e < PER; ++e) {
                const int cc = lane + 32 * e;
                tpre[e] = cc < nc ? __ldg(&P.tau[c0 + cc]) : 1.0;
            }
        }
        sp.mark(2);
        // all CTAs' partials of sub-sequence s
        if (arrived) {
            // the CTA's watcher lane polls the arrival counters (one poller per CTA) and
            // signals this warp's ring slot
            mbar_wait(&arrived[q], ph);
        } else {
            if (lane == 0) spin_until_ge_relaxed_u32(&P.arrive[slot * kArrivePad], (unsigned)(use + 1) * grid);
            __syncwarp();
        }
        sp.mark(3);
        double g[PER], y[PER];
#pragma unroll
        for (int e = 0; e < PER; ++e) {
            const int cc = lane + 32 * e;
            g[e] = 0.0;
            y[e] = 0.0;
            if (cc < nc) {
                if (P.deterministic) {
                    for (unsigned tt = 0; tt < grid; ++tt)
                        g[e] += ld_relaxed_f64(&P.part[(slot * grid + tt) * P.B + cc]);
                } else {
                    double gr[kGaccRep];
#pragma unroll
                    for (int r = 0; r < kGaccRep; ++r) gr[r] = ld_relaxed_f64(&gk[r * P.B + cc]);
#pragma unroll
                    for (int r = 0; r < kGaccRep; ++r) g[e] += gr[r];
                }
                y[e] = ld_relaxed_f64(&xr[c0 + cc]);
            }
        }
        if (!P.deterministic) {
            double* gn = P.gacc + ((slot * 2 + (half ^ 1)) * kGaccRep + rep) * P.B;  // my replica
#pragma unroll
            for (int e = 0; e < PER; ++e) {
                const int cc = lane + 32 * e;
                if (cc < B && cc < CS) gn[cc] = 0.0;
            }
        }
        // block subproblem (Eq. 2, closed form) and (S.4)
        double xn[PER], dd[PER];
#pragma unroll
        for (int e = 0; e < PER; ++e) {
            const int cc = lane + 32 * e;
            xn[e] = y[e];
            dd[e] = 0.0;
            if (cc < nc) {
                const double xh = best_response(P.S, g[e], y[e], tpre[e], c0 + cc);
                xn[e] = y[e] + P.gamma * (xh - y[e]);
                dd[e] = xn[e] - y[e];
            }
        }
        if (s >= kSlabNDX) mbar_wait(&dxempty[q], ph ^ 1u);
#pragma unroll
        for (int e = 0; e < PER; ++e) dxring[q * CS + lane + 32 * e] = dd[e];
        if (md.flags & 2) {
#pragma unroll
            for (int e = 0; e < PER; ++e) {
                const int cc = lane + 32 * e;
                if (cc < nc) xw[c0 + cc] = xn[e];
            }
            fence_acq_rel_gpu();  // x_b visible before this CTA's later arrivals (D4 readers)
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&dxfull[q]);
        sp.mark(4);
    }
}

// CPW = 8, 16 or 32: blocks of up to BMAX = 4 * CPW columns.  LOSS: LOSS_LS / LOSS_LOGISTIC
// (compile-time: keeps the instruction footprint of the hot loops small).
template <int CPW, int LOSS>
__global__ void __launch_bounds__(kSlabThreads, 1)
    dense_slab_kernel(const __grid_constant__ CUtensorMap tmap, const SlabParams P) {
    constexpr int BMAX = kSlabDot * CPW;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    const int nst = P.nst, nsa = P.nsa, Rc = P.Rc, nch = P.nch;
    const int nsw = nst / kSlabDot;                                  // stages per dot warp
    const int64_t SD = P.stage_dbl;
    const int64_t RsP = (P.Rs + 1) & ~(int64_t)1;                   // 16-byte aligned rings below
    double* dstage = reinterpret_cast<double*>(smem_raw);           // nst * SD
    double* astage = dstage + (size_t)nst * SD;                      // nsa * SD
    double* rs = astage + (size_t)nsa * SD;                          // Rs   residual slab
    double* auxs = rs + RsP;                                         // Rs   b / y slab
    double* pring = auxs + RsP;                                      // NP * kSlabDot * BMAX
    double* dxring = pring + kSlabNP * kSlabDot * BMAX;              // NDX * BMAX
    double* wscr = dxring + kSlabNDX * BMAX;                         // kSlabDot * 256 (dot warps' w)
    SeqMeta* meta = reinterpret_cast<SeqMeta*>(wscr + kSlabDot * 256);  // NM
    uint64_t* bars = reinterpret_cast<uint64_t*>(meta + kSlabNM);
    uint64_t* dfull = bars;                      // nst
    uint64_t* dempty = dfull + kSlabMaxStages;   // nst
    uint64_t* afull = dempty + kSlabMaxStages;   // nsa
    uint64_t* aempty = afull + kSlabMaxStages;   // nsa
    uint64_t* pfull = aempty + kSlabMaxStages;   // NP
    uint64_t* pempty = pfull + kSlabNP;          // NP
    uint64_t* dxfull = pempty + kSlabNP;         // NDX
    uint64_t* dxempty = dxfull + kSlabNDX;       // NDX
    unsigned long long* progress = reinterpret_cast<unsigned long long*>(dxempty + kSlabNDX);  // kSlabAx
    unsigned long long* dotdone = progress + kSlabAx;                                          // kSlabDot

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t row0 = (int64_t)blockIdx.x * P.Rs;
    const int rows = (int)max((int64_t)0, min(P.Rs, P.m - row0));  // this CTA's slab rows
    const int B = (int)P.B;
    const int64_t K = P.K, N = P.nblk;
    const int nrg = (Rc + 31) >> 5;  // 32-row groups per chunk

    // ---- init: zero the stages (columns >= B and the tail pads stay zero), load the slab
    for (int64_t i = threadIdx.x; i < (int64_t)(nst + nsa) * SD; i += blockDim.x) dstage[i] = 0.0;
    for (int i = threadIdx.x; i < kSlabNP * kSlabDot * BMAX + kSlabNDX * BMAX; i += blockDim.x) pring[i] = 0.0;
    for (int i = threadIdx.x; i < P.Rs; i += blockDim.x) {
        rs[i] = i < rows ? P.r[row0 + i] : 0.0;
        auxs[i] = i < rows ? P.aux[row0 + i] : 0.0;
    }
    if (threadIdx.x == 0) {
        for (int s = 0; s < nst; ++s) {
            mbar_init(&dfull[s], 1);
            mbar_init(&dempty[s], P.hold ? kSlabAx : 1);
        }
        for (int s = 0; s < nsa; ++s) {
            mbar_init(&afull[s], 1);
            mbar_init(&aempty[s], kSlabAx);
        }
        for (int s = 0; s < kSlabNP; ++s) {
            mbar_init(&pfull[s], kSlabDot);
            mbar_init(&pempty[s], 1);
        }
        for (int s = 0; s < kSlabNDX; ++s) {
            mbar_init(&dxfull[s], 1);
            mbar_init(&dxempty[s], kSlabAx);
        }
        for (int a = 0; a < kSlabAx; ++a) progress[a] = 0ull;
        for (int d = 0; d < kSlabDot; ++d) dotdone[d] = 0ull;
        mbar_fence_init();
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmap) : "memory");
    }
    // generic-proxy zero fill of the stages before the async proxy writes them
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();

    SlabProf sp;
    sp.start();
    const uint32_t box_bytes = (uint32_t)Rc * (uint32_t)B * 8u;
    if (warp == 0) {
        // ---------------------------------------------------------------- dot producer (+ schedule)
        if (lane == 0) {
            const uint64_t pol = P.hold ? policy_evict_first() : policy_evict_last();
            SlabSchedule sch;
            sch.init(N);
            // chunk c goes to sub-ring c mod 4 at position (c / 4) mod nsw: the four sub-rings
            // advance together, one position per group of four chunks
            RingPos gp;
            gp.init(nsw);
            int64_t c = 0;
            for (int64_t k = 0; k < K; ++k) {
                const SeqMeta mk = sch.next(P, k);
                const int64_t b = mk.b;
                // the metadata slot of sequence k - NM is free once its axpy is done
                if (k >= kSlabNM) {
                    for (int a = 0; a < kSlabAx; ++a)
                        while (ld_acquire_cta_u64(&progress[a]) < (unsigned long long)(k - kSlabNM + 1)) __nanosleep(32);
                }
                meta[k & (kSlabNM - 1)] = mk;
                for (int ch = 0; ch < nch; ++ch, ++c) {
                    const int w = (int)(c & (kSlabDot - 1));
                    const int st = w * nsw + gp.i;
                    if ((c >> 2) >= nsw) mbar_wait(&dempty[st], gp.ph ^ 1u);
                    // (the mbarrier arrive releases the metadata written above to the dot warps)
                    mbar_arrive_expect_tx(&dfull[st], box_bytes);
                    slab_tma_2d(dstage + st * SD, &tmap, (int)(row0 + (int64_t)ch * Rc), (int)(b * P.B), &dfull[st],
                                pol);
                    if (w == kSlabDot - 1) gp.next();
                }
            }
        }
        sp.mark(0);
    } else if (warp == 1) {
        // ---------------------------------------------------------------- axpy producer (re-load pass)
        if (lane == 0 && !P.hold) {
            const uint64_t pol = policy_evict_first();
            RingPos rp;
            rp.init(nsa);
            for (int64_t j = 0; j < K; ++j) {
                // every dot warp is past sequence j: the tile is in L2 (and its metadata valid)
                for (int d = 0; d < kSlabDot; ++d)
                    while (ld_acquire_cta_u64(&dotdone[d]) <= (unsigned long long)j) __nanosleep(64);
                const int64_t b = meta[j & (kSlabNM - 1)].b;
                for (int ch = 0; ch < nch; ++ch, rp.next()) {
                    if (j * nch + ch >= nsa) mbar_wait(&aempty[rp.i], rp.ph ^ 1u);
                    mbar_arrive_expect_tx(&afull[rp.i], box_bytes);
                    slab_tma_2d(astage + rp.i * SD, &tmap, (int)(row0 + (int64_t)ch * Rc), (int)(b * P.B),
                                &afull[rp.i], pol);
                }
            }
        }
        sp.mark(0);
    } else if (warp < kSlabAx0) {
        // ---------------------------------------------------------------- dot warps
        const int d = warp - kSlabDot0;
        constexpr int GW = 16;  // columns per register pass
        constexpr int NG = BMAX / GW;
        uint64_t* myfull = dfull + d * nsw;
        uint64_t* myempty = dempty + d * nsw;
        const double* mystage = dstage + (size_t)d * nsw * SD;
        double* myw = wscr + d * 256;
        RingPos rp, pp;
        rp.init(nsw);
        pp.init(kSlabNP);
        int c4 = 0;  // (k * nch) mod 4
        for (int64_t k = 0; k < K; ++k) {
            int ch = d - c4;  // first chunk of sequence k that is this warp's
            if (ch < 0) ch += kSlabDot;
            double tot[NG];
#pragma unroll
            for (int gi = 0; gi < NG; ++gi) tot[gi] = 0.0;
            if (ch < nch) {
                // first chunk landed => the sequence's metadata is there (written before the arrive)
                mbar_wait(&myfull[rp.i], rp.ph);
                sp.mark(2);
                // D1 / D4 guards: axpy(k - delay - 1) and axpy(kprev) applied to this slab
                const int64_t need = meta[k & (kSlabNM - 1)].need;
                if (need > 0) {
#pragma unroll
                    for (int a = 0; a < kSlabAx; ++a)
                        while (ld_acquire_cta_u64(&progress[a]) < (unsigned long long)need) __nanosleep(20);
                }
                sp.mark(1);
                for (; ch < nch; ch += kSlabDot, rp.next()) {
                    mbar_wait(&myfull[rp.i], rp.ph);
                    const double* T = mystage + rp.i * SD + lane;
                    // w = phi'(r) of this lane's chunk rows, staged in the warp's scratch
                    for (int g = 0; g < nrg; ++g) {
                        const int i = g * 32 + lane, srow = ch * Rc + i;
                        myw[i] = (i < Rc && srow < rows) ? loss_prime_t<LOSS>(P.S, rs[srow], auxs[srow]) : 0.0;
                    }
                    __syncwarp();
#pragma unroll
                    for (int gi = 0; gi < NG; ++gi) {
                        double acc[GW];
#pragma unroll
                        for (int cc = 0; cc < GW; ++cc) acc[cc] = 0.0;
                        const double* a = T + (size_t)(gi * GW) * Rc;
                        for (int g = 0; g < nrg; ++g) {
                            const double w = myw[g * 32 + lane];
#pragma unroll
                            for (int cc = 0; cc < GW; ++cc) acc[cc] = fma(a[(size_t)cc * Rc + g * 32], w, acc[cc]);
                        }
                        tot[gi] += slab_reduce16(acc, lane);
                    }
                    __syncwarp();
                    if (!P.hold && lane == 0) mbar_arrive(&myempty[rp.i]);
                }
                sp.mark(3);
            }
            // this warp's partial of sequence k -> its slot (summed in warp order by the
            // sequence warp: deterministic)
            if (k >= kSlabNP) mbar_wait(&pempty[pp.i], pp.ph ^ 1u);
            if (lane < GW) {
#pragma unroll
                for (int gi = 0; gi < NG; ++gi) pring[(pp.i * kSlabDot + d) * BMAX + gi * GW + lane] = tot[gi];
            }
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(&pfull[pp.i]);
                st_release_cta_u64(&dotdone[d], (unsigned long long)(k + 1));
            }
            pp.next();
            c4 = (c4 + nch) & (kSlabDot - 1);
            sp.mark(4);
        }
    } else if (warp < kSlabSeq0) {
        // ---------------------------------------------------------------- axpy warps
        // axpy warp a owns the slab rows of the (chunk, 32-row group) items i = a mod 4 for
        // the whole launch: sequences are applied in order per warp, without a CTA barrier
        const int a = warp - kSlabAx0;
        RingPos gp, ra, xp;
        gp.init(nsw);
        ra.init(nsa > 0 ? nsa : 1);
        xp.init(kSlabNDX);
        int64_t c = 0;  // global chunk index (hold mode: stage of chunk c as in the producer)
        for (int64_t j = 0; j < K; ++j) {
            mbar_wait(&dxfull[xp.i], xp.ph);
            sp.mark(1);
            const double* dxv = dxring + xp.i * BMAX;
            for (int ch = 0; ch < nch; ++ch, ++c) {
                const double* T;
                uint64_t* freeb;
                if (P.hold) {
                    const int st = (int)(c & (kSlabDot - 1)) * nsw + gp.i;
                    T = dstage + st * SD;
                    freeb = &dempty[st];
                    if ((c & (kSlabDot - 1)) == kSlabDot - 1) gp.next();
                } else {
                    mbar_wait(&afull[ra.i], ra.ph);
                    T = astage + ra.i * SD;
                    freeb = &aempty[ra.i];
                    ra.next();
                }
                sp.mark(2);
                int g = a - (ch * nrg) % kSlabAx;
                if (g < 0) g += kSlabAx;
                for (; g < nrg; g += kSlabAx) {
                    const int i = g * 32 + lane;
                    const int srow = ch * Rc + i;
                    if (i < Rc && srow < rows) {
                        double s4[4] = {0.0, 0.0, 0.0, 0.0};
                        const double* t = T + i;
#pragma unroll
                        for (int cc = 0; cc < BMAX; cc += 2) {
                            const double2 d2 = *reinterpret_cast<const double2*>(dxv + cc);
                            s4[cc & 3] = fma(t[(size_t)cc * Rc], d2.x, s4[cc & 3]);
                            s4[(cc + 1) & 3] = fma(t[(size_t)(cc + 1) * Rc], d2.y, s4[(cc + 1) & 3]);
                        }
                        rs[srow] += (s4[0] + s4[1]) + (s4[2] + s4[3]);
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(freeb);
                sp.mark(3);
            }
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(&dxempty[xp.i]);
                st_release_cta_u64(&progress[a], (unsigned long long)(j + 1));
            }
            xp.next();
            sp.mark(4);
        }
    } else {
        slab_sequence_warp<BMAX>(P, warp - kSlabSeq0, lane, pring, dxring, meta, pfull, pempty, dxfull, dxempty, sp);
    }
    sp.flush(P.prof ? P.prof + ((size_t)blockIdx.x * kSlabWarps + warp) * 8 : nullptr, lane);
    __syncthreads();
    for (int i = threadIdx.x; i < rows; i += blockDim.x) P.r[row0 + i] = rs[i];
}

}  // namespace asy
