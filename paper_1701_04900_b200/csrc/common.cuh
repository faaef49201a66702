// common.cuh -- scalar pieces of the AsyFLEXA block update shared by every
// kernel: the schedule (Philox4x32-10 + keyed permutation), the loss
// derivative phi' that turns the shared residual into a gradient, the closed
// form of the Eq. (2) subproblem, and sm_100a PTX wrappers (mbarrier, bulk
// copy, acquire/release).  PAPER.md line numbers in brackets.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#define ASY_HD __host__ __device__ __forceinline__

namespace asy {

enum { LOSS_LS = 0, LOSS_LOGISTIC = 1 };
enum { REG_L1 = 0, REG_EXP = 1, REG_LOG = 2 };
enum { SCHED_CYCLIC = 0, SCHED_RANDOM = 1 };

// ---------------------------------------------------------------------------
// Philox4x32-10 (Random123 constants)
// ---------------------------------------------------------------------------
ASY_HD void philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
    uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
    uint32_t k0 = key[0], k1 = key[1];
#pragma unroll
    for (int i = 0; i < 10; ++i) {
        if (i > 0) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
        const uint64_t p0 = (uint64_t)0xD2511F53u * c0;
        const uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
        const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        c0 = hi1 ^ c1 ^ k0; c1 = lo1; c2 = hi0 ^ c3 ^ k1; c3 = lo0;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

ASY_HD uint32_t fmix32(uint32_t h) {
    h ^= h >> 16; h *= 0x85EBCA6Bu; h ^= h >> 13; h *= 0xC2B2AE35u; h ^= h >> 16;
    return h;
}

// Random schedule: epoch e visits the N blocks in the order of a random
// permutation pi_e, realised as a 4-round Feistel network on [0, 2^d)
// (d even, 2^d >= N) whose round keys are one Philox4x32-10 draw keyed by
// the seed, with cycle-walking back into [0, N).  O(1) state, any k.
struct PermKeys { uint32_t k[4]; };

ASY_HD PermKeys perm_keys(uint64_t seed, int64_t epoch) {
    const uint32_t ctr[4] = {(uint32_t)epoch, (uint32_t)((uint64_t)epoch >> 32), 0x5EEDu, 0xA5F1u};
    const uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    PermKeys pk;
    philox4x32_10(ctr, key, pk.k);
    return pk;
}

ASY_HD int perm_half_bits(int64_t nblocks) {
    int d = 2;
    while (((int64_t)1 << d) < nblocks) ++d;
    if (d & 1) ++d;
    return d / 2;
}

ASY_HD uint64_t feistel(uint64_t v, int half, const PermKeys& pk) {
    const uint64_t mask = ((uint64_t)1 << half) - 1;
    uint64_t L = v >> half, R = v & mask;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        const uint64_t F = (uint64_t)fmix32((uint32_t)R ^ pk.k[r] ^ (uint32_t)(R >> 32)) & mask;
        const uint64_t nL = R;
        R = L ^ F;
        L = nL;
    }
    return (L << half) | R;
}

ASY_HD int64_t schedule_block(int sched, uint64_t seed, int64_t nblocks, int64_t k) {
    const int64_t e = k / nblocks, i = k - e * nblocks;
    if (sched == SCHED_CYCLIC) return i;
    const PermKeys pk = perm_keys(seed, e);
    const int half = perm_half_bits(nblocks);
    uint64_t v = (uint64_t)i;
    do { v = feistel(v, half, pk); } while (v >= (uint64_t)nblocks);
    return (int64_t)v;
}

// inverse of one Feistel pass: round r maps (L, R) -> (R, L ^ F_r(R))
ASY_HD uint64_t feistel_inv(uint64_t v, int half, const PermKeys& pk) {
    const uint64_t mask = ((uint64_t)1 << half) - 1;
    uint64_t L = v >> half, R = v & mask;
#pragma unroll
    for (int r = 3; r >= 0; --r) {
        const uint64_t F = (uint64_t)fmix32((uint32_t)L ^ pk.k[r] ^ (uint32_t)(L >> 32)) & mask;
        const uint64_t oL = R ^ F;
        R = L;
        L = oL;
    }
    return (L << half) | R;
}

// position of block b in epoch e's order (inverse of schedule_block within the
// epoch; cycle-walking inverts the same way it permutes)
ASY_HD int64_t schedule_position(int sched, uint64_t seed, int64_t nblocks, int64_t e, int64_t b) {
    if (sched == SCHED_CYCLIC) return b;
    const PermKeys pk = perm_keys(seed, e);
    const int half = perm_half_bits(nblocks);
    uint64_t v = (uint64_t)b;
    do { v = feistel_inv(v, half, pk); } while (v >= (uint64_t)nblocks);
    return (int64_t)v;
}

// global index of the previous update of the block that sequence k updates
// (-1: none).  Every epoch visits each block once, so it lies in epoch e-1.
ASY_HD int64_t schedule_prev(int sched, uint64_t seed, int64_t nblocks, int64_t k, int64_t b) {
    const int64_t e = k / nblocks;
    if (e == 0) return -1;
    return (e - 1) * nblocks + schedule_position(sched, seed, nblocks, e - 1, b);
}

// ---------------------------------------------------------------------------
// the problem's scalar maps
// ---------------------------------------------------------------------------
struct Scalars {
    int loss, reg;
    double s2;        // 2*s (LS)
    double minv;      // 1/m (logistic)
    double c2;        // 2*c (nonconvex term)
    double lam;       // lambda
    double lam_eff;   // lambda*eta(theta)   (= lambda for l1)
    double theta, eta, inv_log1p_theta;
    double lo_all, hi_all;
    const double* lo; // may be null
    const double* hi; // may be null
};

// w_j = phi_j'(r_j): grad f = A^T w (- 2c x).  LS: r = Ax-b, w = 2s r.
// Logistic: r = z = Ax, w = -(y/m) sigmoid(-y z).  (LOSS fixed at compile time.)
template <int LOSS>
ASY_HD double loss_prime_t(const Scalars& S, double r, double aux) {
    if (LOSS == LOSS_LS) return S.s2 * r;
    const double t = -aux * r;  // sigmoid(t) = 1 / (1 + e^-t) (t >= 0), e^t / (1 + e^t) (t < 0): one exp
    const double e = exp(-fabs(t));
    const double sig = (t >= 0.0 ? 1.0 : e) / (1.0 + e);
    return -aux * S.minv * sig;
}
ASY_HD double loss_prime(const Scalars& S, double r, double aux) {
    return S.loss == LOSS_LS ? loss_prime_t<LOSS_LS>(S, r, aux) : loss_prime_t<LOSS_LOGISTIC>(S, r, aux);
}

// phi_j(r_j): LS: s r^2 (= s2/2 r^2); logistic: (1/m) log(1+exp(-y z)).
ASY_HD double loss_value(const Scalars& S, double r, double aux) {
    if (S.loss == LOSS_LS) return 0.5 * S.s2 * r * r;
    const double t = -aux * r;
    const double sp = (t > 0.0 ? t : 0.0) + log1p(exp(-fabs(t)));
    return S.minv * sp;
}

// d/dt h^-(t), h^- = eta|t| - h(t)  (Eq. 12 [PAPER.md:530]).
// (the DC branch is out of line on the device: it keeps exp/log1p out of the hot
// loops' instruction footprint; l1 never calls it)
#if defined(__CUDA_ARCH__)
__device__ __noinline__
#else
inline
#endif
double grad_h_minus_dc(int reg, double eta, double theta, double t) {
    const double sg = t > 0.0 ? 1.0 : (t < 0.0 ? -1.0 : 0.0);
    const double a = fabs(t);
    if (reg == REG_EXP) return eta * sg * (1.0 - exp(-theta * a));
    return sg * (eta - theta / ((1.0 + theta * a) * log1p(theta)));
}
ASY_HD double grad_h_minus(const Scalars& S, double t) {
    if (S.reg == REG_L1) return 0.0;
    return grad_h_minus_dc(S.reg, S.eta, S.theta, t);
}

// h(t) of G = lambda sum h(x_j).
ASY_HD double reg_value(const Scalars& S, double t) {
    const double a = fabs(t);
    if (S.reg == REG_L1) return a;
    if (S.reg == REG_EXP) return 1.0 - exp(-S.theta * a);
    return log1p(S.theta * a) * S.inv_log1p_theta;
}

ASY_HD double box_lo(const Scalars& S, int64_t j) { return S.lo ? S.lo[j] : S.lo_all; }
ASY_HD double box_hi(const Scalars& S, int64_t j) { return S.hi ? S.hi[j] : S.hi_all; }

// argmin_{t in [lo,hi]} g (t-y) + tau/2 (t-y)^2 + lam_eff |t|: soft-threshold
// [PAPER.md:384] of the unconstrained minimiser, then projection on [lo,hi].
ASY_HD double coord_argmin(double g, double y, double tau, double lam_eff, double lo, double hi) {
    const double v = y - g / tau;
    const double t = lam_eff / tau;
    const double u = v > t ? v - t : (v < -t ? v + t : 0.0);
    return fmin(fmax(u, lo), hi);
}

// Best response of coordinate j of the block (Eq. 2, or Eq. 13 for the DC
// penalties): gs = smooth partial gradient at tilde x (A^T w part only).
ASY_HD double best_response(const Scalars& S, double gs, double y, double tau, int64_t j) {
    double g = gs - S.c2 * y;
    if (S.reg != REG_L1) g -= S.lam * grad_h_minus(S, y);
    return coord_argmin(g, y, tau, S.lam_eff, box_lo(S, j), box_hi(S, j));
}

#if defined(__CUDACC__)
// ---------------------------------------------------------------------------
// device-only PTX wrappers (sm_90+ / sm_100a)
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_fence_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
// 1-D bulk copy global -> shared (TMA engine, SASS UBLKCP), completion on mbarrier.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
        "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ long long ld_acquire_s64(const long long* p) {
    long long v;
    asm volatile("ld.acquire.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_s64(long long* p, long long v) {
    asm volatile("st.release.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_release_u32(unsigned* p, unsigned v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// coherent (L2) read of data other SMs update concurrently
__device__ __forceinline__ double ld_relaxed_f64(const double* p) {
    double v;
    asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void spin_until_ge(const long long* p, long long v) {
    if (ld_acquire_s64(p) >= v) return;
    unsigned ns = 32;
    while (ld_acquire_s64(p) < v) {
        __nanosleep(ns);
        if (ns < 256) ns <<= 1;
    }
}
__device__ __forceinline__ void spin_until_ge_u32(const unsigned* p, unsigned v) {
    if (ld_acquire_u32(p) >= v) return;
    unsigned ns = 32;
    while (ld_acquire_u32(p) < v) {
        __nanosleep(ns);
        if (ns < 256) ns <<= 1;
    }
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
#endif

}  // namespace asy
