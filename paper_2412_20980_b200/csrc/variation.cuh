// Child-gene arithmetic shared by the slot-pool variation kernels (slot_kernels.cu) and the fused
// variation + mask-build kernel of the PC fitness (pc_kernels.cu).  Bit-exact twins of
// ga_ops.cpp:130-178 and :214-238 on the keyed streams of rng.hpp.
#pragma once

#include "internal.cuh"

namespace gapa_b200 {

static constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;
static constexpr uint64_t kCounterStep = 0x632BE59BD9B4E019ull;  // rng.hpp:21

// Hand-expanded integer arithmetic of the hash, measured at C4 (tools/ab_vary_arith.sh, one generation):
//   bit 0 — 64 x 64 -> low 64 as three multiply-adds (one wide, two accumulating into the high word) instead of the
//           compiler's four instructions: 1.78 -> 1.89 ms.  The three-instruction form is one dependent chain, the
//           compiler's has two independent halves: the kernel is bound by dependent-issue latency, not by issue slots.
//   bit 1 — next_index as two wide multiply-adds instead of the generic __umul64hi: 1.781 -> 1.775 ms.  Kept.
//   bits 3-5 — see ShiftMul / stream_at below (round 2, kernel time of the persistent fused kernel at C4):
//           2: 0.822 ms;  2+8: 0.907;  2+16: 1.050;  2+32: 0.812 (kept);  2+16+32: 1.027;  2+8+16+32: 1.026
#ifndef GAPA_VARY_ARITH
#define GAPA_VARY_ARITH 34
#endif
__device__ __forceinline__ uint64_t mul64_const(uint64_t x, uint64_t c) {
#if !(GAPA_VARY_ARITH & 1)
    return x * c;
#endif
    const uint32_t xl = static_cast<uint32_t>(x), xh = static_cast<uint32_t>(x >> 32);
    const uint32_t cl = static_cast<uint32_t>(c), ch = static_cast<uint32_t>(c >> 32);
    const uint64_t w = static_cast<uint64_t>(xl) * cl;
    const uint32_t hi = static_cast<uint32_t>(w >> 32) + xl * ch + xh * cl;
    return (static_cast<uint64_t>(hi) << 32) | static_cast<uint32_t>(w);
}
// Multipliers 2^(32-s) of the hash's three right shifts, passed at RUN time (kernel parameters) so that the compiler
// keeps them as multiplies: x >> s == umulhi(x, 2^(32-s)).  The integer ALU pipe of sm_100 (shifts, logic, adds, compares)
// issues one warp instruction every two cycles per scheduler and is what bounds the fused variation kernel (ncu: ALU
// pipe 62 % busy, top stalls math_pipe_throttle / not_selected; 186 of the 330 instructions of a four-gene pass are ALU
// ones, 106 are multiply-adds on the FMA pipe).  Moving the shifts to the FMA pipe was meant to rebalance the two — measured,
// it does the opposite: IMAD.HI / IMAD.WIDE cost more FMA-pipe time than the shifts cost ALU-pipe time (numbers above):
//   bit 3 (8)  — hi >> s as umulhi (IMAD.HI.U32)
//   bit 4 (16) — the whole 64-bit shift as one wide multiply + one umulhi: x ^ (x >> s) is 2 FMA + 2 ALU instead of 4 ALU
//   bit 5 (32) — key + step * (column + 1) as a wide multiply-add instead of a running 64-bit sum (adds leave the ALU pipe)
struct ShiftMul {
    uint32_t m30, m27, m31;
};
__device__ __forceinline__ uint64_t xorshift_r(uint64_t y, int s, uint32_t m) {
#if GAPA_VARY_ARITH & 16
    const uint32_t lo = static_cast<uint32_t>(y), hi = static_cast<uint32_t>(y >> 32);
    const uint64_t w = static_cast<uint64_t>(hi) * m;  // low word: hi << (32 - s), high word: hi >> s
    const uint32_t t = __umulhi(lo, m);                // lo >> s
    const uint32_t lo2 = lo ^ (t | static_cast<uint32_t>(w));
    const uint32_t hi2 = hi ^ static_cast<uint32_t>(w >> 32);
    return (static_cast<uint64_t>(hi2) << 32) | lo2;
#elif GAPA_VARY_ARITH & 8
    const uint32_t lo = static_cast<uint32_t>(y), hi = static_cast<uint32_t>(y >> 32);
    const uint32_t lo2 = lo ^ __funnelshift_r(lo, hi, s);
    const uint32_t hi2 = hi ^ __umulhi(hi, m);
    return (static_cast<uint64_t>(hi2) << 32) | lo2;
#else
    (void)m;
    return y ^ (y >> s);
#endif
}
// mix64(x) with y = x + kGolden (rng.hpp:8-13)
__device__ __forceinline__ uint64_t hash_tail(uint64_t y, const ShiftMul& M) {
    y = mul64_const(xorshift_r(y, 30, M.m30), 0xBF58476D1CE4E5B9ull);
    y = mul64_const(xorshift_r(y, 27, M.m27), 0x94D049BB133111EBull);
    return xorshift_r(y, 31, M.m31);
}
// key + kCounterStep * col1 (draw col1 - 1 of the stream, rng.hpp:21)
__device__ __forceinline__ uint64_t stream_at(uint64_t key, uint32_t col1) {
#if GAPA_VARY_ARITH & 32
    const uint32_t sl = static_cast<uint32_t>(kCounterStep), sh = static_cast<uint32_t>(kCounterStep >> 32);
    const uint64_t w = static_cast<uint64_t>(col1) * sl + key;  // IMAD.WIDE with a 64-bit addend
    const uint32_t hi = static_cast<uint32_t>(w >> 32) + col1 * sh;
    return (static_cast<uint64_t>(hi) << 32) | static_cast<uint32_t>(w);
#else
    return key + kCounterStep * static_cast<uint64_t>(col1);
#endif
}
// next_index (rng.hpp:28-31): high 64 bits of u64 x u32 in two wide multiply-adds
__device__ __forceinline__ uint32_t mulhi_u64_u32(uint64_t u, uint32_t bound) {
#if !(GAPA_VARY_ARITH & 2)
    return static_cast<uint32_t>(__umul64hi(u, static_cast<uint64_t>(bound)));
#endif
    const uint64_t t = static_cast<uint64_t>(static_cast<uint32_t>(u)) * bound;
    const uint64_t r = static_cast<uint64_t>(static_cast<uint32_t>(u >> 32)) * bound + (t >> 32);
    return static_cast<uint32_t>(r >> 32);
}

struct VariationParams {
    uint64_t pc_limit, pm_limit;  // next_bernoulli(p) == always || u < limit  (u >> 11 < ceil(p 2^53))
    bool pc_always, pm_always;
    uint32_t pool_size;  // gene pool
    uint32_t s;          // population size (elite count of eda_sample, modes.cpp:168)
    uint64_t seed, generation;
    ShiftMul M;  // {4, 32, 2}: see xorshift_r
};

// One child gene.  partner_row < 0 selects the EDA form: eda_sample over the whole parent
// population with add-one smoothing (ga_ops.cpp:214-238), then mutate; otherwise crossover
// (ga_ops.cpp:130-144) then mutate (:164-178).  `col1` = column + 1; the keys already include kGolden.
__device__ __forceinline__ int32_t child_gene(const VariationParams& P, const int32_t* __restrict__ pool,
                                              const int32_t* __restrict__ parent, int k, int col, int mine, int theirs,
                                              bool eda, uint64_t ks, uint64_t kc, uint64_t km, uint64_t ki, uint32_t col1) {
    // Exactly TWO hashes per gene and no divergent branch: the mutation-mask draw decides WHICH second
    // stream is read at this column (MutationIndex for a flipped gene, else CrossoverMask / Select) —
    // a flipped gene never needs its crossover draw (mutate overwrites it, ga_ops.cpp:171-174), and the
    // streams are counter-based, so the unread draw is simply never computed.
    const uint64_t um = hash_tail(stream_at(km, col1), P.M);
    const bool flip = P.pm_always || um < P.pm_limit;
#if GAPA_VARY_ARITH & 4
    // speculative: both candidate second draws, three independent chains per gene instead of two dependent ones
    const uint64_t u2i = hash_tail(stream_at(ki, col1), P.M), u2c = hash_tail(stream_at(eda ? ks : kc, col1), P.M);
    const uint64_t u2 = flip ? u2i : u2c;
#else
    const uint64_t u2 = hash_tail(stream_at(flip ? ki : (eda ? ks : kc), col1), P.M);
#endif
    const uint32_t bound = flip ? P.pool_size : P.s + P.pool_size;  // next_index bound (rng.hpp:28-31)
    const uint32_t idx = mulhi_u64_u32(u2, bound);
    if (flip) return static_cast<int32_t>(idx);
    if (eda) return idx < P.s ? pool[static_cast<size_t>(parent[idx]) * k + col] : static_cast<int32_t>(idx - P.s);
    return (P.pc_always || u2 < P.pc_limit) ? theirs : mine;
}


inline VariationParams make_variation_params(double pc, double pm, uint32_t pool_size, int s, uint64_t seed, uint64_t generation) {
    const uint64_t tc = bernoulli_threshold(pc), tm = bernoulli_threshold(pm);
    VariationParams P;
    P.pc_always = tc >= (1ull << 53);
    P.pm_always = tm >= (1ull << 53);
    P.pc_limit = P.pc_always ? ~0ull : tc << 11;
    P.pm_limit = P.pm_always ? ~0ull : tm << 11;
    P.pool_size = pool_size;
    P.s = static_cast<uint32_t>(s);
    P.seed = seed;
    P.generation = generation;
    P.M = ShiftMul{1u << 2, 1u << 5, 1u << 1};
    return P;
}

// What the evaluators need to BUILD the children they evaluate (row r of the batch = child of
// global row row_first + r): the fused PC path writes each child gene to its slot and into the
// shared-memory bitmap in the same pass.
struct VariationSpec {
    VariationParams P;
    int32_t* pool;           // 2s x k row slots
    const int32_t* parent;   // slot tables
    const int32_t* child;
    const int32_t* partner;  // nullptr = EDA generation
    int row_first;
    // Row-sharded runs over peer memory (run.cu): slot tables are identical on every rank, but a rank holds only the rows
    // it built or has read before.  home[slot] = the rank whose pool holds the row (its builder, or this rank once the
    // row has been adopted); bases[r] = rank r's pool as mapped here (NVLink peer access / CUDA IPC).  A parent row
    // that lives elsewhere is read straight from its builder's HBM and written through to the local slot on the way.
    // bases == nullptr: everything is local.
    const int32_t* const* bases = nullptr;
    const int32_t* home = nullptr;
    int self = 0;
};

// where parent row `slot` is read from; *remote tells the caller to write it through to the local slot
__device__ __forceinline__ const int32_t* parent_row(const VariationSpec& V, int slot, int k, bool* remote) {
    *remote = false;
    if (V.bases) {
        const int h = V.home[slot];
        if (h != V.self) {
            *remote = true;
            return V.bases[h] + static_cast<size_t>(slot) * k;
        }
    }
    return V.pool + static_cast<size_t>(slot) * k;
}

}  // namespace gapa_b200
