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
#ifndef GAPA_VARY_ARITH
#define GAPA_VARY_ARITH 2
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
// mix64(x) up to, but not including, its last xor-shift; y = x + kGolden (rng.hpp:8-13)
__device__ __forceinline__ uint64_t hash_body(uint64_t y) {
    y = mul64_const(y ^ (y >> 30), 0xBF58476D1CE4E5B9ull);
    return mul64_const(y ^ (y >> 27), 0x94D049BB133111EBull);
}
__device__ __forceinline__ uint64_t hash_tail(uint64_t y) {
    y = hash_body(y);
    return y ^ (y >> 31);
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
};

// One child gene.  partner_row < 0 selects the EDA form: eda_sample over the whole parent
// population with add-one smoothing (ga_ops.cpp:214-238), then mutate; otherwise crossover
// (ga_ops.cpp:130-144) then mutate (:164-178).  `prod` = kCounterStep * (column + 1); the keys
// already include kGolden.
__device__ __forceinline__ int32_t child_gene(const VariationParams& P, const int32_t* __restrict__ pool,
                                              const int32_t* __restrict__ parent, int k, int col, int mine, int theirs,
                                              bool eda, uint64_t ks, uint64_t kc, uint64_t km, uint64_t ki, uint64_t prod) {
    // Exactly TWO hashes per gene and no divergent branch: the mutation-mask draw decides WHICH second
    // stream is read at this column (MutationIndex for a flipped gene, else CrossoverMask / Select) —
    // a flipped gene never needs its crossover draw (mutate overwrites it, ga_ops.cpp:171-174), and the
    // streams are counter-based, so the unread draw is simply never computed.
    const uint64_t um = hash_tail(km + prod);
    const bool flip = P.pm_always || um < P.pm_limit;
#if GAPA_VARY_ARITH & 4
    // speculative: both candidate second draws, three independent chains per gene instead of two dependent ones
    const uint64_t u2i = hash_tail(ki + prod), u2c = hash_tail((eda ? ks : kc) + prod);
    const uint64_t u2 = flip ? u2i : u2c;
#else
    const uint64_t u2 = hash_tail((flip ? ki : (eda ? ks : kc)) + prod);
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
