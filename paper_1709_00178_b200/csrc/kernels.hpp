// Ahead-of-time utility kernels (kernels.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace pyrit_b200 {

cudaError_t launch_fill(std::uint64_t seed, std::uint64_t frag, std::uint8_t* dst, std::uint64_t begin,
                        std::uint64_t len, std::uint64_t valid, cudaStream_t stream);
cudaError_t launch_digest(const std::uint8_t* src, std::uint64_t len, std::uint64_t word_offset,
                          std::uint64_t* out, cudaStream_t stream);

// Generic bit-matrix kernel (kernels.cu): all in kernel parameters.
constexpr std::uint32_t kGenericMaxPtrs = 256;     // inputs + outputs
constexpr std::uint32_t kGenericMaxMasks = 12288;  // e * w rows x k inputs
struct GenericArgs {
    std::uint64_t S, off, nwords, nb, ibp, obp, sq, sr; // as the direct kernel (4-byte words)
    std::uint32_t k, e, w, pad;
    const std::uint8_t* ptr[kGenericMaxPtrs];  // k inputs, then e outputs
    std::uint16_t mask[kGenericMaxMasks];      // mask[(i*w + b)*k + j]: strips of input j in output i strip b
};
cudaError_t launch_generic(const GenericArgs& args, unsigned blocks, cudaStream_t stream);

// Runtime-matrix ring kernel (ring_rt.cu): one ahead-of-time kernel per ring
// geometry (w, n) applies any e x k matrix of ring representatives passed in
// kernel parameters -- no per-code or per-erasure-pattern compilation.
constexpr std::uint32_t kRtMaxK = 64;    // inputs per launch (one TMA tensor map each)
constexpr std::uint32_t kRtParts = 4;    // output parts per CTA (all read the same shared-memory tiles)
constexpr std::uint32_t kRtPartE = 8;    // output slots per part
// output groups per launch: a tile is a unit per group, so a code with more
// outputs than one CTA holds is still one launch; the groups of a tile run on
// neighbouring CTAs at about the same time, so only the first reads HBM and
// the others hit L2
constexpr std::uint32_t kRtMaxGroups = 8;
constexpr std::uint32_t kRtMaxOps = 8192; // (output, shift) ops per launch
constexpr std::uint32_t kRtTile = 2048;  // bytes per strip per tile (4*V per thread)
constexpr std::uint32_t kRtBox = kRtTile / 8; // TMA box width in 8-byte elements
// threads per part: one 4*V-byte word group of every strip of the tile each
// (thread 0 of the CTA also issues the TMA copies)
constexpr std::uint32_t rt_part_threads(std::uint32_t v) { return kRtTile / (4 * v); }
struct alignas(64) RtArgs {
    std::uint64_t tm[kRtMaxK][16];       // CUtensorMap per input: (8-byte column element, strip, stripe)
    std::uint8_t* out[kRtMaxGroups][kRtParts * kRtPartE]; // output bases of group g, part p at [g][p*kRtPartE ..]
    std::uint64_t S, off, len, nb, obp;
    std::uint32_t k, tpb, ntiles, nslot, slot0; // slot0: byte offset of slot 0 in shared memory
    std::uint32_t nops;                         // bytes of ops[] (op lists with their sentinels)
    std::uint32_t prod;                         // thread that issues the TMA copies (first of the lightest part)
    std::uint32_t ngrp;                  // output groups (units per tile)
    std::uint32_t epart[kRtMaxGroups][kRtParts]; // outputs of each part of each group
    std::uint32_t fm[256]; // Parity: fm[q*w + i] = ~0 when strip i feeds the parity strip w+q (i = q mod s)
    // op list of input j for part p of group g: ops[opoff[g][p][j] ..], each
    // c = (i*(D+1) + ds)*n + sh with D = rt_pair_d(w, n, V): output i of the part
    // accumulates input j rotated by sh ring positions (ds = 0) or by sh and sh+ds
    // (a pair) -- set bits of the representative of entry (i, j) -- terminated by E*(D+1)*n
    std::uint16_t opoff[kRtMaxGroups][kRtParts][kRtMaxK + 1];
    std::uint8_t ops[kRtMaxOps];
};
struct RtLaunch {
    std::uint32_t w = 0, n = 0, modulus = 0, E = 0, R = 2, V = 2; // E outputs in each of R parts, V words
    bool parity = false, pdl = true;
    bool pw = false; // R = 4, V = 4 only: a producer warp group issues the TMA copies (ring_rt.cuh)
    unsigned blocks = 1;
    std::uint32_t smem = 0;
    cudaStream_t stream = nullptr;
};
// accumulated outputs per part for ring length n and V words per thread:
//   V = 2: e*n*2 accumulator registers within ~72 of the 128 a thread of a
//          512-thread CTA may hold;
//   V = 4: e*n*4 accumulators next to the w*4 input words, within ~104.
constexpr int rt_clamp_e(int e) { return e < 1 ? 1 : (e > 8 ? 8 : e); }
constexpr int rt_part_outputs(int n, int w, int v) {
    return v == 4 ? rt_clamp_e((104 - 4 * w) / (4 * n)) : rt_clamp_e(36 / n);
}
// Paired-shift cases: two shifts (sh, sh+d) of one representative are one op whose
// ring rows reached by both take a 3-input LOP3 (gen_ring_rt.py).  The V = 4 instances
// carry a case for every pair distance d <= PYRIT_RT_PAIR_D, a build-time constant
// (0: no pair cases).  PYRIT_RT_PAIR_AOP_ALL=1 builds every distance, (n-1)/2, in the
// all-one-polynomial fields (w = n-1), where two windows of w strips on the ring of n
// overlap in w-1 rows at ANY distance; measured no better (config 5 encode +2%, its
// four-symbol decode patterns -2%, profiles/r02/ring_rt_pairs/aop_all_distances/), so
// it is off.  Which cases a launch uses is the planner's choice (runtime.cpp
// rt_select_pairs: the cases that pay most within the instruction-cache budget).
// V = 2 instances (single output, HBM-bound) have none.
#ifndef PYRIT_RT_PAIR_D
#define PYRIT_RT_PAIR_D 3
#endif
#ifndef PYRIT_RT_PAIR_AOP_ALL
#define PYRIT_RT_PAIR_AOP_ALL 0
#endif
constexpr std::uint32_t rt_pair_d(std::uint32_t w, std::uint32_t n, std::uint32_t v) {
    return v != 4 || PYRIT_RT_PAIR_D == 0 ? 0u
           : (PYRIT_RT_PAIR_AOP_ALL && w + 1 == n) || (n - 1) / 2 < PYRIT_RT_PAIR_D ? (n - 1) / 2
                                                                                    : PYRIT_RT_PAIR_D;
}
bool rt_supported(std::uint32_t w, std::uint32_t n, std::uint32_t modulus);
cudaError_t launch_ring_rt(const RtArgs& a, const RtLaunch& l);
// load the runtime-matrix kernel's modules (one per ring geometry) on the current
// device now rather than on the first decode of a new pattern
cudaError_t warm_ring_rt();

} // namespace pyrit_b200
