// ring_rt.cuh -- the runtime-matrix ring kernel template and its launchers,
// included by one translation unit per ring geometry (ring_rt_w*_n*.cu): each
// geometry's instances form their own CUDA module, so the first decode of a
// process loads only the module of its field (lazy module loading loads a whole
// module on first use: ~29 ms for all geometries in one module, measured).
#pragma once
// Runtime-matrix ring kernel (K2 of SURVEY.md section 8): one ahead-of-time
// sm_100a kernel per ring geometry (w, n) that applies ANY e x k matrix of
// ring representatives -- the encode generator or the survivor-inverse
// rows of a decode -- without generating or compiling code for it.
//
// Semantics are those of the generated ring programs (program.cpp), i.e.
// the reference's compile_schedule + replay (schedule.hpp:94-163,
// codec.hpp:118-157): ring row t of output i accumulates input strip
// (t - sh) mod n for every set bit sh of the representative of entry (i, j);
// Embedding inputs have w strips (strips >= w are zero, transform.hpp:32-35)
// and the output folds row t >= w onto the rows of x^t mod p
// (transform.hpp:39-46, generalised); Parity inputs are extended by their
// column parities (phi_P, transform.hpp:50-60) and the output is truncated
// to rows < w (transform.hpp:63-66).
//
// Layout of the work (persistent CTAs, 16 warps per SM):
//   * one elected thread streams every input fragment tile (all w strips x
//     2 KiB) into a ring of shared-memory slots with one TMA tensor box
//     (cp.async.bulk.tensor.3d) per (tile, fragment), tracked by FULL/EMPTY
//     mbarriers: in the four-part shape a thread of a producer warp group that
//     has handed its registers to the consumers (setmaxnreg), filling slots as
//     fast as they empty; in the smaller shapes the first thread of the
//     lightest part, NSLOT-1 fragments ahead;
//   * R parts of 2048/(4V) threads split the outputs (E accumulated outputs
//     each); a thread owns 4V bytes of every strip of the tile: it reads the w strip
//     words of a fragment from shared memory into registers and runs the
//     fragment's op list -- each op (i, sh) a warp-uniform jump (brx.idx)
//     into a compile-time XOR block "acc_i ^= x rotated by sh", so every
//     accumulator index is a fixed register although the matrix is runtime;
//     two shifts sh, sh+d (d <= PYRIT_RT_PAIR_D) of one representative may be
//     one op (i, sh, d): rows both reach take one 3-input LOP3;
//   * after the last fragment the accumulators are folded (Embedding:
//     x^t mod p, compile-time per field) and stored once with st.global.cs.
// Every input byte is read from HBM once and every output byte written once.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.hpp"

namespace pyrit_b200 {

namespace rt_detail {

typedef std::uint32_t u32;
typedef std::uint64_t u64;

__device__ __forceinline__ u32 smem_u32(const void* p) {
    return static_cast<u32>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(u32 bar, u32 count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(u32 bar, u32 bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
                 : "memory");
}
// lane 0 arrives, predicated rather than branched (no divergent region)
__device__ __forceinline__ void mbar_arrive_lane0(u32 bar, u32 lane) {
    asm volatile(
        "{\n .reg .pred p;\n setp.eq.u32 p, %1, 0;\n @p mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];\n}" ::"r"(bar),
        "r"(lane)
        : "memory");
}
__device__ __forceinline__ void mbar_wait(u32 bar, u32 parity) {
    asm volatile(
        "{\n .reg .pred P1;\n WAIT:\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n @P1 bra DONE;\n"
        " bra WAIT;\n DONE:\n}" ::"r"(bar),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma3d(u32 dst, const void* map, u32 x, u32 y, u32 z, u32 bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];" ::"r"(dst),
        "l"(map), "r"(x), "r"(y), "r"(z), "r"(bar)
        : "memory");
}
template <int V>
__device__ __forceinline__ void lds(u32 (&v)[V], u32 addr) {
    if constexpr (V == 1) asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v[0]) : "r"(addr));
    else if constexpr (V == 2) asm volatile("ld.shared.v2.b32 {%0, %1}, [%2];" : "=r"(v[0]), "=r"(v[1]) : "r"(addr));
    else asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]) : "r"(addr));
}
template <int V>
__device__ __forceinline__ void st_cs(std::uint8_t* p, const u32 (&v)[V]) {
    if constexpr (V == 1) asm volatile("st.global.cs.b32 [%0], %1;" ::"l"(p), "r"(v[0]) : "memory");
    else if constexpr (V == 2) asm volatile("st.global.cs.v2.b32 [%0], {%1, %2};" ::"l"(p), "r"(v[0]), "r"(v[1]) : "memory");
    else asm volatile("st.global.cs.v4.b32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]) : "memory");
}

// One pipeline op: c = (i*(D+1) + ds)*N + sh XORs the input, rotated by sh ring
// positions (ds = 0) or by sh and sh+ds (a pair), into the accumulators of output i (Embedding: W nonzero input strips, all N
// rows kept for the fold; Parity: N input strips, rows >= W dropped).  The
// specialisations (build/generated/ring_rt_ops.inc, gen_ring_rt.py) are one
// inline-PTX brx.idx jump table each: warp-uniform, and every accumulator
// index inside a case is a compile-time register.
template <int W, int N, int E, int V, bool PAR>
struct RtOps;
#include "ring_rt_ops.inc"

constexpr u32 kTile = kRtTile; // bytes per strip per tile (2 KiB)

// x^t mod p (the Embedding fold row of ring position t >= w)
__host__ __device__ constexpr u32 xpow_mod(int t, u32 p, int w) {
    u64 a = u64(1) << t;
    for (int d = t; d >= w; --d)
        if ((a >> d) & 1u) a ^= u64(p) << (d - w);
    return static_cast<u32>(a);
}

// R parts of CPP threads, V 32-bit words of every strip per thread; a CTA is
// 256 or 512 threads and an SM holds 512 (16 warps, <= 128 registers each)
// GRP: more than one output group (units = tiles x groups); without it the
// group is the constant 0 and its parameters are loop invariant
// PW (the four-part shape only): a producer warp group of 128 threads after the R parts;
// lane 0 of its first warp issues every TMA copy, so the consumer loop carries no producer
// code and no consumer warp waits on an EMPTY barrier.  20 warps would cap every thread at
// 96 registers, so the producer group gives its registers back (setmaxnreg.dec 24) and
// the consumers take them (setmaxnreg.inc 112): the CTA was given 640 x 96 registers
// and 512 x 112 + 128 x 24 fit in them (120 would not: the increase would wait for ever).
template <int W, int N, u32 P, int E, int R, int V, bool PAR, bool GRP, bool PW>
__global__ void __launch_bounds__(R * (kRtTile / (4 * V)) + (PW ? 128 : 0), 512 / (R * (kRtTile / (4 * V))))
    ring_rt_kernel(const __grid_constant__ RtArgs a) {
    constexpr u32 TILE = kTile, CPP = kRtTile / (4u * V);
    constexpr u32 SLOT = W * TILE;  // one fragment tile
    constexpr int AR = PAR ? W : N; // accumulator rows
    constexpr int XR = PAR ? N : W; // input rows held in registers
    extern __shared__ __align__(1024) std::uint8_t sm[];
    const u32 sbase = smem_u32(sm);
    const u32 ns = a.nslot;
    const u32 k = a.k;
    const u32 ntiles = a.ntiles, tpb = a.tpb;
    const u32 G = GRP ? a.ngrp : 1u, nunits = ntiles * G; // unit u = (tile u / G, output group u % G)
#define FULL(s) (sbase + 8u * (s))
#define EMPTY(s) (sbase + 8u * (ns + (s)))
    if (threadIdx.x == 0) {
        for (u32 s = 0; s < ns; ++s) {
            mbar_init(FULL(s), 1);
            mbar_init(EMPTY(s), R * CPP / 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    // the op lists go to shared memory (after the barriers), where the
    // threaded dispatch reads them one byte per op
    const u32 ops_s = sbase + 16u * ns;
    for (u32 i = threadIdx.x; i < a.nops; i += blockDim.x) sm[16u * ns + i] = a.ops[i];
    __syncthreads();
    // programmatic dependent launch: the setup above overlaps the previous
    // grid's tail; global memory is touched only after it has completed
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const u32 lane = threadIdx.x & 31u;
    // producer (the first thread of the part whose outputs weigh least, so the
    // copies are not issued from the critical path):
    // the next unit to load, (tile pt of this CTA, fragment pj) into slot psl
    // of phase pph; NSLOT-1 units run ahead
    u32 pj = 0, pu = blockIdx.x, psl = 0, pph = 0, pb = 0, px = 0;
    auto produce = [&]() {
        if (pu >= nunits) return;
        if (pj == 0) {
            const u32 pt = GRP ? pu / G : pu;
            pb = pt / tpb;
            px = static_cast<u32>((a.off + u64(pt - pb * tpb) * TILE) / 8u); // 8-byte TMA elements
        }
        mbar_wait(EMPTY(psl), pph ^ 1u);
        mbar_expect_tx(FULL(psl), SLOT);
        tma3d(a.slot0 + sbase + psl * SLOT, &a.tm[pj], px, 0u, pb, FULL(psl));
        if (++psl == ns) psl = 0, pph ^= 1u;
        if (++pj == k) pj = 0, pu += gridDim.x;
    };
    const u32 PROD = a.prod;
    if constexpr (PW) {
        if (threadIdx.x >= R * CPP) { // the producer group: slots fill as fast as they empty
            asm volatile("setmaxnreg.dec.sync.aligned.u32 24;");
            if (threadIdx.x == R * CPP)
                while (pu < nunits) produce();
            return; // (exited threads count as having let dependents launch)
        }
        asm volatile("setmaxnreg.inc.sync.aligned.u32 112;");
    } else {
        if (threadIdx.x == PROD)
            for (u32 u2 = 0; u2 + 1 < ns; ++u2) produce();
    }
    const u32 part = R == 1 ? 0u : threadIdx.x / CPP;
    const u32 col = R == 1 ? threadIdx.x : threadIdx.x % CPP;
    const u64 S = a.S;
    u32 sl = 0, ph = 0;
    for (u32 u = blockIdx.x; u < nunits; u += gridDim.x) {
        const u32 t = GRP ? u / G : u, g = GRP ? u - t * G : 0u;
        const u32 b = t / tpb, tt = t - b * tpb;
        const u32 ep = a.epart[g][part];
        const u32 list0 = ops_s + a.opoff[g][part][0]; // this part's op lists, input 0 first
        u32 acc[E][AR][V];
#pragma unroll
        for (int i = 0; i < E; ++i)
#pragma unroll
            for (int r = 0; r < AR; ++r)
#pragma unroll
                for (int v = 0; v < V; ++v) acc[i][r][v] = 0;
        // op cursor: q the next byte, d the op already loaded; the lists of
        // inputs 0..k-1 follow each other, each ended by its sentinel
        u32 q = list0 + 1, d;
        asm volatile("ld.shared.u8 %0, [%1];" : "=r"(d) : "r"(list0));
        // not unrolled: ptxas would duplicate the whole case table per copy of the
        // body (the instruction cache holds one)
#pragma unroll 1
        for (u32 j = 0; j < k; ++j) {
            if constexpr (!PW)
                if (threadIdx.x == PROD) produce();
            mbar_wait(FULL(sl), ph);
            u32 x[XR][V];
            const u32 src = a.slot0 + sbase + sl * SLOT + col * (4u * V);
#pragma unroll
            for (int s = 0; s < W; ++s) lds<V>(x[s], src + s * TILE);
            __syncwarp();
            mbar_arrive_lane0(EMPTY(sl), lane);
            if (++sl == ns) sl = 0, ph ^= 1u;
            if constexpr (PAR) {
                // column parities: strip W+q = XOR of strips i = q (mod s)
                // (word masks in the constant bank, fm[q*W + i])
#pragma unroll
                for (int q = W; q < N; ++q)
#pragma unroll
                    for (int v = 0; v < V; ++v) {
                        u32 p = 0;
#pragma unroll
                        for (int i = 0; i < W; ++i) p ^= x[i][v] & a.fm[(q - W) * W + i];
                        x[q][v] = p;
                    }
            }
            // this part's op list of input j (shared memory, sentinel-terminated)
            RtOps<W, N, E, V, PAR>::run(q, d, acc, x);
        }
        const u64 rel = u64(tt) * TILE + col * (4u * V);
        const bool live = rel < a.len;
        const u64 o = a.off + rel + u64(b) * a.obp;
#pragma unroll
        for (int i = 0; i < E; ++i) {
            if (i >= static_cast<int>(ep)) break;
            if constexpr (!PAR) {
                // fold: ring row t >= W onto the rows of x^t mod p
#pragma unroll
                for (int t2 = W; t2 < N; ++t2)
#pragma unroll
                    for (int r = 0; r < W; ++r)
                        if ((xpow_mod(t2, P, W) >> r) & 1u)
#pragma unroll
                            for (int v = 0; v < V; ++v) acc[i][r][v] ^= acc[i][t2][v];
            }
            if (live) {
                std::uint8_t* dst = a.out[g][part * kRtPartE + i] + o;
#pragma unroll
                for (int r = 0; r < W; ++r) st_cs<V>(dst + r * S, acc[i][r]);
            }
        }
    }
#undef FULL
#undef EMPTY
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

template <int W, int N, u32 P, int E, int R, int V, bool PAR, bool GRP, bool PW>
cudaError_t launch_pw(const RtArgs& a, const RtLaunch& l) {
    auto fn = ring_rt_kernel<W, N, P, E, R, V, PAR, GRP, PW>;
    static bool attr_set[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 64 && !attr_set[dev]) {
        const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        if (e != cudaSuccess) return e;
        attr_set[dev] = true;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(l.blocks);
    cfg.blockDim = dim3(R * rt_part_threads(V) + (PW ? 128 : 0));
    cfg.dynamicSmemBytes = l.smem;
    cfg.stream = l.stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = l.pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, fn, a);
}

template <int W, int N, u32 P, int E, int R, int V, bool PAR, bool GRP>
cudaError_t launch_grp(const RtArgs& a, const RtLaunch& l) {
    if constexpr (R == 4 && V == 4)
        if (l.pw) return launch_pw<W, N, P, E, R, V, PAR, GRP, true>(a, l);
    return launch_pw<W, N, P, E, R, V, PAR, GRP, false>(a, l);
}

template <int W, int N, u32 P, int E, int R, int V, bool PAR>
cudaError_t launch_one(const RtArgs& a, const RtLaunch& l) {
    if (a.ngrp > 1) return launch_grp<W, N, P, E, R, V, PAR, true>(a, l);
    return launch_grp<W, N, P, E, R, V, PAR, false>(a, l);
}

template <int W, int N, u32 P, int R, int V, bool PAR, int E>
cudaError_t launch_e(const RtArgs& a, const RtLaunch& l) {
    if constexpr (E >= 1) {
        if (l.E == E) return launch_one<W, N, P, E, R, V, PAR>(a, l);
        return launch_e<W, N, P, R, V, PAR, E - 1>(a, l);
    }
    return cudaErrorInvalidValue;
}

template <int W, int N, u32 P, int R, int V>
cudaError_t launch_rv(const RtArgs& a, const RtLaunch& l) {
    constexpr int EP = rt_part_outputs(N, W, V);
    return l.parity ? launch_e<W, N, P, R, V, true, EP>(a, l) : launch_e<W, N, P, R, V, false, EP>(a, l);
}

// (R, V) shapes: a single output runs one 256-thread part per CTA (two CTAs
// per SM); V = 2 pairs two 256-thread parts, V = 4 two (two CTAs per SM) or
// four 128-thread parts
template <int W, int N, u32 P>
cudaError_t launch_wn(const RtArgs& a, const RtLaunch& l) {
    if (l.R == 1 && l.V == 2)
        return l.parity ? launch_one<W, N, P, 1, 1, 2, true>(a, l) : launch_one<W, N, P, 1, 1, 2, false>(a, l);
    if (l.R == 2 && l.V == 2) return launch_rv<W, N, P, 2, 2>(a, l);
    if (l.R == 2 && l.V == 4) return launch_rv<W, N, P, 2, 4>(a, l);
    if (l.R == 4 && l.V == 4) return launch_rv<W, N, P, 4, 4>(a, l);
    return cudaErrorInvalidValue;
}

} // namespace rt_detail

} // namespace pyrit_b200
