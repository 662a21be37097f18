// Ahead-of-time sm_100a kernels that sit beside the generated ring
// programs: the seeded synthetic fragment generator and the K3 slice
// digest used for sharded verification.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "kernels.hpp"

namespace pyrit_b200 {

namespace {

__device__ __forceinline__ std::uint64_t mix64(std::uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// Byte o of fragment `frag` = byte o%8 (little endian) of
// mix64((seed << 48) ^ (frag << 36) ^ (o / 8)) for o < valid, else 0.
// One 8-byte word per thread; begin is a multiple of 8, dst 8-aligned.
__global__ void __launch_bounds__(256) fill_kernel(std::uint64_t seed, std::uint64_t frag, std::uint8_t* dst,
                                                   std::uint64_t begin, std::uint64_t len, std::uint64_t valid) {
    const std::uint64_t key = (seed << 48) ^ (frag << 36);
    const std::uint64_t words = (len + 7) / 8;
    for (std::uint64_t q = blockIdx.x * std::uint64_t(blockDim.x) + threadIdx.x; q < words;
         q += std::uint64_t(gridDim.x) * blockDim.x) {
        const std::uint64_t o = begin + 8 * q;
        std::uint64_t v = mix64(key ^ (o >> 3));
        if (o + 8 > valid) v = o >= valid ? 0 : (v & ((1ull << (8 * (valid - o))) - 1));
        if (8 * q + 8 <= len) {
            *reinterpret_cast<std::uint64_t*>(dst + 8 * q) = v;
        } else {
            for (std::uint64_t b = 8 * q; b < len; ++b) dst[b] = static_cast<std::uint8_t>(v >> (8 * (b - 8 * q)));
        }
    }
}

// D += sum_q mix64(word_q ^ ((word_offset + q) * 0xD6E8FEB86659FD93)),
// words little endian, trailing partial word zero padded.
__global__ void __launch_bounds__(256) digest_kernel(const std::uint8_t* src, std::uint64_t len,
                                                     std::uint64_t word_offset, unsigned long long* out) {
    const std::uint64_t words = (len + 7) / 8;
    std::uint64_t acc = 0;
    for (std::uint64_t q = blockIdx.x * std::uint64_t(blockDim.x) + threadIdx.x; q < words;
         q += std::uint64_t(gridDim.x) * blockDim.x) {
        std::uint64_t v;
        if (8 * q + 8 <= len) {
            v = __ldcs(reinterpret_cast<const unsigned long long*>(src + 8 * q));
        } else {
            v = 0;
            for (std::uint64_t b = 8 * q; b < len; ++b) v |= std::uint64_t(src[b]) << (8 * (b - 8 * q));
        }
        acc += mix64(v ^ ((word_offset + q) * 0xD6E8FEB86659FD93ull));
    }
    for (int s = 16; s > 0; s >>= 1) acc += __shfl_xor_sync(0xFFFFFFFFu, acc, s);
    __shared__ std::uint64_t part[8];
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        std::uint64_t t = 0;
        for (unsigned w = 0; w < blockDim.x / 32; ++w) t += part[w];
        atomicAdd(out, static_cast<unsigned long long>(t));
    }
}

unsigned grid_for(std::uint64_t words) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const std::uint64_t want = (words + 255) / 256;
    const std::uint64_t cap = std::uint64_t(sms) * 8;
    return static_cast<unsigned>(want < 1 ? 1 : (want < cap ? want : cap));
}

} // namespace

cudaError_t launch_fill(std::uint64_t seed, std::uint64_t frag, std::uint8_t* dst, std::uint64_t begin,
                        std::uint64_t len, std::uint64_t valid, cudaStream_t stream) {
    if (len == 0) return cudaSuccess;
    fill_kernel<<<grid_for((len + 7) / 8), 256, 0, stream>>>(seed, frag, dst, begin, len, valid);
    return cudaGetLastError();
}

cudaError_t launch_digest(const std::uint8_t* src, std::uint64_t len, std::uint64_t word_offset,
                          std::uint64_t* out, cudaStream_t stream) {
    if (len == 0) return cudaSuccess;
    digest_kernel<<<grid_for((len + 7) / 8), 256, 0, stream>>>(src, len, word_offset,
                                                               reinterpret_cast<unsigned long long*>(out));
    return cudaGetLastError();
}

} // namespace pyrit_b200

namespace pyrit_b200 {

// ---- generic bit-matrix kernel (no per-code compilation) -------------------
//
// Output strip b of output i = XOR over inputs j and strips c in mask(i, b, j)
// of input strip c -- the plain-field bitmatrix form of any code this library
// compiles (every ring program computes the GF(2^w) code, codec.hpp:444-469).
// It runs while a code's specialised kernel is still being compiled (tiered
// compilation, runtime.cpp) and on demand (kernel mode 3).  One 4-byte column
// word per thread, grid-stride over (stripe, word); the masks are uniform
// across a warp and come from the constant bank (__grid_constant__).
__global__ void __launch_bounds__(256) generic_kernel(const __grid_constant__ GenericArgs a) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const std::uint32_t k = a.k, e = a.e, w = a.w;
    const std::uint64_t S = a.S;
    std::uint64_t c0 = blockIdx.x * std::uint64_t(blockDim.x) + threadIdx.x;
    std::uint64_t b = c0 / a.nwords, cw = c0 - b * a.nwords;
    while (b < a.nb) {
        const std::uint64_t o = a.off + cw * 4;
        const std::uint64_t oi = o + b * a.ibp, oo = o + b * a.obp;
        for (std::uint32_t i = 0; i < e; ++i)
            for (std::uint32_t r = 0; r < w; ++r) {
                const std::uint16_t* row = &a.mask[(i * w + r) * k];
                std::uint32_t acc = 0;
                for (std::uint32_t j = 0; j < k; ++j) {
                    std::uint32_t m = row[j];
                    const std::uint8_t* p = a.ptr[j] + oi;
                    while (m) {
                        const std::uint32_t c = __ffs(m) - 1;
                        m &= m - 1;
                        acc ^= __ldg(reinterpret_cast<const std::uint32_t*>(p + c * S));
                    }
                }
                __stcs(reinterpret_cast<unsigned int*>(const_cast<std::uint8_t*>(a.ptr[k + i]) + oo + r * S), acc);
            }
        b += a.sq;
        cw += a.sr;
        if (cw >= a.nwords) {
            cw -= a.nwords;
            ++b;
        }
    }
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// The same with w a compile-time constant: the strips of an input are walked
// by an unrolled, warp-uniform predicate chain instead of a bit-scan loop.
template <int W>
__global__ void __launch_bounds__(256) generic_kernel_w(const __grid_constant__ GenericArgs a) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const std::uint32_t k = a.k, e = a.e;
    const std::uint64_t S = a.S;
    std::uint64_t c0 = blockIdx.x * std::uint64_t(blockDim.x) + threadIdx.x;
    std::uint64_t b = c0 / a.nwords, cw = c0 - b * a.nwords;
    while (b < a.nb) {
        const std::uint64_t o = a.off + cw * 4;
        const std::uint64_t oi = o + b * a.ibp, oo = o + b * a.obp;
        for (std::uint32_t i = 0; i < e; ++i)
#pragma unroll
            for (int r = 0; r < W; ++r) {
                const std::uint16_t* row = &a.mask[(i * W + r) * k];
                std::uint32_t acc = 0;
                for (std::uint32_t j = 0; j < k; ++j) {
                    const std::uint32_t m = row[j];
                    const std::uint8_t* p = a.ptr[j] + oi;
#pragma unroll
                    for (int c = 0; c < W; ++c)
                        if (m & (1u << c)) acc ^= __ldg(reinterpret_cast<const std::uint32_t*>(p + c * S));
                }
                __stcs(reinterpret_cast<unsigned int*>(const_cast<std::uint8_t*>(a.ptr[k + i]) + oo + r * S), acc);
            }
        b += a.sq;
        cw += a.sr;
        if (cw >= a.nwords) {
            cw -= a.nwords;
            ++b;
        }
    }
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

cudaError_t launch_generic(const GenericArgs& args, unsigned blocks, cudaStream_t stream) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(blocks);
    cfg.blockDim = dim3(256);
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    static const bool unrolled = [] {
        const char* v = std::getenv("PYRIT_B200_GENERIC_UNROLL");
        return !v || std::atoi(v) != 0;
    }();
    if (unrolled) switch (args.w) {
        case 4: return cudaLaunchKernelEx(&cfg, generic_kernel_w<4>, args);
        case 6: return cudaLaunchKernelEx(&cfg, generic_kernel_w<6>, args);
        case 8: return cudaLaunchKernelEx(&cfg, generic_kernel_w<8>, args);
        case 10: return cudaLaunchKernelEx(&cfg, generic_kernel_w<10>, args);
        case 12: return cudaLaunchKernelEx(&cfg, generic_kernel_w<12>, args);
        default: break;
        }
    return cudaLaunchKernelEx(&cfg, generic_kernel, args);
}

} // namespace pyrit_b200
