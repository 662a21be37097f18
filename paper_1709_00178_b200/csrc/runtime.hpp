// Device runtime: compiles generated ring programs for sm_100a (prebuilt
// cubins shipped next to the library, else NVRTC at first use), caches the
// loaded modules per device, and launches them.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "program.hpp"

namespace pyrit_b200 {

// CUDA-side failure: carries a negative C-ABI code (see pyrit_b200.h)
class CudaFailure : public std::runtime_error {
public:
    CudaFailure(int code, const std::string& what) : std::runtime_error(what), code_(code) {}
    int code() const noexcept { return code_; }

private:
    int code_;
};

void check_cuda(cudaError_t e, const char* what);

struct LaunchInfo {
    std::uint32_t lanes = 1, threads = 0, blocks = 0;
    bool staged = false;
    std::string kernel;
};

// Apply the program to the byte window [off, off+len) of every strip.
// in[j] / out[i] are device base pointers of input / output symbols; strip
// s of a symbol starts at base + s * strip.  Asynchronous on `stream`.
LaunchInfo launch_program(const Program& p, const std::uint8_t* const* in, std::uint8_t* const* out,
                          std::uint64_t strip, std::uint64_t off, std::uint64_t len, cudaStream_t stream);

// Stripe batch: the same window of `nb` stripes in one launch; input j of
// stripe b is at in[j] + b * in_pitch, output i at out[i] + b * out_pitch
// (the per-stripe encode()/decode() calls of encode_file/decode_file,
// container.hpp:207-218 and :284-297, batched).
LaunchInfo launch_batch(const Program& p, const std::uint8_t* const* in, std::uint8_t* const* out,
                        std::uint64_t strip, std::uint64_t off, std::uint64_t len, std::uint64_t nb,
                        std::uint64_t in_pitch, std::uint64_t out_pitch, cudaStream_t stream);

// Force compilation/loading for the current device (no launch).
std::string prepare_program(const Program& p, std::uint32_t lanes);

// Lanes (32-bit words per thread per strip) preferred when alignment allows.
std::uint32_t preferred_lanes();
void set_preferred_lanes(std::uint32_t lanes);

// Is plan_key `key` one of the programs with a prebuilt specialised kernel
// (kernels/prebuilt.tsv, written by build.py)?
bool prebuilt_plan(const std::string& key);

// Directory searched for prebuilt <kernel>.cubin files.
void set_kernel_dir(const std::string& dir);
std::string kernel_dir();

LaunchInfo last_launch(); // this thread's most recent launch_program
std::uint64_t jit_compiles(); // number of NVRTC compilations performed so far
void jit_time(double* last_ms, double* total_ms); // wall time of the last / all compiles
std::string jit_info();
void jit_wait(); // wait for every background (tiered) compile started so far       // "nvrtc <major>.<minor> (<library file>)"; throws if NVRTC cannot be loaded
std::uint64_t kernel_launches(); // number of generated-kernel launches so far

KernelShape shape_for(std::uint32_t lanes);
// direct-kernel shape for p: rows split over thread groups when p has several output parts
KernelShape direct_shape(const Program& p, std::uint32_t lanes);

// 0 = auto (TMA-staged whenever alignment allows), 1 = direct LDG only, 2 = staged,
// 3 = generic bit-matrix kernel, 4 = runtime-matrix ring kernel (ring_rt.cu)
int kernel_mode();
// PYRIT_B200_RT: 0 = never use the runtime-matrix ring kernel, 1 (default) =
// for launches whose generated kernel is not ready and for ad-hoc programs
// (decode patterns), 2 = for every eligible launch
int rt_policy();
// can the runtime-matrix ring kernel run this launch (prebuilt geometry,
// 16-byte alignment, k <= 64, outputs aliasing inputs only column for column)
void ring_rt_plan_info(const Program& p, std::uint32_t info[4]);
void interpret_ring_rt(const Program& p, const std::uint8_t* const* in, std::uint8_t* const* out, std::uint64_t strip,
                       std::uint64_t off, std::uint64_t len, std::uint64_t nb, std::uint64_t in_pitch,
                       std::uint64_t out_pitch);
bool ring_rt_eligible(const Program& p, const std::uint8_t* const* in, std::uint8_t* const* out, std::uint64_t strip,
                      std::uint64_t off, std::uint64_t len, std::uint64_t nb, std::uint64_t in_pitch,
                      std::uint64_t out_pitch);
LaunchInfo launch_ring_rt_program(const Program& p, const std::uint8_t* const* in, std::uint8_t* const* out,
                                  std::uint64_t strip, std::uint64_t off, std::uint64_t len, std::uint64_t nb,
                                  std::uint64_t in_pitch, std::uint64_t out_pitch, cudaStream_t stream);
void set_kernel_mode(int mode);
// the kernel shape a launch with these arguments uses
KernelShape choose_shape(const Program& p, const std::uint8_t* const* in, std::uint8_t* const* out,
                         std::uint64_t strip, std::uint64_t off, std::uint64_t len, std::uint64_t nb = 1,
                         std::uint64_t in_pitch = 0, std::uint64_t out_pitch = 0);

} // namespace pyrit_b200
