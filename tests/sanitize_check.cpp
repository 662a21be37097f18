// sanitize_check.cpp -- TEST INFRASTRUCTURE: a small, allocation-exact driver
// of every generated-kernel shape (staged 16/8/4-byte chunks, direct 4/8/16-byte
// lanes and byte mode, rows split over thread groups, stripe batches) for
// compute-sanitizer (memcheck / racecheck / synccheck), one tool per run:
//
//   compute-sanitizer --tool memcheck --error-exitcode 3 build/sanitize_check
//
// Every device buffer is allocated at exactly the size the launch may touch,
// so an out-of-bounds access is reported; results are compared with the
// library's host interpreter of the same compiled program.  (compute-sanitizer
// is closed on the GPU pool used here, so the driver also brackets every
// buffer with 4 KiB canary regions and checks that no launch wrote outside
// its buffers: plain runs catch stray stores too.)
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <random>
#include <vector>

#include "pyrit_b200.h"

namespace {

int failures = 0;

#define CK(x)                                                                                    \
    do {                                                                                         \
        cudaError_t e_ = (x);                                                                    \
        if (e_ != cudaSuccess) {                                                                 \
            std::printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
            std::exit(2);                                                                        \
        }                                                                                        \
    } while (0)

struct Case {
    const char* name;
    const char* field;
    unsigned k, r;
    unsigned transform;
    unsigned long long strip; // bytes per strip (symbol = w strips)
    unsigned long long stripes;
    int mode; // 0 auto, 1 direct, 2 staged, 3 generic bit-matrix, 4 runtime-matrix ring kernel
    const char* expect = nullptr; // prefix the launched kernel's name must have
};

void run(const Case& c) {
    pyrit_field f;
    if (pyrit_field_named(c.field, &f)) {
        std::printf("%s: bad field\n", c.name);
        ++failures;
        return;
    }
    pyrit_code code{c.k, c.r, f, c.transform};
    pyrit_plan* plan = nullptr;
    if (pyrit_plan_encode(&code, &plan)) {
        std::printf("%s: plan failed\n", c.name);
        ++failures;
        return;
    }
    pyrit_set_kernel_mode(c.mode);
    const unsigned long long sym = f.w * c.strip;
    std::mt19937_64 rng(c.k * 1000 + c.r + c.strip);
    // stripe b of input j at in[j] + b * sym (pitch = symbol), exact allocations
    std::vector<std::vector<unsigned char>> hin(c.k, std::vector<unsigned char>(sym * c.stripes));
    for (auto& v : hin)
        for (auto& x : v) x = static_cast<unsigned char>(rng());
    // one allocation per buffer: [canary | data | canary]
    constexpr unsigned long long kGuard = 4096;
    const unsigned long long bytes = sym * c.stripes;
    std::vector<unsigned char*> base(c.k + c.r), din(c.k), dout(c.r);
    std::vector<unsigned char> canary(kGuard);
    for (unsigned long long i = 0; i < kGuard; ++i) canary[i] = static_cast<unsigned char>(0xA5 ^ (i * 7));
    for (unsigned s = 0; s < c.k + c.r; ++s) {
        CK(cudaMalloc(&base[s], bytes + 2 * kGuard));
        CK(cudaMemcpy(base[s], canary.data(), kGuard, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(base[s] + kGuard + bytes, canary.data(), kGuard, cudaMemcpyHostToDevice));
        CK(cudaMemset(base[s] + kGuard, 0x5A, bytes));
    }
    for (unsigned j = 0; j < c.k; ++j) {
        din[j] = base[j] + kGuard;
        CK(cudaMemcpy(din[j], hin[j].data(), bytes, cudaMemcpyHostToDevice));
    }
    for (unsigned i = 0; i < c.r; ++i) dout[i] = base[c.k + i] + kGuard;
    int rc = pyrit_cu_apply_batch(plan, const_cast<const unsigned char* const*>(din.data()), dout.data(), c.strip,
                                  0, c.strip, c.stripes, sym, sym, nullptr);
    CK(cudaDeviceSynchronize());
    char kname[128] = {0};
    unsigned blocks = 0, threads = 0;
    pyrit_cu_last_launch(kname, sizeof kname, &blocks, &threads);
    bool ok = rc == 0;
    for (unsigned long long b = 0; ok && b < c.stripes; ++b) {
        std::vector<const unsigned char*> hi(c.k);
        std::vector<std::vector<unsigned char>> want(c.r, std::vector<unsigned char>(sym));
        std::vector<unsigned char*> ho(c.r);
        for (unsigned j = 0; j < c.k; ++j) hi[j] = hin[j].data() + b * sym;
        for (unsigned i = 0; i < c.r; ++i) ho[i] = want[i].data();
        pyrit_plan_interpret(plan, hi.data(), ho.data(), c.strip, 0, c.strip);
        std::vector<unsigned char> got(sym);
        for (unsigned i = 0; ok && i < c.r; ++i) {
            CK(cudaMemcpy(got.data(), dout[i] + b * sym, sym, cudaMemcpyDeviceToHost));
            ok = std::memcmp(got.data(), want[i].data(), sym) == 0;
        }
    }
    bool guards = true;
    std::vector<unsigned char> g(kGuard);
    for (unsigned s = 0; s < c.k + c.r; ++s)
        for (unsigned long long at : {0ull, kGuard + bytes}) {
            CK(cudaMemcpy(g.data(), base[s] + at, kGuard, cudaMemcpyDeviceToHost));
            guards = guards && std::memcmp(g.data(), canary.data(), kGuard) == 0;
        }
    for (unsigned j = 0; guards && j < c.k; ++j) { // inputs are read-only
        std::vector<unsigned char> back(bytes);
        CK(cudaMemcpy(back.data(), din[j], bytes, cudaMemcpyDeviceToHost));
        guards = back == hin[j];
    }
    const bool kind = !c.expect || std::strncmp(kname, c.expect, std::strlen(c.expect)) == 0;
    std::printf("%-34s mode %d %-52s %s%s%s\n", c.name, c.mode, kname, ok ? "OK" : "MISMATCH",
                guards ? "" : " (STRAY WRITE)", kind ? "" : " (UNEXPECTED KERNEL)");
    failures += !ok + !guards + !kind;
    for (auto* p : base) CK(cudaFree(p));
    pyrit_plan_destroy(plan);
    pyrit_set_kernel_mode(0);
}

} // namespace

int main() {
    const Case cases[] = {
        {"cfg1 gf16 k4 r2 (staged 16B)", "gf16", 4, 2, 0, 4096 + 48, 3, 2},
        {"cfg1 gf16 k4 r2 (direct)", "gf16", 4, 2, 0, 4096 + 48, 3, 1},
        {"cfg2 gf256/R17 k10 r4 (staged)", "gf256_r17", 10, 4, 0, 2048 + 16, 2, 2},
        {"cfg3 gf1024 k12 r4 (staged)", "gf1024", 12, 4, 0, 1024 + 32, 2, 2},
        {"cfg5 gf4096 k16 r4 (staged)", "gf4096", 16, 4, 0, 2048 + 16, 2, 2},
        {"cfg5 gf4096 k16 r4 (direct)", "gf4096", 16, 4, 0, 2048 + 16, 2, 1},
        {"gf64 k6 r3 (staged 8B chunks)", "gf64", 6, 3, 0, 1000, 2, 2},
        {"gf64 k6 r3 (staged 4B chunks)", "gf64", 6, 3, 0, 1004, 2, 2},
        {"gf64 k40 r20 (split rows)", "gf64", 40, 20, 0, 684, 2, 1},
        {"gf64 k20 r40 parity (staged)", "gf64", 20, 40, 1, 1024, 2, 2},
        {"gf16 k8 r4 (byte mode)", "gf16", 8, 4, 0, 129, 3, 1},
        {"gf16 k8 r4 (many tiny stripes)", "gf16", 8, 4, 0, 32, 257, 0},
        // runtime-matrix ring kernel (ring_rt.cu): one part (R=1), 2 parts in
        // 2 CTAs/SM, 4 parts with one idle, several launches, Parity transform
        {"cfg5 gf4096 k16 r4 (runtime 4 parts)", "gf4096", 16, 4, 0, 2048 + 16, 2, 4, "pyrit_ring_rt_"},
        {"cfg4 gf256/R17 k10 r4 (runtime)", "gf256_r17", 10, 4, 0, 4096 + 32, 2, 4, "pyrit_ring_rt_"},
        {"gf1024 k12 r3 (runtime, idle part)", "gf1024", 12, 3, 0, 2048 + 48, 2, 4, "pyrit_ring_rt_"},
        {"gf16 k4 r1 (runtime, one output)", "gf16", 4, 1, 0, 4096 + 16, 3, 4, "pyrit_ring_rt_"},
        {"gf16 k8 r2 (runtime, 2 parts)", "gf16", 8, 2, 0, 2048, 2, 4, "pyrit_ring_rt_"},
        {"gf64 k6 r9 (runtime, 2 launches)", "gf64", 6, 9, 0, 1024 + 16, 2, 4, "pyrit_ring_rt_"},
        {"gf64 k20 r4 parity (runtime)", "gf64", 20, 4, 1, 2048 + 32, 2, 4, "pyrit_ring_rt_"},
        {"gf4096 k16 r4 (generic bitmatrix)", "gf4096", 16, 4, 0, 1024 + 4, 2, 3, "pyrit_generic"},
    };
    for (const Case& c : cases) run(c);
    std::printf(failures ? "SANITIZE CHECK FAILED\n" : "SANITIZE CHECK PASSED\n");
    return failures ? 1 : 0;
}
