// Host-side sanitizer driver, GPU half (test infrastructure; see
// tests/host_sanitize_check.cpp for the device-free half).  Linked against the
// library's host sources built with -fsanitize=address,undefined, it runs the
// HOST-BUFFER entry points on a real device -- pyrit_encode_host /
// pyrit_decode_host / pyrit_encode_crs_host / pyrit_apply_host (pageable,
// exact-size malloc buffers: ASan red zones sit right behind every buffer the
// staging copies touch), the multi-device shard variants with a repeated
// device, small pipeline chunks (many chunks, several staging slots), the
// device-pointer batch calls, the runtime-matrix path on a new erasure
// pattern, the file codec into a temporary directory, and concurrent callers
// -- and checks every result against the library's host interpreter.
//   ASAN_OPTIONS=protect_shadow_gap=0:detect_leaks=0 build/asan/host_sanitize_gpu
#include <cuda_runtime.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "pyrit_b200.h"

namespace {

std::atomic<int> g_fail{0};
std::atomic<unsigned long> g_checks{0};

#define CHECK(cond, ...)                                               \
    do {                                                               \
        ++g_checks;                                                    \
        if (!(cond)) {                                                 \
            ++g_fail;                                                  \
            std::fprintf(stderr, "FAIL %s:%d: ", __FILE__, __LINE__);  \
            std::fprintf(stderr, __VA_ARGS__);                         \
            std::fprintf(stderr, "\n");                                \
        }                                                              \
    } while (0)

struct Heap { // exact-size pageable block
    std::uint8_t* p;
    std::size_t n;
    explicit Heap(std::size_t bytes, std::mt19937_64* rng = nullptr) : n(bytes) {
        if (posix_memalign(reinterpret_cast<void**>(&p), 64, std::max<std::size_t>(bytes, 1)) != 0) std::abort();
        if (rng) {
            std::size_t i = 0;
            for (; i + 8 <= bytes; i += 8) {
                const std::uint64_t v = (*rng)();
                std::memcpy(p + i, &v, 8);
            }
            for (; i < bytes; ++i) p[i] = static_cast<std::uint8_t>((*rng)());
        } else {
            std::memset(p, 0x5A, bytes);
        }
    }
    Heap(const Heap&) = delete;
    Heap& operator=(const Heap&) = delete;
    ~Heap() { std::free(p); }
};

// expected parity / repaired symbols through the host interpreter of the plan
void reference_encode(const pyrit_code& code, const std::uint8_t* data, std::uint8_t* parity, std::uint64_t sym) {
    pyrit_plan* plan = nullptr;
    CHECK(pyrit_plan_encode(&code, &plan) == 0, "plan_encode");
    std::vector<const std::uint8_t*> in(code.k);
    std::vector<std::uint8_t*> out(code.r);
    for (std::uint32_t j = 0; j < code.k; ++j) in[j] = data + j * sym;
    for (std::uint32_t i = 0; i < code.r; ++i) out[i] = parity + i * sym;
    const std::uint64_t strip = sym / code.field.w;
    CHECK(pyrit_plan_interpret(plan, in.data(), out.data(), strip, 0, strip) == 0, "interpret");
    pyrit_plan_destroy(plan);
}

void host_calls(const char* field, std::uint32_t k, std::uint32_t r, std::uint64_t strip, std::uint64_t chunk,
                std::mt19937_64& rng) {
    pyrit_field f{};
    CHECK(pyrit_field_named(field, &f) == 0, "field %s", field);
    pyrit_code code{k, r, f, 0};
    const std::uint64_t sym = strip * f.w;
    char what[96];
    std::snprintf(what, sizeof what, "%s k%u r%u strip %llu chunk %llu", field, k, r, static_cast<unsigned long long>(strip),
                  static_cast<unsigned long long>(chunk));
    CHECK(pyrit_set_host_chunk(chunk) == 0, "%s set chunk", what);
    Heap all((k + r) * sym, &rng), want(r * sym), got(r * sym);
    reference_encode(code, all.p, want.p, sym);
    CHECK(pyrit_encode_host(&code, all.p, got.p, sym, 0) == 0, "%s encode_host", what);
    CHECK(std::memcmp(got.p, want.p, r * sym) == 0, "%s: encode_host parity differs from the interpreter", what);
    std::memset(got.p, 0, r * sym);
    CHECK(pyrit_encode_crs_host(&code, all.p, got.p, sym, 0) == 0, "%s encode_crs_host", what);
    CHECK(std::memcmp(got.p, want.p, r * sym) == 0, "%s: CRS parity differs", what);
    const int devs[3] = {0, 0, 0};
    std::memset(got.p, 0, r * sym);
    CHECK(pyrit_encode_host_devices(&code, all.p, got.p, sym, devs, 3) == 0, "%s encode_host_devices", what);
    CHECK(std::memcmp(got.p, want.p, r * sym) == 0, "%s: 3-shard parity differs", what);
    std::memcpy(all.p + k * sym, want.p, r * sym);
    // decode: random patterns, in place
    for (int t = 0; t < 3; ++t) {
        std::vector<std::uint32_t> idx(k + r);
        for (std::uint32_t i = 0; i < k + r; ++i) idx[i] = i;
        std::shuffle(idx.begin(), idx.end(), rng);
        const std::uint32_t e = 1 + static_cast<std::uint32_t>(rng() % r);
        Heap work((k + r) * sym);
        std::memcpy(work.p, all.p, (k + r) * sym);
        for (std::uint32_t i = 0; i < e; ++i) std::memset(work.p + idx[i] * sym, 0xEE, sym);
        int rc;
        if (t == 2)
            rc = pyrit_decode_host_devices(&code, work.p, idx.data(), e, sym, devs, 2);
        else
            rc = pyrit_decode_host(&code, work.p, idx.data(), e, sym, 0);
        CHECK(rc == 0, "%s decode_host -> %d", what, rc);
        CHECK(std::memcmp(work.p, all.p, (k + r) * sym) == 0, "%s: decode of %u erasures differs", what, e);
    }
    // apply_host on a window of every strip
    if (strip >= 64) {
        pyrit_plan* plan = nullptr;
        CHECK(pyrit_plan_encode(&code, &plan) == 0, "plan");
        std::vector<const std::uint8_t*> in(k);
        std::vector<std::uint8_t*> o1(r), o2(r);
        Heap a(r * sym), b(r * sym);
        for (std::uint32_t j = 0; j < k; ++j) in[j] = all.p + j * sym;
        for (std::uint32_t i = 0; i < r; ++i) o1[i] = a.p + i * sym, o2[i] = b.p + i * sym;
        const std::uint64_t off = 16, len = strip - 32;
        CHECK(pyrit_apply_host(plan, in.data(), o1.data(), strip, off, len, 0) == 0, "%s apply_host", what);
        CHECK(pyrit_plan_interpret(plan, in.data(), o2.data(), strip, off, len) == 0, "%s interpret window", what);
        CHECK(std::memcmp(a.p, b.p, r * sym) == 0, "%s: apply_host window differs", what);
        pyrit_plan_destroy(plan);
    }
    CHECK(pyrit_set_host_chunk(0) == 0, "reset chunk");
}

void device_batches(std::mt19937_64& rng) {
    pyrit_field f{};
    pyrit_field_named("gf256_r17", &f);
    pyrit_code code{10, 4, f, 0};
    const std::uint64_t strip = 4096, sym = strip * f.w, nb = 5, total = 14;
    Heap host(total * nb * sym, &rng), back(total * nb * sym);
    std::uint8_t* dev = nullptr;
    CHECK(cudaMalloc(&dev, total * nb * sym) == cudaSuccess, "cudaMalloc");
    CHECK(cudaMemcpy(dev, host.p, total * nb * sym, cudaMemcpyHostToDevice) == cudaSuccess, "H2D");
    std::vector<std::uint8_t*> symp(total);
    for (std::uint64_t i = 0; i < total; ++i) symp[i] = dev + i * nb * sym;
    std::vector<const std::uint8_t*> dp(symp.begin(), symp.begin() + 10);
    CHECK(pyrit_cu_encode_batch(&code, dp.data(), symp.data() + 10, sym, nb, sym, sym, nullptr) == 0, "encode_batch");
    CHECK(cudaMemcpy(back.p, dev, total * nb * sym, cudaMemcpyDeviceToHost) == cudaSuccess, "D2H");
    for (std::uint64_t b = 0; b < nb; ++b) {
        Heap data(10 * sym), want(4 * sym);
        for (std::uint32_t j = 0; j < 10; ++j) std::memcpy(data.p + j * sym, back.p + (j * nb + b) * sym, sym);
        reference_encode(code, data.p, want.p, sym);
        bool ok = true;
        for (std::uint32_t i = 0; i < 4; ++i) ok = ok && std::memcmp(want.p + i * sym, back.p + ((10 + i) * nb + b) * sym, sym) == 0;
        CHECK(ok, "encode_batch stripe %llu differs", static_cast<unsigned long long>(b));
    }
    // a never-seen erasure pattern: the runtime-matrix kernel path, in place on device
    const std::uint32_t erased[3] = {2, 7, 12};
    for (std::uint32_t e : erased) CHECK(cudaMemset(symp[e], 0x11, nb * sym) == cudaSuccess, "memset");
    CHECK(pyrit_cu_decode_batch(&code, symp.data(), erased, 3, sym, nb, sym, nullptr) == 0, "decode_batch");
    Heap after(total * nb * sym);
    CHECK(cudaMemcpy(after.p, dev, total * nb * sym, cudaMemcpyDeviceToHost) == cudaSuccess, "D2H");
    CHECK(std::memcmp(after.p, back.p, total * nb * sym) == 0, "decode_batch does not restore the stripes");
    char kernel[128];
    std::uint32_t blocks = 0, threads = 0;
    CHECK(pyrit_cu_last_launch(kernel, sizeof kernel, &blocks, &threads) == 0 && blocks > 0, "last launch");
    std::printf("  decode_batch ran %s (%u x %u)\n", kernel, blocks, threads);
    cudaFree(dev);
}

void file_codec(std::mt19937_64& rng) {
    char dir[] = "/tmp/pyrit_asan_XXXXXX";
    CHECK(mkdtemp(dir) != nullptr, "mkdtemp");
    const std::string input = std::string(dir) + "/input.bin", output = std::string(dir) + "/output.bin";
    const std::size_t bytes = 3 * 1000 * 1000 + 17; // not a multiple of anything
    Heap content(bytes, &rng);
    FILE* fp = std::fopen(input.c_str(), "wb");
    CHECK(fp && std::fwrite(content.p, 1, bytes, fp) == bytes, "write input");
    if (fp) std::fclose(fp);
    pyrit_field f{};
    pyrit_field_named("gf16", &f);
    pyrit_code code{4, 2, f, 0};
    CHECK(pyrit_set_file_chunk(1 << 20) == 0, "file chunk"); // several batches
    CHECK(pyrit_encode_file(&code, input.c_str(), dir, 4096, 0) == 0, "encode_file");
    std::vector<std::string> paths;
    for (std::uint32_t i : {0u, 2u, 4u, 5u}) { // shards 1 and 3 lost
        char buf[512];
        CHECK(pyrit_shard_path(input.c_str(), dir, i, buf, sizeof buf) == 0, "shard path");
        paths.emplace_back(buf);
    }
    std::vector<const char*> cp;
    for (auto& s : paths) cp.push_back(s.c_str());
    CHECK(pyrit_decode_file(cp.data(), 4, output.c_str(), 0) == 0, "decode_file");
    Heap got(bytes);
    fp = std::fopen(output.c_str(), "rb");
    CHECK(fp && std::fread(got.p, 1, bytes, fp) == bytes && std::fgetc(fp) == EOF, "read output");
    if (fp) std::fclose(fp);
    CHECK(std::memcmp(got.p, content.p, bytes) == 0, "decode_file output differs from the input");
    // too few shards, a truncated shard: typed errors, no crash
    CHECK(pyrit_decode_file(cp.data(), 3, output.c_str(), 0) != 0, "3 of 4 shards accepted");
    CHECK(truncate(paths[1].c_str(), 40) == 0, "truncate");
    CHECK(pyrit_decode_file(cp.data(), 4, output.c_str(), 0) != 0, "truncated shard accepted");
    CHECK(pyrit_set_file_chunk(0) == 0, "file chunk reset");
    const std::string rm = std::string("rm -rf ") + dir;
    if (std::system(rm.c_str()) != 0) std::fprintf(stderr, "could not remove %s\n", dir);
}

void concurrent_callers() {
    std::vector<std::thread> th;
    for (unsigned t = 0; t < 4; ++t)
        th.emplace_back([t] {
            std::mt19937_64 rng(500 + t);
            host_calls(t % 2 ? "gf1024" : "gf4096", 6 + t, 3, 2048 + 512 * t, 1024, rng);
        });
    for (auto& x : th) x.join();
}

} // namespace

int main() {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
        std::printf("host_sanitize_gpu: no CUDA device\n");
        return 77;
    }
    std::mt19937_64 rng(31337);
    // (field, k, r, strip bytes, pipeline chunk): one chunk, many chunks, strips that are not chunk multiples
    host_calls("gf16", 4, 2, 16, 0, rng);
    host_calls("gf16", 4, 2, 65536 + 48, 4096, rng);
    host_calls("gf64", 6, 3, 8192, 2048, rng);
    host_calls("gf256_r17", 10, 4, 100000 / 16 * 16, 16384, rng);
    host_calls("gf1024", 12, 4, 50000 / 16 * 16, 0, rng);
    host_calls("gf4096", 16, 4, 262144, 65536, rng);
    host_calls("gf4096", 5, 3, 24, 0, rng); // 8-byte aligned strips only: the cp.async / direct kernels
    device_batches(rng);
    file_codec(rng);
    concurrent_callers();
    CHECK(pyrit_jit_wait() == 0, "jit_wait");
    std::printf("host_sanitize_gpu: %lu checks, %d failed\n", g_checks.load(), g_fail.load());
    return g_fail.load() ? 1 : 0;
}
