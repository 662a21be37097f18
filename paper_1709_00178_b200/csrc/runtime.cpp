#include "runtime.hpp"

#include "kernels.hpp"

#include <cuda.h>
#include <dlfcn.h>
#include <nvrtc.h>
#include <unistd.h>

#include <filesystem>

#include <algorithm>
#include <atomic>
#include <bit>
#include <cstdio>
#include <cerrno>
#include <thread>
#include <sys/wait.h>
#include <spawn.h>
#include <sys/stat.h>
#include <chrono>
#include <future>
#include <cstring>
#include <cstdlib>
#include <fstream>
#include <iterator>
#include <memory>
#include <mutex>
#include <unordered_map>
#include <type_traits>
#include <vector>

extern char** environ;

namespace pyrit_b200 {

void check_cuda(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        throw CudaFailure(-static_cast<int>(e), std::string(what) + ": " + cudaGetErrorString(e));
}

namespace {

// Driver entry points, resolved through the runtime so the library loads
// on machines without a driver (the build container).
struct Driver {
    CUresult (*moduleLoadData)(CUmodule*, const void*) = nullptr;
    CUresult (*moduleGetFunction)(CUfunction*, CUmodule, const char*) = nullptr;
    CUresult (*launchKernel)(CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned,
                             CUstream, void**, void**) = nullptr;
    CUresult (*occupancy)(int*, CUfunction, int, size_t) = nullptr;
    CUresult (*getErrorString)(CUresult, const char**) = nullptr;
    CUresult (*funcSetAttribute)(CUfunction, CUfunction_attribute, int) = nullptr;
    CUresult (*launchKernelEx)(const CUlaunchConfig*, CUfunction, void**, void**) = nullptr;
    CUresult (*tensorMapEncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                     const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                     CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill) = nullptr;
};

template <class F>
void resolve(const char* sym, F& fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    check_cuda(cudaGetDriverEntryPoint(sym, &p, cudaEnableDefault, &q), sym);
    if (!p || q != cudaDriverEntryPointSuccess) throw CudaFailure(-1, std::string("driver symbol missing: ") + sym);
    fn = reinterpret_cast<F>(p);
}

const Driver& driver() {
    static std::once_flag once;
    static Driver d;
    std::call_once(once, [] {
        resolve("cuModuleLoadData", d.moduleLoadData);
        resolve("cuModuleGetFunction", d.moduleGetFunction);
        resolve("cuLaunchKernel", d.launchKernel);
        resolve("cuOccupancyMaxActiveBlocksPerMultiprocessor", d.occupancy);
        resolve("cuGetErrorString", d.getErrorString);
        resolve("cuFuncSetAttribute", d.funcSetAttribute);
        resolve("cuLaunchKernelEx", d.launchKernelEx);
        resolve("cuTensorMapEncodeTiled", d.tensorMapEncodeTiled);
    });
    return d;
}

void check_cu(CUresult r, const char* what) {
    if (r == CUDA_SUCCESS) return;
    const char* msg = "unknown";
    if (driver().getErrorString) driver().getErrorString(r, &msg);
    throw CudaFailure(-2000 - static_cast<int>(r), std::string(what) + ": " + msg);
}

struct LoadedKernel {
    CUfunction fn = nullptr;
    int blocks_per_sm = 1;
    int sms = 148;
};

std::mutex g_mu;
std::unordered_map<std::string, LoadedKernel> g_kernels; // name@device
std::unordered_map<std::string, CUmodule> g_modules;
std::atomic<std::uint64_t> g_jit{0}, g_launches{0};
// wall time of compiles (NVRTC in process, or the helper process), nanoseconds
std::atomic<std::uint64_t> g_jit_ns_last{0}, g_jit_ns_total{0};
void note_compile(std::chrono::steady_clock::time_point t0) {
    const auto ns = static_cast<std::uint64_t>(
        std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t0).count());
    g_jit_ns_last = ns;
    g_jit_ns_total += ns;
}
std::atomic<std::uint32_t> g_lanes{0};
std::string g_kernel_dir;

std::string default_kernel_dir() {
    Dl_info info{};
    if (dladdr(reinterpret_cast<void*>(&default_kernel_dir), &info) && info.dli_fname) {
        std::string so = info.dli_fname;
        const auto slash = so.rfind('/');
        return (slash == std::string::npos ? std::string(".") : so.substr(0, slash)) + "/kernels";
    }
    return "kernels";
}

std::vector<char> read_file(const std::string& path) {
    std::ifstream f(path, std::ios::binary);
    if (!f) return {};
    return std::vector<char>(std::istreambuf_iterator<char>(f), {});
}

// Kernels compiled by NVRTC are kept on disk so a program is compiled once
// per machine, not once per process (large codes take tens of seconds).
// The kernel name carries the generator version and a hash of the program
// and shape, so a cached cubin is never stale.  PYRIT_B200_JIT_CACHE = a
// directory, or "0" / "" to disable; default $XDG_CACHE_HOME/pyrit_b200 or
// ~/.cache/pyrit_b200.
std::string jit_cache_dir() {
    static const std::string& dir = *new std::string([] {
        if (const char* env = std::getenv("PYRIT_B200_JIT_CACHE"))
            return std::string(env) == "0" ? std::string() : std::string(env);
        if (const char* x = std::getenv("XDG_CACHE_HOME"); x && *x) return std::string(x) + "/pyrit_b200";
        if (const char* h = std::getenv("HOME"); h && *h) return std::string(h) + "/.cache/pyrit_b200";
        return std::string();
    }());
    return dir;
}

void write_cache(const std::string& dir, const std::string& name, const std::vector<char>& cubin) {
    std::error_code ec;
    std::filesystem::create_directories(dir, ec);
    if (ec) return; // the cache is an optimisation only
    const std::string tmp = dir + "/." + name + "." + std::to_string(::getpid()) + ".tmp";
    {
        std::ofstream f(tmp, std::ios::binary);
        if (!f) return;
        f.write(cubin.data(), static_cast<std::streamsize>(cubin.size()));
        if (!f) {
            std::filesystem::remove(tmp, ec);
            return;
        }
    }
    std::filesystem::rename(tmp, dir + "/" + name + ".cubin", ec); // atomic: readers never see a partial file
    if (ec) std::filesystem::remove(tmp, ec);
}

// NVRTC, loaded by path from the toolkit the library was built with.  A
// process resolves the soname libnvrtc.so.12 to whichever copy was loaded
// first -- in a torch process that is torch's bundled (older) NVRTC, whose
// code measured 4.5% slower on config 4 than the toolkit's
// (profiles/r01_s3/jit/).  Opening the toolkit's file explicitly
// (RTLD_LOCAL | RTLD_DEEPBIND) gives the same compiler as the prebuilt
// kernels in every process; PYRIT_B200_NVRTC names another file, and the
// plain soname is the fallback.
struct Nvrtc {
    void* handle = nullptr;
    std::string path;
    nvrtcResult (*create)(nvrtcProgram*, const char*, const char*, int, const char* const*, const char* const*) = nullptr;
    nvrtcResult (*compile)(nvrtcProgram, int, const char* const*) = nullptr;
    nvrtcResult (*log_size)(nvrtcProgram, size_t*) = nullptr;
    nvrtcResult (*log)(nvrtcProgram, char*) = nullptr;
    nvrtcResult (*cubin_size)(nvrtcProgram, size_t*) = nullptr;
    nvrtcResult (*cubin)(nvrtcProgram, char*) = nullptr;
    nvrtcResult (*destroy)(nvrtcProgram*) = nullptr;
    const char* (*error)(nvrtcResult) = nullptr;
    nvrtcResult (*version)(int*, int*) = nullptr;
};

#ifndef PYRIT_NVRTC_PATH
#define PYRIT_NVRTC_PATH "libnvrtc.so.12"
#endif

const Nvrtc& nvrtc() {
    static std::once_flag once;
    static Nvrtc& n = *new Nvrtc; // never destroyed (background compiles may outlive exit)
    std::call_once(once, [] {
        std::vector<std::string> tries;
        if (const char* e = std::getenv("PYRIT_B200_NVRTC"); e && *e) tries.emplace_back(e);
        tries.emplace_back(PYRIT_NVRTC_PATH);
        tries.emplace_back("libnvrtc.so.12");
#if defined(__SANITIZE_ADDRESS__) || defined(__SANITIZE_THREAD__)
        const int deepbind = 0; // the sanitizer runtimes refuse RTLD_DEEPBIND (tests/test_host_sanitizers.py)
#else
        const int deepbind = RTLD_DEEPBIND;
#endif
        for (const std::string& t : tries) {
            n.handle = dlopen(t.c_str(), RTLD_NOW | RTLD_LOCAL | deepbind);
            if (n.handle) {
                n.path = t;
                break;
            }
        }
        if (!n.handle) return;
        auto sym = [&](const char* name, auto& fn) { fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(n.handle, name)); };
        sym("nvrtcCreateProgram", n.create);
        sym("nvrtcCompileProgram", n.compile);
        sym("nvrtcGetProgramLogSize", n.log_size);
        sym("nvrtcGetProgramLog", n.log);
        sym("nvrtcGetCUBINSize", n.cubin_size);
        sym("nvrtcGetCUBIN", n.cubin);
        sym("nvrtcDestroyProgram", n.destroy);
        sym("nvrtcGetErrorString", n.error);
        sym("nvrtcVersion", n.version);
    });
    if (!n.handle || !n.create || !n.compile || !n.cubin || !n.cubin_size || !n.destroy || !n.error)
        throw CudaFailure(-1000, "NVRTC (libnvrtc.so.12) could not be loaded: kernels that are not prebuilt cannot be "
                                 "compiled");
    return n;
}

// file the NVRTC in use was loaded from (the helper loads the same one)
std::string nvrtc_path() { return nvrtc().path; }

// "nvrtc12.9": the compiler version in cache file names
std::string nvrtc_tag() {
    static const std::string& tag = *new std::string([] {
        const Nvrtc& n = nvrtc();
        int major = 0, minor = 0;
        if (n.version) n.version(&major, &minor);
        return "nvrtc" + std::to_string(major) + "." + std::to_string(minor);
    }());
    return tag;
}

std::vector<char> nvrtc_compile(const std::string& src, const std::string& name) {
    const auto t0 = std::chrono::steady_clock::now();
    const Nvrtc& rt = nvrtc();
    nvrtcProgram prog;
    auto chk = [&](nvrtcResult r, const char* what) {
        if (r != NVRTC_SUCCESS)
            throw CudaFailure(-1000 - static_cast<int>(r), std::string(what) + ": " + rt.error(r));
    };
    chk(rt.create(&prog, src.c_str(), (name + ".cu").c_str(), 0, nullptr, nullptr), "nvrtcCreateProgram");
    const char* opts[] = {"--gpu-architecture=sm_100a", "--std=c++17", "-lineinfo", "-DNDEBUG"};
    const nvrtcResult rc = rt.compile(prog, 4, opts);
    if (rc != NVRTC_SUCCESS) {
        size_t n = 0;
        rt.log_size(prog, &n);
        std::string log(n, '\0');
        rt.log(prog, log.data());
        rt.destroy(&prog);
        throw CudaFailure(-1000 - static_cast<int>(rc), "NVRTC failed for " + name + ":\n" + log);
    }
    size_t n = 0;
    chk(rt.cubin_size(prog, &n), "nvrtcGetCUBINSize");
    std::vector<char> cubin(n);
    chk(rt.cubin(prog, cubin.data()), "nvrtcGetCUBIN");
    rt.destroy(&prog);
    ++g_jit;
    note_compile(t0);
    return cubin;
}

// Tiered compilation: a kernel that is neither loaded, prebuilt nor in the
// disk cache is compiled in the background while the generic bit-matrix
// kernel (kernels.cu) serves the launches; load_kernel picks the result up.
// (heap objects that are never destroyed, so the exit-time waiter below can
// still use them whatever the destruction order)
std::mutex& g_async_mu = *new std::mutex;
std::unordered_map<std::string, std::shared_future<std::vector<char>>>& g_async =
    *new std::unordered_map<std::string, std::shared_future<std::vector<char>>>;

std::string cache_name(const std::string& name) { return name + "." + nvrtc_tag(); }

bool file_exists(const std::string& path) {
    struct stat sb {};
    return ::stat(path.c_str(), &sb) == 0;
}

// true when load_kernel would not have to compile (or wait for) this kernel
bool kernel_ready(const std::string& name, int device) {
    {
        std::lock_guard<std::mutex> lk(g_mu);
        if (g_kernels.count(name + "@" + std::to_string(device))) return true;
    }
    if (file_exists(kernel_dir() + "/" + name + ".cubin")) return true;
    const std::string cache = jit_cache_dir();
    if (!cache.empty() && file_exists(cache + "/" + cache_name(name) + ".cubin")) return true;
    std::lock_guard<std::mutex> lk(g_async_mu);
    auto it = g_async.find(name);
    return it != g_async.end() && it->second.wait_for(std::chrono::seconds(0)) == std::future_status::ready;
}

// The helper executable next to the library (pyrit_jit_helper, jit_helper.cpp):
// background compiles run NVRTC in their own process, so the library's
// process may exit at any moment (an in-process NVRTC compile still running
// at exit() crashed: its statics were being destroyed under it).
std::string helper_path() {
    static const std::string& path = *new std::string([] {
        Dl_info info{};
        if (dladdr(reinterpret_cast<void*>(&helper_path), &info) && info.dli_fname) {
            std::string so = info.dli_fname;
            const auto slash = so.rfind('/');
            return (slash == std::string::npos ? std::string(".") : so.substr(0, slash)) + "/pyrit_jit_helper";
        }
        return std::string("pyrit_jit_helper");
    }());
    return path;
}

// compile `src` in a helper process into `out` (blocking; runs on a background thread)
std::vector<char> helper_compile(const std::string& src, const std::string& name, const std::string& out,
                                 const std::string& lib) {
    const auto t0 = std::chrono::steady_clock::now();
    const std::string base = out + ".src" + std::to_string(::getpid()) + "_" +
                             std::to_string(std::hash<std::thread::id>{}(std::this_thread::get_id()));
    {
        std::ofstream f(base, std::ios::binary);
        f.write(src.data(), static_cast<std::streamsize>(src.size()));
        if (!f) throw CudaFailure(-1000, "cannot write " + base);
    }
    const std::string helper = helper_path();
    std::vector<char*> argv = {const_cast<char*>(helper.c_str()), const_cast<char*>(base.c_str()),
                               const_cast<char*>(name.c_str()), const_cast<char*>(out.c_str()),
                               const_cast<char*>(lib.c_str()), nullptr};
    pid_t pid = 0;
    const int rc = posix_spawn(&pid, helper.c_str(), nullptr, nullptr, argv.data(), environ);
    int status = 0;
    if (rc == 0)
        while (::waitpid(pid, &status, 0) < 0 && errno == EINTR) {
        }
    std::remove(base.c_str());
    if (rc != 0 || !WIFEXITED(status) || WEXITSTATUS(status) != 0)
        throw CudaFailure(-1000, "background compile of " + name + " failed");
    std::vector<char> cubin = read_file(out);
    if (cubin.empty()) throw CudaFailure(-1000, "background compile of " + name + " produced nothing");
    ++g_jit;
    note_compile(t0);
    return cubin;
}

// false when no helper is available (the caller then compiles synchronously)
bool start_async_compile(const Program& p, const KernelShape& ks, const std::string& name) {
    static const bool have_helper = ::access(helper_path().c_str(), X_OK) == 0;
    if (!have_helper) return false;
    std::lock_guard<std::mutex> lk(g_async_mu);
    if (g_async.count(name)) return true;
    std::string src = generate_cuda(p, ks); // the program need not outlive this call
    std::string cache = jit_cache_dir();
    std::string out;
    if (!cache.empty()) {
        std::error_code ec;
        std::filesystem::create_directories(cache, ec);
        if (ec || ::access(cache.c_str(), W_OK) != 0) cache.clear(); // unwritable cache: compile into /tmp
    }
    if (!cache.empty()) {
        out = cache + "/" + cache_name(name) + ".cubin";
    } else {
        std::error_code ec;
        const auto tmp = std::filesystem::temp_directory_path(ec);
        out = ((ec ? std::filesystem::path("/tmp") : tmp) / (name + "." + std::to_string(::getpid()) + ".cubin")).string();
    }
    g_async[name] = std::async(std::launch::async, [src = std::move(src), name, out, keep = !cache.empty(),
                                                    lib = nvrtc_path()] {
                        std::vector<char> cubin = helper_compile(src, name, out, lib);
                        if (!keep) std::remove(out.c_str());
                        return cubin;
                    }).share();
    return true;
}

LoadedKernel load_kernel(const Program& p, const KernelShape& ks, int device) {
    const std::string name = kernel_name(p, ks);
    const std::string key = name + "@" + std::to_string(device);
    {
        std::lock_guard<std::mutex> lk(g_mu);
        auto it = g_kernels.find(key);
        if (it != g_kernels.end()) return it->second;
    }
    // prebuilt (next to the library), else the on-disk JIT cache, else NVRTC
    std::vector<char> cubin = read_file(kernel_dir() + "/" + name + ".cubin");
    const std::string cache = jit_cache_dir();
    // cached cubins are keyed by the compiler too: one from another NVRTC is not reused
    const std::string cname = cache.empty() || !cubin.empty() ? std::string() : name + "." + nvrtc_tag();
    if (cubin.empty() && !cache.empty()) cubin = read_file(cache + "/" + cname + ".cubin");
    if (cubin.empty()) { // a background compile of it, else compile now
        std::shared_future<std::vector<char>> pending;
        {
            std::lock_guard<std::mutex> lk(g_async_mu);
            auto it = g_async.find(name);
            if (it != g_async.end()) pending = it->second;
        }
        bool compiled = false;
        if (pending.valid()) {
            try {
                cubin = pending.get();
                compiled = true;
            } catch (const std::exception&) {
                // the background compile failed (e.g. an unwritable cache): forget
                // it and compile here, in process, with a best-effort cache write
                std::lock_guard<std::mutex> lk(g_async_mu);
                g_async.erase(name);
            }
        }
        if (!compiled) {
            cubin = nvrtc_compile(generate_cuda(p, ks), name);
            if (!cache.empty()) write_cache(cache, cname, cubin);
        }
    }
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_kernels.find(key);
    if (it != g_kernels.end()) return it->second;
    check_cuda(cudaSetDevice(device), "cudaSetDevice");
    CUmodule mod = nullptr;
    check_cu(driver().moduleLoadData(&mod, cubin.data()), "cuModuleLoadData");
    LoadedKernel k;
    check_cu(driver().moduleGetFunction(&k.fn, mod, name.c_str()), "cuModuleGetFunction");
    if (ks.smem_bytes > 48 * 1024)
        check_cu(driver().funcSetAttribute(k.fn, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES,
                                           static_cast<int>(ks.smem_bytes)),
                 "cuFuncSetAttribute(max dynamic smem)");
    check_cu(driver().occupancy(&k.blocks_per_sm, k.fn, static_cast<int>(ks.threads), ks.smem_bytes), "occupancy");
    if (k.blocks_per_sm < 1) k.blocks_per_sm = 1;
    check_cuda(cudaDeviceGetAttribute(&k.sms, cudaDevAttrMultiProcessorCount, device), "sm count");
    g_modules[key] = mod;
    g_kernels[key] = k;
    return k;
}

bool aligned(const void* p, std::uint64_t v) { return reinterpret_cast<std::uintptr_t>(p) % v == 0; }

// SM count of the current device (cached per device)
int sm_count() {
    static std::atomic<int> cache[64];
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
    int n = cache[dev].load();
    if (n == 0) {
        if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
        cache[dev] = n;
    }
    return n;
}

} // namespace

std::uint32_t preferred_lanes() {
    std::uint32_t l = g_lanes.load();
    if (l == 0) {
        const char* env = std::getenv("PYRIT_B200_LANES");
        l = env ? static_cast<std::uint32_t>(std::atoi(env)) : 1;
        if (l != 1 && l != 2 && l != 4) l = 1;
        g_lanes = l;
    }
    return l;
}

void set_preferred_lanes(std::uint32_t lanes) {
    if (lanes != 1 && lanes != 2 && lanes != 4) raise(Errc::InvalidArgument, "lanes must be 1, 2 or 4");
    g_lanes = lanes;
}

void set_kernel_dir(const std::string& dir) {
    std::lock_guard<std::mutex> lk(g_mu);
    g_kernel_dir = dir;
}

std::string kernel_dir() {
    // first use may come from several host threads at once (run_host_devices)
    std::lock_guard<std::mutex> lk(g_mu);
    if (g_kernel_dir.empty()) {
        const char* env = std::getenv("PYRIT_B200_KERNEL_DIR");
        g_kernel_dir = env ? env : default_kernel_dir();
    }
    return g_kernel_dir;
}

bool prebuilt_plan(const std::string& key) {
    static std::once_flag once;
    static std::unordered_map<std::string, int>& keys = *new std::unordered_map<std::string, int>;
    std::call_once(once, [] {
        // kernels/prebuilt.tsv (build.py): plan keys of the programs whose
        // specialised kernels ship prebuilt
        std::ifstream f(kernel_dir() + "/prebuilt.tsv");
        std::string k;
        while (f >> k) keys[k] = 1;
    });
    return keys.count(key) != 0;
}

void jit_wait() {
    std::vector<std::shared_future<std::vector<char>>> pending;
    {
        std::lock_guard<std::mutex> lk(g_async_mu);
        for (auto& kv : g_async) pending.push_back(kv.second);
    }
    for (auto& f : pending) f.get(); // rethrows a failed compile
}

std::string jit_info() {
    const Nvrtc& n = nvrtc();
    int major = 0, minor = 0;
    if (n.version) n.version(&major, &minor);
    return "nvrtc " + std::to_string(major) + "." + std::to_string(minor) + " (" + n.path + ")";
}

std::uint64_t jit_compiles() { return g_jit.load(); }
void jit_time(double* last_ms, double* total_ms) {
    if (last_ms) *last_ms = static_cast<double>(g_jit_ns_last.load()) * 1e-6;
    if (total_ms) *total_ms = static_cast<double>(g_jit_ns_total.load()) * 1e-6;
}
std::uint64_t kernel_launches() { return g_launches.load(); }

KernelShape direct_shape(const Program& p, std::uint32_t lanes) {
    KernelShape ks = shape_for(lanes);
    const std::uint32_t R = static_cast<std::uint32_t>(p.parts.size());
    if (R > 1 && ks.threads % R == 0 && ks.threads / R >= 32) {
        ks.split = R;
        // two CTAs per SM (128 registers) while a part's accumulators are few
        const std::uint32_t acc_rows =
            p.kind == TransformKind::Embedding && !p.crs ? p.field.n : p.field.w;
        std::uint32_t acc = 0;
        for (const Program& q : p.parts) acc = std::max(acc, q.rows * acc_rows);
        ks.min_blocks = acc <= 64 ? 2 : 1;
    }
    return ks;
}

KernelShape shape_for(std::uint32_t lanes) {
    KernelShape ks;
    ks.lanes = lanes;
    ks.threads = 256;
    // one block per SM guaranteed: lets ptxas keep the larger ring programs
    // (up to ~240 live words) spill-free; occupancy follows actual usage
    ks.min_blocks = 1;
    return ks;
}

namespace {

std::atomic<int> g_mode{-1};
thread_local LaunchInfo g_last;

int env_int(const char* name, int dflt) {
    const char* v = std::getenv(name);
    return v ? std::atoi(v) : dflt;
}

// staged shape for p (PYRIT_B200_COPY=0 selects the TMA bulk-copy producer)
KernelShape staged_for(const Program& p) {
    KernelShape ks = staged_shape(p, 227 * 1024);
    const int copy = env_int("PYRIT_B200_COPY", static_cast<int>(ks.copy));
    ks.copy = copy == 2 ? 2u : copy ? 1u : 0u;
    ks.ws = env_int("PYRIT_B200_WS", static_cast<int>(ks.ws)) ? 1u : 0u;
    ks.spb = static_cast<std::uint32_t>(env_int("PYRIT_B200_TMA_SPB", static_cast<int>(ks.spb)));
    if (ks.spb && p.field.w % ks.spb) ks.spb = 0;
    return ks;
}

} // namespace

int kernel_mode() {
    int m = g_mode.load();
    if (m < 0) {
        m = env_int("PYRIT_B200_MODE", 0);
        if (m < 0 || m > 4) m = 0;
        g_mode = m;
    }
    return m;
}

void set_kernel_mode(int mode) {
    if (mode < 0 || mode > 4)
        raise(Errc::InvalidArgument,
              "mode must be 0 (auto), 1 (direct), 2 (staged), 3 (generic) or 4 (runtime-matrix ring kernel)");
    g_mode = mode;
}

int rt_policy() {
    static const int v = [] {
        const int x = env_int("PYRIT_B200_RT", 1);
        return x < 0 || x > 2 ? 1 : x;
    }();
    return v;
}

KernelShape choose_shape(const Program& p, const std::uint8_t* const* in, std::uint8_t* const* out,
                         std::uint64_t strip, std::uint64_t off, std::uint64_t len, std::uint64_t nb,
                         std::uint64_t in_pitch, std::uint64_t out_pitch) {
    const auto all_aligned = [&](std::uint64_t v) {
        bool ok = strip % v == 0 && off % v == 0 && len % v == 0;
        if (nb > 1) ok = ok && in_pitch % v == 0 && out_pitch % v == 0;
        for (std::uint32_t j = 0; ok && j < p.cols; ++j) ok = aligned(in[j], v);
        for (std::uint32_t i = 0; ok && i < p.rows; ++i) ok = aligned(out[i], v);
        return ok;
    };
    // staged kernel: cp.async chunks of the widest alignment every pointer,
    // pitch and the window share (the TMA producer needs 16)
    const std::uint32_t chunk = all_aligned(16) ? 16 : all_aligned(8) ? 8 : all_aligned(4) ? 4 : 0;
    if (kernel_mode() != 1 && chunk) {
        KernelShape ks = staged_for(p);
        ks.chunk = chunk;
        if (ks.copy != 1 && chunk != 16) ks.copy = 1; // TMA needs 16-byte alignment: cp.async chunks
        if (ks.copy != 2) ks.ws = 0;
        // PYRIT_B200_TMAP4=1: inputs at a constant 16-byte-multiple spacing get one
        // 4D tensor map and one box per unit -- measured slower than a box per
        // fragment (cfg2 0.894 vs 0.956, cfg3 0.926 vs 1.032), so off by default
        if (ks.copy == 2 && p.cols > 1 && env_int("PYRIT_B200_TMAP4", 0)) {
            const std::int64_t d = reinterpret_cast<std::intptr_t>(in[1]) - reinterpret_cast<std::intptr_t>(in[0]);
            bool uni = d > 0 && d % 16 == 0;
            for (std::uint32_t j = 2; uni && j < p.cols; ++j)
                uni = reinterpret_cast<std::intptr_t>(in[j]) - reinterpret_cast<std::intptr_t>(in[j - 1]) == d;
            ks.tmap4 = uni ? 1u : 0u;
        }
        // auto mode keeps the staged kernel where it measured faster than the
        // direct one (profiles/r01_s2/sizes_*): 16-byte chunks, at most two
        // output parts, and per-stripe windows that fill at least half a tile
        const std::uint64_t tiles = ks.staged ? (len + ks.tile - 1) / ks.tile : 0;
        const bool dense = tiles && 2 * len >= tiles * ks.tile;
        const bool fits = tiles * nb < (std::uint64_t(1) << 32);
        // ... and enough tiles for its pipeline to pay for the ring setup (small
        // launches -- config 1's 6 MiB -- run faster on the direct kernel)
        const bool big = tiles * nb >= 2ull * static_cast<std::uint64_t>(sm_count());
        const bool suited = dense && big && chunk == 16 && p.parts.size() <= 2;
        if (ks.staged && fits && (suited || kernel_mode() == 2)) return ks;
    }
    // direct mode: widest vector the alignment of every pointer, the strip
    // pitch and the window allows; byte mode otherwise.  Programs compiled
    // with several output parts (large codes) split their rows over thread
    // groups instead of holding every accumulator in one thread.
    std::uint32_t lanes = 0;
    for (std::uint32_t l = preferred_lanes(); l >= 1; l /= 2)
        if (all_aligned(4ull * l)) {
            lanes = l;
            break;
        }
    KernelShape ks = direct_shape(p, lanes);
    if (lanes == 0 && all_aligned(2)) ks.half = 1; // e.g. GF(2^12) symbols of 24k bytes: 2-byte strips
    return ks;
}

namespace {

// PYRIT_B200_TIERED=0 compiles every new kernel before its first launch
bool tiered() {
    static const bool on = env_int("PYRIT_B200_TIERED", 1) != 0;
    return on;
}

bool generic_ok(const Program& p, const std::uint8_t* const* in, std::uint8_t* const* out, std::uint64_t strip,
                std::uint64_t off, std::uint64_t len, std::uint64_t nb, std::uint64_t in_pitch,
                std::uint64_t out_pitch) {
    if (p.field_masks.empty() || p.rows == 0 || p.cols + p.rows > kGenericMaxPtrs ||
        p.field_masks.size() > kGenericMaxMasks)
        return false;
    bool ok = strip % 4 == 0 && off % 4 == 0 && len % 4 == 0 && (nb <= 1 || (in_pitch % 4 == 0 && out_pitch % 4 == 0));
    for (std::uint32_t j = 0; ok && j < p.cols; ++j) ok = aligned(in[j], 4);
    for (std::uint32_t i = 0; ok && i < p.rows; ++i) ok = aligned(out[i], 4);
    return ok;
}

LaunchInfo launch_generic_program(const Program& p, const std::uint8_t* const* in, std::uint8_t* const* out,
                                  std::uint64_t strip, std::uint64_t off, std::uint64_t len, std::uint64_t nb,
                                  std::uint64_t in_pitch, std::uint64_t out_pitch, cudaStream_t stream) {
    thread_local GenericArgs a; // ~27 KB of kernel parameters
    const std::uint64_t nwords = len / 4;
    a.S = strip;
    a.off = off;
    a.nwords = nwords;
    a.nb = nb;
    a.ibp = nb > 1 ? in_pitch : 0;
    a.obp = nb > 1 ? out_pitch : 0;
    a.k = p.cols;
    a.e = p.rows;
    a.w = p.field.w;
    for (std::uint32_t j = 0; j < p.cols; ++j) a.ptr[j] = in[j];
    for (std::uint32_t i = 0; i < p.rows; ++i) a.ptr[p.cols + i] = out[i];
    std::copy(p.field_masks.begin(), p.field_masks.end(), a.mask);
    const std::uint64_t want = (nwords * nb + 255) / 256;
    const unsigned blocks = static_cast<unsigned>(std::max<std::uint64_t>(1, std::min<std::uint64_t>(want, 8ull * sm_count())));
    const std::uint64_t stride = std::uint64_t(blocks) * 256;
    a.sq = stride / nwords;
    a.sr = stride % nwords;
    check_cuda(launch_generic(a, blocks, stream), "generic kernel launch");
    ++g_launches;
    LaunchInfo info;
    info.kernel = "pyrit_generic_bitmatrix";
    info.blocks = blocks;
    info.threads = 256;
    info.lanes = 1;
    g_last = info;
    return info;
}

// ---- runtime-matrix ring kernel (ring_rt.cu) ------------------------------

bool overlaps(const std::uint8_t* a, std::uint64_t alen, const std::uint8_t* b, std::uint64_t blen) {
    const auto x = reinterpret_cast<std::uintptr_t>(a), y = reinterpret_cast<std::uintptr_t>(b);
    return x < y + blen && y < x + alen;
}

// Does any output span overlap any input span at all?
bool any_alias(const Program& p, const std::uint8_t* const* in, std::uint8_t* const* out, std::uint64_t strip,
               std::uint64_t nb, std::uint64_t in_pitch, std::uint64_t out_pitch) {
    const std::uint64_t w = p.field.w;
    const std::uint64_t ispan = (nb - 1) * in_pitch + w * strip, ospan = (nb - 1) * out_pitch + w * strip;
    for (std::uint32_t i = 0; i < p.rows; ++i)
        for (std::uint32_t j = 0; j < p.cols; ++j)
            if (overlaps(out[i], ospan, in[j], ispan)) return true;
    return false;
}

// Does any output span overlap an input span where a column of one is not the
// same column of the other?  Kernels that read every input of a tile before
// storing its outputs (ring_rt, staged, unsplit direct) are exact when outputs
// alias inputs column for column (decode() in place, slot aliasing of replay);
// anything else must not run them concurrently with a read of the same bytes.
bool unsafe_alias(const Program& p, const std::uint8_t* const* in, std::uint8_t* const* out, std::uint64_t strip,
                  std::uint64_t nb, std::uint64_t in_pitch, std::uint64_t out_pitch) {
    const std::uint64_t w = p.field.w;
    const std::uint64_t ispan = (nb - 1) * in_pitch + w * strip, ospan = (nb - 1) * out_pitch + w * strip;
    for (std::uint32_t i = 0; i < p.rows; ++i)
        for (std::uint32_t j = 0; j < p.cols; ++j) {
            if (!overlaps(out[i], ospan, in[j], ispan)) continue;
            const std::int64_t d = reinterpret_cast<std::intptr_t>(out[i]) - reinterpret_cast<std::intptr_t>(in[j]);
            if (nb > 1 && (in_pitch != out_pitch || d != 0)) return true;
            if (d % static_cast<std::int64_t>(strip) != 0) return true;
        }
    return false;
}

} // namespace

bool ring_rt_eligible(const Program& p, const std::uint8_t* const* in, std::uint8_t* const* out, std::uint64_t strip,
                      std::uint64_t off, std::uint64_t len, std::uint64_t nb, std::uint64_t in_pitch,
                      std::uint64_t out_pitch) {
    if (p.crs || p.sched || p.reps.empty() || p.rows == 0 || p.cols > kRtMaxK) return false;
    if (!rt_supported(p.field.w, p.field.n, p.field.modulus)) return false;
    if (p.kind == TransformKind::Parity && p.field.n - p.field.w > 256 / p.field.w) return false;
    bool ok = strip % 16 == 0 && off % 16 == 0 && len % 16 == 0 && (nb <= 1 || (in_pitch % 16 == 0 && out_pitch % 16 == 0));
    for (std::uint32_t j = 0; ok && j < p.cols; ++j) ok = aligned(in[j], 16);
    for (std::uint32_t i = 0; ok && i < p.rows; ++i) ok = aligned(out[i], 16);
    if (!ok) return false;
    if ((len + kRtTile - 1) / kRtTile * nb * kRtMaxGroups >= (std::uint64_t(1) << 31)) return false;
    return !unsafe_alias(p, in, out, strip, nb, in_pitch, out_pitch);
}

namespace {

// The launches of one runtime-matrix call, kept per thread: a call with the same
// program (plan key), buffers and window as the previous one reuses its kernel
// parameters (tensor maps, op lists) and only launches.
struct RtCall {
    std::string key;
    int dev = -1;
    std::vector<const std::uint8_t*> in;
    std::vector<std::uint8_t*> out;
    std::uint64_t strip = 0, off = 0, len = 0, nb = 0, ip = 0, op = 0;
    std::vector<std::unique_ptr<RtArgs>> args; // ~24 KB of kernel parameters each
    std::vector<RtLaunch> launches;
    // per launch: the program rows of every (group, part) bin and the CTAs an SM holds --
    // what bind_ring_rt needs to point a planned launch at other buffers
    std::vector<std::vector<std::vector<std::uint32_t>>> bins;
    std::vector<std::uint32_t> ctas_per_sm;
    std::vector<std::uint32_t> case_bytes, op_count; // per launch: bytes of case code named, ops (without sentinels)
    LaunchInfo info;
};

// The buffer-dependent kernel parameters: tensor maps of the inputs and the window.
void bind_rt_geometry(RtArgs& a, const Program& p, const std::uint8_t* const* in, std::uint64_t strip, std::uint64_t off,
                      std::uint64_t len, std::uint64_t nb, std::uint64_t in_pitch, std::uint64_t out_pitch, bool device) {
    const std::uint32_t w = p.field.w, k = p.cols;
    const std::uint32_t elem = 8;
    const std::uint64_t tpb = (len + kRtTile - 1) / kRtTile;
    static const int promo_knob = env_int("PYRIT_B200_TMA_PROMO", 3);
    const CUtensorMapL2promotion promo = static_cast<CUtensorMapL2promotion>(std::min(3, std::max(0, promo_knob)));
    for (std::uint32_t j = 0; device && j < k; ++j) {
        CUtensorMap m;
        const cuuint64_t dims[3] = {strip / elem, w, nb};
        const cuuint64_t strides[2] = {strip, nb > 1 ? in_pitch : strip * w};
        const cuuint32_t box[3] = {kRtBox, w, 1};
        const cuuint32_t es[3] = {1, 1, 1};
        check_cu(driver().tensorMapEncodeTiled(&m, CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, const_cast<std::uint8_t*>(in[j]),
                                               dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                               CU_TENSOR_MAP_SWIZZLE_NONE, promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE),
                 "cuTensorMapEncodeTiled(ring_rt)");
        std::memcpy(a.tm[j], &m, sizeof m);
    }
    a.S = strip;
    a.off = off;
    a.len = len;
    a.nb = nb;
    a.obp = nb > 1 ? out_pitch : 0;
    a.k = k;
    a.tpb = static_cast<std::uint32_t>(tpb);
    a.ntiles = static_cast<std::uint32_t>(tpb * nb);
}

unsigned rt_blocks(std::uint64_t units, std::uint32_t ctas_per_sm, bool device) {
    return !device ? 1u
                   : static_cast<unsigned>(std::max<std::uint64_t>(
                         1, std::min<std::uint64_t>(units, std::uint64_t(ctas_per_sm) * sm_count())));
}

// A planned call (op lists, parts, groups: functions of the matrix only) pointed at
// other buffers or another window: new tensor maps, output bases and grid sizes.
void bind_ring_rt(RtCall& call, const Program& p, const std::uint8_t* const* in, std::uint8_t* const* out,
                  std::uint64_t strip, std::uint64_t off, std::uint64_t len, std::uint64_t nb, std::uint64_t in_pitch,
                  std::uint64_t out_pitch) {
    for (std::size_t c = 0; c < call.launches.size(); ++c) {
        RtArgs& a = *call.args[c];
        RtLaunch& l = call.launches[c];
        if (c == 0)
            bind_rt_geometry(a, p, in, strip, off, len, nb, in_pitch, out_pitch, true);
        else {
            const RtArgs& a0 = *call.args[0];
            std::memcpy(a.tm, a0.tm, sizeof a.tm);
            a.S = a0.S, a.off = a0.off, a.len = a0.len, a.nb = a0.nb, a.obp = a0.obp, a.k = a0.k, a.tpb = a0.tpb,
            a.ntiles = a0.ntiles;
        }
        const auto& bins = call.bins[c];
        for (std::size_t q = 0; q < bins.size(); ++q)
            for (std::size_t i = 0; i < bins[q].size(); ++i)
                a.out[q / l.R][(q % l.R) * kRtPartE + i] = out[bins[q][i]];
        l.blocks = rt_blocks(std::uint64_t(a.ntiles) * a.ngrp, call.ctas_per_sm[c], true);
        call.info.blocks = l.blocks;
    }
}

// One matrix entry of a part: the representative (set bits = shifts) of local output
// i, and the ops chosen for it: singles (sh, 0) and pairs (sh, d) standing for the
// shifts sh and (sh + d) mod n.
struct RtEntry {
    std::uint32_t i, mask;
    std::vector<std::pair<std::uint32_t, std::uint32_t>> ops;
};

// Choose the pair cases of a launch.  A case (i, sh, d) serves every entry of local
// output i whose representative has both shifts still unpaired; taking it removes,
// per use, the rows both shifts reach (one 3-input LOP3 instead of two XORs) and one
// dispatch.  Greedy: the case with the largest total saving first, applied wherever it
// fits, until the distinct cases named (pairs chosen + singles still needed) would
// outgrow `budget` bytes of case code.  Returns the bytes of cases named.
template <class Rows>
std::uint32_t rt_select_pairs(std::vector<RtEntry>& entries, std::uint32_t n, std::uint32_t D, std::uint32_t E,
                              std::uint32_t V, std::uint32_t budget, Rows case_rows) {
    constexpr std::uint32_t kDispatch = 6; // instructions of a case besides its LOP3s
    auto bytes_of = [&](std::uint32_t sh, std::uint32_t ds) { return 16u * (case_rows(sh, ds) * V + kDispatch); };
    static const std::uint32_t min_uses = static_cast<std::uint32_t>(std::max(1, env_int("PYRIT_B200_RT_PAIR_MINUSE", 1)));
    std::vector<std::uint32_t> rem(entries.size());
    // need[i*n + sh]: entries of local output i whose shift sh is still unpaired (a single
    // case (i, sh) is named while it is > 0); singles: bytes of those cases
    std::vector<std::uint32_t> need(std::size_t(E) * n, 0), single_bytes(n);
    for (std::uint32_t sh = 0; sh < n; ++sh) single_bytes[sh] = bytes_of(sh, 0);
    std::uint32_t singles = 0;
    for (std::size_t x = 0; x < entries.size(); ++x) {
        rem[x] = entries[x].mask;
        entries[x].ops.clear();
        for (std::uint32_t m = rem[x]; m; m &= m - 1) {
            const std::uint32_t sh = static_cast<std::uint32_t>(std::countr_zero(m));
            if (need[entries[x].i * n + sh]++ == 0) singles += single_bytes[sh];
        }
    }
    std::uint32_t pair_bytes = 0;
    if (D > 0) {
        // per-use saving of a pair at distance d (independent of sh for the Embedding; the
        // Parity transform truncates rows, so take sh = 0 as the estimate)
        std::vector<std::uint32_t> saving(D + 1, 0);
        for (std::uint32_t d = 1; d <= D; ++d) {
            const std::uint32_t two = case_rows(0, 0) + case_rows(d % n, 0), one = case_rows(0, d);
            saving[d] = (two > one ? two - one : 0) * V + kDispatch;
        }
        // cnt[(i*(D+1) + d)*n + sh]: entries of output i with shifts sh and sh+d both unpaired
        std::vector<std::uint32_t> cnt(std::size_t(E) * (D + 1) * n, 0);
        std::vector<bool> taken(cnt.size(), false);
        for (std::size_t x = 0; x < entries.size(); ++x)
            for (std::uint32_t m = rem[x]; m; m &= m - 1) {
                const std::uint32_t sh = static_cast<std::uint32_t>(std::countr_zero(m));
                for (std::uint32_t d = 1; d <= D; ++d)
                    if ((rem[x] >> ((sh + d) % n)) & 1u) ++cnt[(entries[x].i * (D + 1) + d) * n + sh];
            }
        auto drop_bit = [&](std::size_t x, std::uint32_t b) { // shift b of entry x is now paired
            const std::uint32_t i = entries[x].i;
            for (std::uint32_t d = 1; d <= D; ++d) {
                if ((rem[x] >> ((b + d) % n)) & 1u) --cnt[(i * (D + 1) + d) * n + b];
                const std::uint32_t q = (b + n - d) % n;
                if ((rem[x] >> q) & 1u) --cnt[(i * (D + 1) + d) * n + q];
            }
            rem[x] &= ~(1u << b);
            if (--need[i * n + b] == 0) singles -= single_bytes[b];
        };
        for (;;) {
            std::size_t best = cnt.size();
            std::uint64_t best_score = 0;
            for (std::size_t c = 0; c < cnt.size(); ++c) {
                if (cnt[c] < min_uses && !taken[c]) continue; // (A/B knob: a case hardly used only adds code)
                const std::uint64_t score = std::uint64_t(cnt[c]) * saving[(c / n) % (D + 1)];
                if (score > best_score) best = c, best_score = score;
            }
            if (best == cnt.size()) break;
            const std::uint32_t sh = static_cast<std::uint32_t>(best % n), d = static_cast<std::uint32_t>((best / n) % (D + 1)),
                                i = static_cast<std::uint32_t>(best / n / (D + 1)), sh2 = (sh + d) % n;
            const std::uint32_t both = (1u << sh) | (1u << sh2), hits = cnt[best];
            // the budget with the singles that would remain: every hit entry drops both shifts
            const std::uint32_t add = taken[best] ? 0u : bytes_of(sh, d);
            const std::uint32_t freed = (need[i * n + sh] == hits ? single_bytes[sh] : 0u) +
                                        (need[i * n + sh2] == hits ? single_bytes[sh2] : 0u);
            if (pair_bytes + add + singles - freed > budget) break;
            for (std::size_t x = 0; x < entries.size(); ++x)
                if (entries[x].i == i && (rem[x] & both) == both) {
                    drop_bit(x, sh);
                    drop_bit(x, sh2);
                    entries[x].ops.emplace_back(sh, d);
                }
            pair_bytes += add;
            taken[best] = true;
        }
    }
    for (std::size_t x = 0; x < entries.size(); ++x)
        for (std::uint32_t m = rem[x]; m; m &= m - 1)
            entries[x].ops.emplace_back(static_cast<std::uint32_t>(std::countr_zero(m)), 0u);
    return pair_bytes + singles;
}

// device = false: the same launch plan without tensor maps or a device query
// (interpret_ring_rt, the host check of the planner)
void build_ring_rt(RtCall& call, const Program& p, const std::uint8_t* const* in, std::uint8_t* const* out,
                   std::uint64_t strip, std::uint64_t off, std::uint64_t len, std::uint64_t nb, std::uint64_t in_pitch,
                   std::uint64_t out_pitch, bool device = true) {
    call.args.clear();
    call.launches.clear();
    call.bins.clear();
    call.ctas_per_sm.clear();
    call.case_bytes.clear();
    call.op_count.clear();
    RtArgs tmpl;
    RtArgs& a = tmpl;
    const std::uint32_t w = p.field.w, n = p.field.n, k = p.cols;
    const std::uint32_t tile = kRtTile, slot = w * tile;
    const std::uint64_t tpb = (len + tile - 1) / tile;
    bind_rt_geometry(a, p, in, strip, off, len, nb, in_pitch, out_pitch, device);
    std::memset(a.fm, 0, sizeof a.fm);
    const bool par = p.kind == TransformKind::Parity;
    if (par) // strip w+q of the extended input = XOR of strips i = q (mod s) (phi_P, transform.hpp:50-60)
        for (std::uint32_t q = 0; q + w < n; ++q)
            for (std::uint32_t i = q; i < w; i += p.field.s) a.fm[q * w + i] = ~0u;
    RtLaunch l;
    l.w = w;
    l.n = n;
    l.modulus = p.field.modulus;
    l.parity = par;
    static const bool pdl = env_int("PYRIT_B200_PDL", 1) != 0;
    l.pdl = pdl;
    // Outputs go to R parts of 2048/(4V) threads that all read the same tiles
    // (16 warps per SM): V = 4 (16 bytes of each strip per thread) halves the
    // dispatch per XOR and doubles the XORs between jumps; V = 2 holds more
    // outputs per part.  A single output runs one 256-thread part per CTA, two
    // CTAs per SM.  More outputs than one CTA holds form output groups: each
    // (tile, group) is a unit of the same launch, and the groups of a tile run on
    // neighbouring CTAs, so the tile's re-reads come from L2, not HBM.  Past
    // kRtMaxGroups groups, further launches.
    static const int vknob = env_int("PYRIT_B200_RT_V", 4);
    const std::uint32_t V = vknob == 2 ? 2u : 4u;
    const std::uint32_t ep = static_cast<std::uint32_t>(rt_part_outputs(static_cast<int>(n), static_cast<int>(w),
                                                                        static_cast<int>(V)));
    // PYRIT_B200_RT_PARTS=2: at most two parts per CTA (two CTAs per SM, more groups)
    static const int parts_knob = env_int("PYRIT_B200_RT_PARTS", 4);
    const std::uint32_t max_parts = V == 4 && parts_knob != 2 ? 4u : 2u;
    // PYRIT_B200_RT_SOLO=1: every output its own group of one 256-thread part
    // (two CTAs per SM, no lockstep between outputs; a tile's inputs re-read from L2)
    static const bool solo = env_int("PYRIT_B200_RT_SOLO", 0) != 0;
    const std::uint32_t per_group = solo ? 1u : max_parts * ep;
    LaunchInfo info;
    auto r_for = [&](std::uint32_t e) {
        return e == 1 || solo ? 1u : V == 2 || max_parts == 2 ? 2u : e <= 2 * ep ? 2u : 4u;
    };
    for (std::uint32_t i0 = 0, e = 0; i0 < p.rows; i0 += e) {
        // as many groups as fit the op budget (ring terms + one sentinel per list)
        e = std::min(per_group * kRtMaxGroups, p.rows - i0);
        for (;;) {
            std::uint64_t terms = 0;
            for (std::uint32_t i = 0; i < e; ++i)
                for (std::uint32_t j = 0; j < k; ++j) terms += std::popcount(p.reps[std::size_t(i0 + i) * k + j]);
            const std::uint64_t lists = std::uint64_t((e + per_group - 1) / per_group) * r_for(e) * k;
            if (terms + lists + 2 < kRtMaxOps || e == 1) break;
            e = e > per_group ? (e - 1) / per_group * per_group : e - 1;
        }
        if (e == 1 || solo) {
            l.V = 2;
            l.R = 1;
        } else if (V == 2) {
            l.V = 2;
            l.R = 2;
        } else {
            l.V = 4;
            l.R = r_for(e);
        }
        // the four-part shape feeds its slots from a producer warp group (ring_rt.cuh; measured
        // config 4 0.785 -> 0.946 of peak, profiles/r02/ring_rt_pairs/producer_group/);
        // PYRIT_B200_RT_PW=0: from the first thread of the lightest part, as the smaller shapes do
        static const bool pw_knob = env_int("PYRIT_B200_RT_PW", 1) != 0;
        l.pw = pw_knob && l.R == 4 && l.V == 4;
        const std::uint32_t G = (e + per_group - 1) / per_group;
        l.E = (e + l.R * G - 1) / (l.R * G);
        a.ngrp = G;
        // the parts of a group run in lockstep on the shared slots, so give
        // them equal ring terms: heaviest output first onto the lightest
        // (group, part) bin with room (config 5's rows weigh 16/62/72/80)
        std::vector<std::uint32_t> wt(e, 0), order(e);
        for (std::uint32_t i = 0; i < e; ++i) {
            order[i] = i;
            for (std::uint32_t j = 0; j < k; ++j) wt[i] += std::popcount(p.reps[std::size_t(i0 + i) * k + j]);
        }
        std::stable_sort(order.begin(), order.end(), [&](std::uint32_t x, std::uint32_t y) { return wt[x] > wt[y]; });
        const std::uint32_t bins = G * l.R;
        std::vector<std::vector<std::uint32_t>> rows_of(bins);
        std::vector<std::uint32_t> load(bins, 0);
        for (std::uint32_t i : order) {
            std::uint32_t best = bins;
            for (std::uint32_t q = 0; q < bins; ++q)
                if (rows_of[q].size() < l.E && (best == bins || load[q] < load[best])) best = q;
            rows_of[best].push_back(i0 + i);
            load[best] += wt[i];
        }
        std::memset(a.epart, 0, sizeof a.epart);
        for (std::uint32_t q = 0; q < bins; ++q) {
            std::sort(rows_of[q].begin(), rows_of[q].end());
            a.epart[q / l.R][q % l.R] = static_cast<std::uint32_t>(rows_of[q].size());
        }
        // the TMA producer: the first thread of the part that carries least over all groups
        std::uint32_t light = 0, light_load = ~0u;
        for (std::uint32_t part = 0; part < l.R; ++part) {
            std::uint32_t sum = 0;
            for (std::uint32_t g = 0; g < G; ++g) sum += load[g * l.R + part];
            if (sum <= light_load) light = part, light_load = sum;
        }
        a.prod = light * rt_part_threads(l.V);
        const std::uint32_t cta_threads = l.R * rt_part_threads(l.V);
        const std::uint32_t ctas_per_sm = 512 / cta_threads;
        // op lists, one per (group, part, input), each ended by the sentinel E*(D+1)*n;
        // with paired-shift cases (D > 0) two set bits of a representative at most D
        // ring positions apart become one op
        // Which pair cases THIS matrix uses: the jumps are data dependent, so the hot
        // code is every case the op lists name, and it has to stay well inside the
        // instruction cache (measured on config 5: ~36 KB of cases 0.68 of peak, 23-32 KB
        // 0.75-0.79; profiles/r02/ring_rt_pairs/).  rt_select_pairs spends the budget on
        // the cases that remove most instructions.  Knobs for A/B runs only:
        // PYRIT_B200_RT_PAIRS=0 (singles only), _RT_CODE_KB, _RT_PAIR_DMAX, _RT_PAIR_MINUSE.
        static const int pairs_knob = env_int("PYRIT_B200_RT_PAIRS", 1);
        static const int code_kb = env_int("PYRIT_B200_RT_CODE_KB", 26);
        const std::uint32_t D = rt_pair_d(w, n, l.V);
        const std::uint32_t xr = par ? n : w, ar = par ? w : n;
        auto case_rows = [&](std::uint32_t sh, std::uint32_t ds) { // gen_ring_rt.py emit(): one LOP3 per reached row and word
            std::uint32_t rows = 0;
            for (std::uint32_t r = 0; r < ar; ++r)
                rows += (r + n - sh) % n < xr || (ds && (r + 2 * n - sh - ds) % n < xr);
            return rows;
        };
        std::vector<RtEntry> entries;
        for (std::uint32_t q = 0; q < bins; ++q)
            for (std::uint32_t j = 0; j < k; ++j)
                for (std::uint32_t i = 0; i < rows_of[q].size(); ++i)
                    entries.push_back({i, p.reps[std::size_t(rows_of[q][i]) * k + j], {}});
        static const int dmax_knob = env_int("PYRIT_B200_RT_PAIR_DMAX", 64);
        const std::uint32_t code = rt_select_pairs(entries, n, pairs_knob ? std::min<std::uint32_t>(D, static_cast<std::uint32_t>(std::max(0, dmax_knob))) : 0, l.E, l.V,
                                                   static_cast<std::uint32_t>(code_kb) * 1024u, case_rows);
        std::uint32_t nops = 0;
        std::size_t ent = 0;
        for (std::uint32_t g = 0; g < G; ++g)
            for (std::uint32_t part = 0; part < l.R; ++part) {
                const std::vector<std::uint32_t>& pr = rows_of[g * l.R + part];
                const std::uint32_t ne = static_cast<std::uint32_t>(pr.size());
                for (std::uint32_t j = 0; j < k; ++j) {
                    a.opoff[g][part][j] = static_cast<std::uint16_t>(nops);
                    for (std::uint32_t i = 0; i < ne; ++i)
                        for (const auto& [sh, ds] : entries[ent++].ops) {
                            if (nops + 2 >= kRtMaxOps)
                                raise(Errc::InvalidArgument, "ring_rt: too many ring terms per launch");
                            a.ops[nops++] = static_cast<std::uint8_t>((i * (D + 1) + ds) * n + sh);
                        }
                    a.ops[nops++] = static_cast<std::uint8_t>(l.E * (D + 1) * n);
                }
                a.opoff[g][part][k] = static_cast<std::uint16_t>(nops);
                for (std::uint32_t i = 0; i < ne; ++i) a.out[g][part * kRtPartE + i] = out[pr[i]];
            }
        static const bool trace = env_int("PYRIT_B200_RT_TRACE", 0) != 0;
        if (trace)
            std::fprintf(stderr, "ring_rt w%u n%u e%u k%u: %u ops, %u B of cases\n", w, n, e, k, nops - G * l.R * k, code);
        a.ops[nops] = 0; // the byte the last list's look-ahead reads
        a.nops = nops + 1;
        // shared memory: mbarriers, op lists, then as many fragment slots as fit (<= 32)
        std::uint32_t ns = 32, bar = 0;
        const std::uint32_t budget = (ctas_per_sm == 2 ? 113 : 227) * 1024;
        for (; ns >= 2; --ns) {
            bar = (16 * ns + a.nops + 127) / 128 * 128;
            if (bar + ns * slot <= budget) break;
        }
        a.nslot = ns;
        a.slot0 = bar;
        l.smem = bar + ns * slot;
        l.blocks = rt_blocks(tpb * nb * G, ctas_per_sm, device);
        call.args.push_back(std::make_unique<RtArgs>(a));
        call.launches.push_back(l);
        call.bins.push_back(rows_of);
        call.ctas_per_sm.push_back(ctas_per_sm);
        call.case_bytes.push_back(code);
        call.op_count.push_back(nops - G * l.R * k);
        info.blocks = l.blocks;
        info.threads = l.R * rt_part_threads(l.V) + (l.pw ? 128u : 0u); // + the producer warp group
    }
    info.kernel = "pyrit_ring_rt_w" + std::to_string(w) + "_n" + std::to_string(n) + (par ? "_par" : "");
    info.lanes = 2;
    info.staged = true;
    call.info = info;
}

// x^t mod p (ring_rt.cu xpow_mod)
std::uint32_t rt_xpow_mod(std::uint32_t t, std::uint32_t p, std::uint32_t w) {
    std::uint64_t a = std::uint64_t(1) << t;
    for (std::uint32_t d = t; d >= w; --d)
        if ((a >> d) & 1u) a ^= std::uint64_t(p) << (d - w);
    return static_cast<std::uint32_t>(a);
}

} // namespace

// Host restatement of what the runtime-matrix kernel computes from the launch
// plan it would be given: same units (tile, group), parts, op lists (read back
// from the kernel parameters), parity extension, fold and column window, one
// 8-byte column word at a time.  Lets CPU tests check the planner (balancing,
// groups, op encoding, op budget) against the oracle without a GPU.
void interpret_ring_rt(const Program& p, const std::uint8_t* const* in, std::uint8_t* const* out, std::uint64_t strip,
                       std::uint64_t off, std::uint64_t len, std::uint64_t nb, std::uint64_t in_pitch,
                       std::uint64_t out_pitch) {
    if (nb == 1) in_pitch = out_pitch = 0;
    if (!ring_rt_eligible(p, in, out, strip, off, len, nb, in_pitch, out_pitch))
        raise(Errc::InvalidArgument, "not a runtime-matrix kernel launch (geometry, alignment or aliasing)");
    RtCall call;
    build_ring_rt(call, p, in, out, strip, off, len, nb, in_pitch, out_pitch, false);
    const std::uint32_t w = p.field.w, n = p.field.n, k = p.cols;
    const bool par = p.kind == TransformKind::Parity;
    const std::uint32_t xr = par ? n : w, ar = par ? w : n;
    const std::uint64_t ibp = nb > 1 ? in_pitch : strip * w;
    for (std::size_t c = 0; c < call.launches.size(); ++c) {
        const RtArgs& a = *call.args[c];
        const RtLaunch& l = call.launches[c];
        const std::uint32_t E = l.E, G = a.ngrp, D = rt_pair_d(w, n, l.V);
        std::vector<std::uint64_t> acc(std::size_t(E) * ar), x(n);
        for (std::uint64_t u = 0; u < std::uint64_t(a.ntiles) * G; ++u) {
            const std::uint64_t t = u / G, g = u % G, b = t / a.tpb, tt = t - b * a.tpb;
            for (std::uint32_t part = 0; part < l.R; ++part) {
                const std::uint32_t ep = a.epart[g][part];
                for (std::uint64_t col = 0; col < kRtTile; col += 8) {
                    const std::uint64_t rel = tt * kRtTile + col;
                    if (rel >= a.len) break; // the kernel loads these columns but never stores them
                    std::fill(acc.begin(), acc.end(), 0);
                    std::uint32_t q = a.opoff[g][part][0];
                    for (std::uint32_t j = 0; j < k; ++j) {
                        for (std::uint32_t s2 = 0; s2 < w; ++s2)
                            std::memcpy(&x[s2], in[j] + b * ibp + s2 * strip + a.off + rel, 8);
                        if (par)
                            for (std::uint32_t q2 = w; q2 < n; ++q2) {
                                x[q2] = 0;
                                for (std::uint32_t i = 0; i < w; ++i)
                                    if (a.fm[(q2 - w) * w + i]) x[q2] ^= x[i];
                            }
                        for (;;) {
                            const std::uint32_t op = a.ops[q++];
                            if (op == E * (D + 1) * n) break;
                            const std::uint32_t ids = op / n, sh = op % n, i = ids / (D + 1), ds = ids % (D + 1);
                            for (std::uint32_t half = 0; half < (ds ? 2u : 1u); ++half)
                                for (std::uint32_t s2 = 0; s2 < xr; ++s2) {
                                    const std::uint32_t r = (s2 + sh + half * ds) % n;
                                    if (par && r >= w) continue;
                                    acc[std::size_t(i) * ar + r] ^= x[s2];
                                }
                        }
                    }
                    for (std::uint32_t i = 0; i < ep; ++i) {
                        std::uint64_t* A = &acc[std::size_t(i) * ar];
                        if (!par)
                            for (std::uint32_t t2 = w; t2 < n; ++t2)
                                for (std::uint32_t r = 0; r < w; ++r)
                                    if ((rt_xpow_mod(t2, p.field.modulus, w) >> r) & 1u) A[r] ^= A[t2];
                        std::uint8_t* dst = a.out[g][part * kRtPartE + i] + a.off + rel + b * a.obp;
                        for (std::uint32_t r = 0; r < w; ++r) std::memcpy(dst + r * strip, &A[r], 8);
                    }
                }
            }
        }
    }
}

// launches, ring terms of the matrix, ops the launches run for them (a pair op covers
// two terms), and the largest case-code footprint of a launch
void ring_rt_plan_info(const Program& p, std::uint32_t info[4]) {
    if (p.crs || p.sched || p.reps.empty() || p.rows == 0 || p.cols > kRtMaxK ||
        !rt_supported(p.field.w, p.field.n, p.field.modulus))
        raise(Errc::InvalidArgument, "not a runtime-matrix kernel program");
    std::vector<const std::uint8_t*> in(p.cols, nullptr);
    std::vector<std::uint8_t*> out(p.rows, nullptr);
    RtCall call;
    build_ring_rt(call, p, in.data(), out.data(), kRtTile, 0, kRtTile, 1, 0, 0, false);
    info[0] = static_cast<std::uint32_t>(call.launches.size());
    info[1] = info[2] = info[3] = 0;
    for (std::uint32_t m : p.reps) info[1] += static_cast<std::uint32_t>(std::popcount(m));
    for (std::size_t c = 0; c < call.launches.size(); ++c) {
        info[2] += call.op_count[c];
        info[3] = std::max(info[3], call.case_bytes[c]);
    }
}

LaunchInfo launch_ring_rt_program(const Program& p, const std::uint8_t* const* in, std::uint8_t* const* out,
                                  std::uint64_t strip, std::uint64_t off, std::uint64_t len, std::uint64_t nb,
                                  std::uint64_t in_pitch, std::uint64_t out_pitch, cudaStream_t stream) {
    thread_local RtCall last;
    int dev = 0;
    check_cuda(cudaGetDevice(&dev), "cudaGetDevice");
    bool same = !p.key.empty() && last.key == p.key && last.dev == dev && last.strip == strip && last.off == off &&
                last.len == len && last.nb == nb && last.ip == in_pitch && last.op == out_pitch &&
                last.in.size() == p.cols && last.out.size() == p.rows;
    for (std::uint32_t j = 0; same && j < p.cols; ++j) same = last.in[j] == in[j];
    for (std::uint32_t i = 0; same && i < p.rows; ++i) same = last.out[i] == out[i];
    if (!same) {
        // the planned launches of the last programs of this thread (a function of the
        // matrix only): a known program on new buffers is re-bound, not re-planned
        struct Planned {
            std::vector<RtArgs> args;
            std::vector<RtLaunch> launches;
            std::vector<std::vector<std::vector<std::uint32_t>>> bins;
            std::vector<std::uint32_t> ctas_per_sm;
            LaunchInfo info;
        };
        thread_local std::unordered_map<std::string, std::shared_ptr<Planned>> planned;
        const bool keep = last.key == p.key && !p.key.empty(); // same program, other buffers: args are in place
        last.key.clear(); // invalid until fully built
        auto hit = keep || p.key.empty() ? planned.end() : planned.find(p.key);
        if (keep)
            bind_ring_rt(last, p, in, out, strip, off, len, nb, in_pitch, out_pitch);
        else if (hit != planned.end()) {
            const Planned& pl = *hit->second;
            last.args.clear();
            for (const RtArgs& a : pl.args) last.args.push_back(std::make_unique<RtArgs>(a));
            last.launches = pl.launches;
            last.bins = pl.bins;
            last.ctas_per_sm = pl.ctas_per_sm;
            last.info = pl.info;
            bind_ring_rt(last, p, in, out, strip, off, len, nb, in_pitch, out_pitch);
        } else {
            build_ring_rt(last, p, in, out, strip, off, len, nb, in_pitch, out_pitch);
            if (!p.key.empty()) {
                if (planned.size() >= 32) planned.clear();
                auto pl = std::make_shared<Planned>();
                for (const auto& a : last.args) pl->args.push_back(*a);
                pl->launches = last.launches;
                pl->bins = last.bins;
                pl->ctas_per_sm = last.ctas_per_sm;
                pl->info = last.info;
                planned.emplace(p.key, std::move(pl));
            }
        }
        last.key = p.key;
        last.dev = dev;
        last.strip = strip;
        last.off = off;
        last.len = len;
        last.nb = nb;
        last.ip = in_pitch;
        last.op = out_pitch;
        last.in.assign(in, in + p.cols);
        last.out.assign(out, out + p.rows);
    }
    for (std::size_t c = 0; c < last.launches.size(); ++c) {
        RtLaunch l = last.launches[c];
        l.stream = stream;
        check_cuda(launch_ring_rt(*last.args[c], l), "ring_rt launch");
        ++g_launches;
    }
    g_last = last.info;
    return last.info;
}

std::string prepare_program(const Program& p, std::uint32_t lanes) {
    int dev = 0;
    check_cuda(cudaGetDevice(&dev), "cudaGetDevice");
    KernelShape ks = direct_shape(p, lanes);
    if (kernel_mode() != 1) {
        const KernelShape st = staged_for(p);
        if (st.staged) ks = st;
    }
    load_kernel(p, ks, dev);
    return kernel_name(p, ks);
}

LaunchInfo launch_program(const Program& p, const std::uint8_t* const* in, std::uint8_t* const* out,
                          std::uint64_t strip, std::uint64_t off, std::uint64_t len, cudaStream_t stream) {
    return launch_batch(p, in, out, strip, off, len, 1, 0, 0, stream);
}

LaunchInfo launch_batch(const Program& p0, const std::uint8_t* const* in, std::uint8_t* const* out,
                        std::uint64_t strip, std::uint64_t off, std::uint64_t len, std::uint64_t nb,
                        std::uint64_t in_pitch, std::uint64_t out_pitch, cudaStream_t stream) {
    LaunchInfo info;
    if (off + len > strip) raise(Errc::BufferShape, "column window out of range");
    if (len == 0 || nb == 0) return info;
    if (nb == 1) in_pitch = out_pitch = 0;
    int dev = 0;
    check_cuda(cudaGetDevice(&dev), "cudaGetDevice");
    const int mode = kernel_mode();
    const bool rt_ok = mode != 3 && rt_policy() != 0 &&
                       ring_rt_eligible(p0, in, out, strip, off, len, nb, in_pitch, out_pitch);
    if (rt_ok && (mode == 4 || rt_policy() == 2))
        return launch_ring_rt_program(p0, in, out, strip, off, len, nb, in_pitch, out_pitch, stream);
    // a light (decode-pattern) program stays on the runtime-matrix kernel unless
    // a specialised kernel was prebuilt for it (the benchmarked patterns) or a
    // kernel mode asks for the generated kernels
    if (p0.light && rt_ok && mode == 0 && !prebuilt_plan(p0.key)) {
        // a hot pattern (PYRIT_B200_HOT_PATTERN launches, default 8, with tiered
        // compilation on) gets its specialised kernel compiled in the background;
        // once that is ready its launches take it, until then the runtime kernel
        static const int hot = env_int("PYRIT_B200_HOT_PATTERN", 8);
        bool specialised = false;
        if (hot > 0 && tiered() && p0.lazy) {
            const std::uint32_t uses = ++p0.lazy->uses;
            if (uses >= static_cast<std::uint32_t>(hot)) {
                const Program& fp = full_program(p0);
                const KernelShape ks = choose_shape(fp, in, out, strip, off, len, nb, in_pitch, out_pitch);
                const std::string name = kernel_name(fp, ks);
                specialised = kernel_ready(name, dev);
                if (!specialised && uses == static_cast<std::uint32_t>(hot)) start_async_compile(fp, ks, name);
            }
        }
        if (!specialised)
            return launch_ring_rt_program(p0, in, out, strip, off, len, nb, in_pitch, out_pitch, stream);
    }
    const Program& p = full_program(p0);
    KernelShape ks = choose_shape(p, in, out, strip, off, len, nb, in_pitch, out_pitch);
    if (ks.split > 1 && any_alias(p, in, out, strip, nb, in_pitch, out_pitch)) {
        // split kernels walk a column with several thread groups: one group may
        // store an output column before another loads the input it aliases
        ks.split = 0;
        ks.min_blocks = 1;
    }
    const bool gen_ok = generic_ok(p, in, out, strip, off, len, nb, in_pitch, out_pitch) &&
                        !unsafe_alias(p, in, out, strip, nb, in_pitch, out_pitch);
    if (gen_ok && mode == 3) return launch_generic_program(p, in, out, strip, off, len, nb, in_pitch, out_pitch, stream);
    if ((rt_ok || gen_ok) && (tiered() || (rt_ok && p.adhoc))) {
        // a kernel that is not ready yet: the runtime-matrix ring kernel (else
        // the generic bit-matrix kernel) serves the launch; programs of one of
        // many erasure patterns (decode) never compile, others compile in the
        // background for the next launches
        const std::string name = kernel_name(p, ks);
        if (!kernel_ready(name, dev)) {
            if (rt_ok && p.adhoc) return launch_ring_rt_program(p, in, out, strip, off, len, nb, in_pitch, out_pitch, stream);
            if (start_async_compile(p, ks, name))
                return rt_ok ? launch_ring_rt_program(p, in, out, strip, off, len, nb, in_pitch, out_pitch, stream)
                             : launch_generic_program(p, in, out, strip, off, len, nb, in_pitch, out_pitch, stream);
        }
    }
    const LoadedKernel k = load_kernel(p, ks, dev);
    // Args: in[cols], out[rows], S, off, len|nwords, nb, ibp, obp (, sq, sr)
    // (, tensor maps tm[cols] at the next 64-byte boundary for TMA tensor copies)
    const std::size_t head = std::size_t(p.cols) + p.rows + 8;
    const std::size_t tm_off = (8 * (std::size_t(p.cols) + p.rows + 6) + 63) / 64 * 8; // in u64 words
    const bool tensor = ks.staged && ks.copy == 2;
    const std::size_t nmaps = tensor ? (ks.tmap4 ? 1 : p.cols) : 0;
    std::vector<std::uint64_t> args(tensor ? tm_off + 16 * nmaps : head, 0);
    for (std::uint32_t j = 0; j < p.cols; ++j) args[j] = reinterpret_cast<std::uint64_t>(in[j]);
    for (std::uint32_t i = 0; i < p.rows; ++i) args[p.cols + i] = reinterpret_cast<std::uint64_t>(out[i]);
    std::uint64_t* tail = &args[p.cols + p.rows];
    tail[0] = strip;
    tail[1] = off;
    tail[3] = nb;
    tail[4] = in_pitch;
    tail[5] = out_pitch;
    const std::uint64_t cap = std::uint64_t(k.sms) * std::uint64_t(k.blocks_per_sm);
    const std::uint64_t cpb = ks.split > 1 ? ks.threads / ks.split : ks.threads; // column threads per block
    std::uint64_t want, nwords = 0;
    if (ks.staged) {
        tail[2] = len; // bytes; tiles of ks.tile bytes per strip
        want = (len + ks.tile - 1) / ks.tile * nb;
    } else {
        const std::uint64_t vbytes = ks.lanes ? 4ull * ks.lanes : ks.half ? 2ull : 1ull;
        nwords = len / vbytes;
        tail[2] = nwords;
        want = (nwords * nb + cpb - 1) / cpb;
    }
    const unsigned blocks = static_cast<unsigned>(std::max<std::uint64_t>(1, std::min(want, cap)));
    if (tensor) {
        // 3D map per input: (column element, strip, stripe); box = one tile of
        // all w strips of one stripe; elements of 4 bytes (8 for 2 KiB tiles)
        const std::uint32_t elem = ks.tile > 1024 ? 8 : 4;
        static const int promo_knob = env_int("PYRIT_B200_TMA_PROMO", 3); // tuning: 0 none .. 3 = 256B
        const CUtensorMapL2promotion promo = static_cast<CUtensorMapL2promotion>(std::min(3, std::max(0, promo_knob)));
        if (ks.tmap4) {
            // 4D: (column element, strip, fragment, stripe)
            CUtensorMap m;
            const std::uint64_t d = reinterpret_cast<std::uintptr_t>(in[1]) - reinterpret_cast<std::uintptr_t>(in[0]);
            const std::uint32_t G = p.parts.empty() ? 1 : p.parts[0].group;
            const cuuint64_t dims[4] = {strip / elem, p.field.w, p.cols, nb};
            const cuuint64_t strides[3] = {strip, d, nb > 1 ? in_pitch : d * p.cols};
            const cuuint32_t box[4] = {ks.tile / elem, p.field.w, G, 1};
            const cuuint32_t es[4] = {1, 1, 1, 1};
            check_cu(driver().tensorMapEncodeTiled(&m, elem == 8 ? CU_TENSOR_MAP_DATA_TYPE_UINT64 : CU_TENSOR_MAP_DATA_TYPE_UINT32,
                                                   4, const_cast<std::uint8_t*>(in[0]), dims, strides, box, es,
                                                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, promo,
                                                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE),
                     "cuTensorMapEncodeTiled(4D)");
            std::memcpy(&args[tm_off], &m, sizeof m);
        }
        for (std::uint32_t j = 0; !ks.tmap4 && j < p.cols; ++j) {
            CUtensorMap m;
            const cuuint64_t dims[3] = {strip / elem, p.field.w, nb};
            const cuuint64_t strides[2] = {strip, nb > 1 ? in_pitch : strip * p.field.w};
            const cuuint32_t box[3] = {ks.tile / elem, ks.spb ? ks.spb : p.field.w, 1};
            const cuuint32_t es[3] = {1, 1, 1};
            check_cu(driver().tensorMapEncodeTiled(&m, elem == 8 ? CU_TENSOR_MAP_DATA_TYPE_UINT64 : CU_TENSOR_MAP_DATA_TYPE_UINT32,
                                                   3, const_cast<std::uint8_t*>(in[j]), dims, strides, box, es,
                                                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, promo,
                                                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE),
                     "cuTensorMapEncodeTiled");
            std::memcpy(&args[tm_off + 16 * std::size_t(j)], &m, sizeof m);
        }
    }
    if (!ks.staged) {
        const std::uint64_t stride = std::uint64_t(blocks) * cpb;
        tail[6] = stride / nwords;
        tail[7] = stride % nwords;
    }
    void* params[] = {args.data()};
    // programmatic stream serialisation: the kernel may be scheduled while the
    // previous work on the stream drains; it waits (griddepcontrol.wait) before
    // touching global memory, so ordering is unchanged (PYRIT_B200_PDL=0 disables)
    static const bool pdl = env_int("PYRIT_B200_PDL", 1) != 0;
    CUlaunchAttribute attr{};
    attr.id = CU_LAUNCH_ATTRIBUTE_PROGRAMMATIC_STREAM_SERIALIZATION;
    attr.value.programmaticStreamSerializationAllowed = 1;
    CUlaunchConfig cfg{};
    cfg.gridDimX = blocks;
    cfg.gridDimY = cfg.gridDimZ = 1;
    cfg.blockDimX = ks.threads + (ks.staged && ks.copy == 2 && ks.ws ? 32u : 0u);
    cfg.blockDimY = cfg.blockDimZ = 1;
    cfg.sharedMemBytes = ks.staged ? ks.smem_bytes : 0;
    cfg.hStream = reinterpret_cast<CUstream>(stream);
    cfg.attrs = pdl ? &attr : nullptr;
    cfg.numAttrs = pdl ? 1 : 0;
    check_cu(driver().launchKernelEx(&cfg, k.fn, params, nullptr), "cuLaunchKernelEx");
    ++g_launches;
    info.lanes = ks.lanes;
    info.threads = ks.threads;
    info.blocks = blocks;
    info.staged = ks.staged;
    info.kernel = kernel_name(p, ks);
    g_last = info;
    return info;
}

LaunchInfo last_launch() { return g_last; }

} // namespace pyrit_b200
