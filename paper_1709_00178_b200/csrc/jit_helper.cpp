// pyrit_jit_helper: compiles one generated kernel with NVRTC in its own
// process.  The library's background (tiered) compiles run here, so a
// program may exit at any time without NVRTC being torn down under a
// running compile -- an orphaned helper just finishes and writes its cubin.
//
//   pyrit_jit_helper <source.cu> <kernel name> <output.cubin> [libnvrtc path]
//
// Same compiler and options as the in-process path (runtime.cpp): the
// toolkit's NVRTC, sm_100a, -lineinfo.  The cubin is written to a temporary
// name and renamed, so readers never see a partial file.
#include <dlfcn.h>
#include <nvrtc.h>
#include <unistd.h>

#include <cstdio>
#include <fstream>
#include <iterator>
#include <string>
#include <vector>

#ifndef PYRIT_NVRTC_PATH
#define PYRIT_NVRTC_PATH "libnvrtc.so.12"
#endif

int main(int argc, char** argv) {
    if (argc < 4) {
        std::fprintf(stderr, "usage: %s source.cu name out.cubin [libnvrtc]\n", argv[0]);
        return 2;
    }
    const char* lib = argc > 4 ? argv[4] : PYRIT_NVRTC_PATH;
    void* h = dlopen(lib, RTLD_NOW | RTLD_LOCAL);
    if (!h) h = dlopen("libnvrtc.so.12", RTLD_NOW | RTLD_LOCAL);
    if (!h) {
        std::fprintf(stderr, "cannot load NVRTC\n");
        return 3;
    }
    auto create = reinterpret_cast<nvrtcResult (*)(nvrtcProgram*, const char*, const char*, int, const char* const*,
                                                   const char* const*)>(dlsym(h, "nvrtcCreateProgram"));
    auto compile = reinterpret_cast<nvrtcResult (*)(nvrtcProgram, int, const char* const*)>(dlsym(h, "nvrtcCompileProgram"));
    auto log_size = reinterpret_cast<nvrtcResult (*)(nvrtcProgram, size_t*)>(dlsym(h, "nvrtcGetProgramLogSize"));
    auto get_log = reinterpret_cast<nvrtcResult (*)(nvrtcProgram, char*)>(dlsym(h, "nvrtcGetProgramLog"));
    auto cubin_size = reinterpret_cast<nvrtcResult (*)(nvrtcProgram, size_t*)>(dlsym(h, "nvrtcGetCUBINSize"));
    auto get_cubin = reinterpret_cast<nvrtcResult (*)(nvrtcProgram, char*)>(dlsym(h, "nvrtcGetCUBIN"));
    if (!create || !compile || !log_size || !get_log || !cubin_size || !get_cubin) return 3;

    std::ifstream in(argv[1], std::ios::binary);
    const std::string src((std::istreambuf_iterator<char>(in)), {});
    if (src.empty()) return 4;
    const std::string name = argv[2];
    nvrtcProgram prog;
    if (create(&prog, src.c_str(), (name + ".cu").c_str(), 0, nullptr, nullptr) != NVRTC_SUCCESS) return 5;
    const char* opts[] = {"--gpu-architecture=sm_100a", "--std=c++17", "-lineinfo", "-DNDEBUG"};
    if (compile(prog, 4, opts) != NVRTC_SUCCESS) {
        size_t n = 0;
        log_size(prog, &n);
        std::string log(n, '\0');
        get_log(prog, log.data());
        std::fprintf(stderr, "NVRTC failed for %s:\n%s\n", name.c_str(), log.c_str());
        return 6;
    }
    size_t n = 0;
    if (cubin_size(prog, &n) != NVRTC_SUCCESS) return 7;
    std::vector<char> cubin(n);
    if (get_cubin(prog, cubin.data()) != NVRTC_SUCCESS) return 7;
    const std::string out = argv[3];
    const std::string tmp = out + ".part" + std::to_string(::getpid());
    {
        std::ofstream f(tmp, std::ios::binary);
        f.write(cubin.data(), static_cast<std::streamsize>(cubin.size()));
        if (!f) return 8;
    }
    return std::rename(tmp.c_str(), out.c_str()) == 0 ? 0 : 8;
}
