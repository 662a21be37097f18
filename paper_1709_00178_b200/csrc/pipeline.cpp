// Host-buffer path: the end-to-end encode()/decode() a reference user calls
// with SymbolBuffer-resident bytes (codec.hpp:212, :241).  Strips are moved
// in column chunks through a ring of device staging slots, one stream per
// slot, so the H2D copy of chunk c+1, the fused kernel of chunk c and the
// D2H copy of chunk c-1 overlap on the two copy engines and the SMs.
#include "pipeline.hpp"

#include <immintrin.h>
#include <sched.h>

#include <cstdio>
#include <cstring>

#include "hostpool.hpp"

#include <algorithm>
#include <cctype>
#include <cstdlib>
#include <map>
#include <memory>
#include <mutex>
#include <thread>

namespace pyrit_b200 {

namespace {

constexpr int kSlots = 3;

struct Slot {
    cudaStream_t stream = nullptr;
    std::uint8_t* buf = nullptr;
    std::size_t bytes = 0;
    // pageable callers: pinned mirror of buf, and the event after the slot's D2H
    std::uint8_t* hbuf = nullptr;
    std::size_t hbytes = 0;
    cudaEvent_t done = nullptr;
};

// true when the driver can DMA straight from/to p (page-locked or managed)
bool dma_capable(const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        (void)cudaGetLastError(); // unregistered pointers can report an error on older drivers
        return false;
    }
    return a.type == cudaMemoryTypeHost || a.type == cudaMemoryTypeManaged;
}

struct DeviceCtx {
    std::mutex mu;
    int device = 0;
    Slot slots[kSlots];
};

std::mutex g_ctx_mu;
std::map<int, std::unique_ptr<DeviceCtx>> g_ctx;
std::uint64_t g_chunk = 0;

DeviceCtx& ctx_for(int device) {
    std::lock_guard<std::mutex> lk(g_ctx_mu);
    auto& c = g_ctx[device];
    if (!c) {
        c = std::make_unique<DeviceCtx>();
        c->device = device;
    }
    return *c;
}

} // namespace

void set_host_chunk(std::uint64_t bytes) { g_chunk = bytes; }

namespace {

// "0-13,28-41" -> cpu set (sysfs cpulist)
bool parse_cpulist(const std::string& text, cpu_set_t& set) {
    CPU_ZERO(&set);
    bool any = false;
    std::size_t i = 0;
    while (i < text.size()) {
        while (i < text.size() && !std::isdigit(static_cast<unsigned char>(text[i]))) ++i;
        if (i >= text.size()) break;
        long a = 0, b;
        while (i < text.size() && std::isdigit(static_cast<unsigned char>(text[i]))) a = a * 10 + (text[i++] - '0');
        b = a;
        if (i < text.size() && text[i] == '-') {
            ++i;
            b = 0;
            while (i < text.size() && std::isdigit(static_cast<unsigned char>(text[i]))) b = b * 10 + (text[i++] - '0');
        }
        for (long c = a; c <= b && c < CPU_SETSIZE; ++c) CPU_SET(static_cast<int>(c), &set), any = true;
    }
    return any;
}

// the calling thread keeps only those of its CPUs that are in `want`; false (nothing
// changed) when none is
bool bind_thread_to(const cpu_set_t& want) {
    cpu_set_t have, both;
    if (sched_getaffinity(0, sizeof have, &have) != 0) return false;
    CPU_AND(&both, &want, &have);
    if (CPU_COUNT(&both) == 0) return false;
    return sched_setaffinity(0, sizeof both, &both) == 0;
}

std::string read_small_file(const std::string& path) {
    std::string out;
    if (FILE* f = std::fopen(path.c_str(), "r")) {
        char buf[4096];
        const std::size_t n = std::fread(buf, 1, sizeof buf, f);
        out.assign(buf, n);
        std::fclose(f);
    }
    return out;
}

} // namespace

int numa_bind_thread(int device) {
    static const bool enabled = [] {
        const char* e = std::getenv("PYRIT_B200_NUMA");
        return !e || std::atoi(e) != 0;
    }();
    if (!enabled) return -1;
    // the node and its CPUs per device, looked up in sysfs once per process
    struct Node {
        int node = -1;
        cpu_set_t cpus;
    };
    static std::mutex mu;
    static std::map<int, Node> known;
    Node nd;
    {
        std::lock_guard<std::mutex> lk(mu);
        auto it = known.find(device);
        if (it == known.end()) {
            Node found;
            CPU_ZERO(&found.cpus);
            char bus[32] = {};
            if (cudaDeviceGetPCIBusId(bus, sizeof bus, device) == cudaSuccess) {
                std::string id(bus);
                for (char& c : id) c = static_cast<char>(std::tolower(static_cast<unsigned char>(c)));
                const std::string node_text = read_small_file("/sys/bus/pci/devices/" + id + "/numa_node");
                const int node = node_text.empty() ? -1 : std::atoi(node_text.c_str()); // < 0: one node, or not said
                if (node >= 0 &&
                    parse_cpulist(read_small_file("/sys/devices/system/node/node" + std::to_string(node) + "/cpulist"),
                                  found.cpus))
                    found.node = node;
            } else {
                (void)cudaGetLastError();
            }
            it = known.emplace(device, found).first;
        }
        nd = it->second;
    }
    if (nd.node < 0) return -1;
    return bind_thread_to(nd.cpus) ? nd.node : -1;
}

int bind_thread_cpulist(const char* cpulist) {
    cpu_set_t want;
    if (!cpulist || !parse_cpulist(cpulist, want)) return -1;
    return bind_thread_to(want) ? CPU_COUNT(&want) : -1;
}

void run_host(const Program& p, const std::vector<const std::uint8_t*>& host_in,
              const std::vector<std::uint8_t*>& host_out, std::uint64_t strip, int device) {
    run_host_window(p, host_in, host_out, strip, 0, strip, device);
}

void run_host_devices(const Program& p, const std::vector<const std::uint8_t*>& host_in,
                      const std::vector<std::uint8_t*>& host_out, std::uint64_t strip,
                      const std::vector<int>& devices) {
    if (devices.empty()) raise(Errc::InvalidArgument, "no devices");
    // byte-offset shards of every strip: device d owns
    // [floor(d S / N), floor((d+1) S / N)) rounded down to 16 bytes, the last
    // one takes the tail; the shards are independent, one host thread each
    const std::size_t n = devices.size();
    std::vector<std::exception_ptr> errs(n);
    std::vector<std::thread> th;
    for (std::size_t d = 0; d < n; ++d) {
        const std::uint64_t lo = strip * d / n / 16 * 16;
        const std::uint64_t hi = d + 1 == n ? strip : strip * (d + 1) / n / 16 * 16;
        th.emplace_back([&, d, lo, hi] {
            try {
                // staging copies and pinned staging buffers of this shard stay on the
                // NUMA node its GPU hangs off (best effort)
                if (n > 1) numa_bind_thread(devices[d]);
                run_host_window(p, host_in, host_out, strip, lo, hi - lo, devices[d]);
            } catch (...) {
                errs[d] = std::current_exception();
            }
        });
    }
    for (auto& x : th) x.join();
    for (auto& e : errs)
        if (e) std::rethrow_exception(e);
}

namespace {

// Large host copies for the pageable staging: non-temporal (streaming)
// stores skip the read-for-ownership of the destination lines, one of the
// three memory passes of a plain memcpy (PYRIT_B200_NT_COPY=0 disables).
__attribute__((target("avx512f"))) void copy_nt512(std::uint8_t* dst, const std::uint8_t* src, std::size_t n) {
    const std::size_t head = (64 - (reinterpret_cast<std::uintptr_t>(dst) & 63)) & 63;
    std::memcpy(dst, src, head);
    dst += head;
    src += head;
    n -= head;
    std::size_t i = 0;
    for (; i + 256 <= n; i += 256) {
        const __m512i a = _mm512_loadu_si512(src + i), b = _mm512_loadu_si512(src + i + 64);
        const __m512i c = _mm512_loadu_si512(src + i + 128), d = _mm512_loadu_si512(src + i + 192);
        _mm512_stream_si512(reinterpret_cast<__m512i*>(dst + i), a);
        _mm512_stream_si512(reinterpret_cast<__m512i*>(dst + i + 64), b);
        _mm512_stream_si512(reinterpret_cast<__m512i*>(dst + i + 128), c);
        _mm512_stream_si512(reinterpret_cast<__m512i*>(dst + i + 192), d);
    }
    std::memcpy(dst + i, src + i, n - i);
    _mm_sfence();
}

void host_copy(std::uint8_t* dst, const std::uint8_t* src, std::size_t n) {
    static const bool nt = [] {
        const char* e = std::getenv("PYRIT_B200_NT_COPY");
        return (!e || std::atoi(e) != 0) && __builtin_cpu_supports("avx512f");
    }();
    if (nt && n >= (64u << 10)) copy_nt512(dst, src, n);
    else std::memcpy(dst, src, n);
}

// strips of output i that the program stores (all, except for schedule programs)
bool stores_strip(const Program& p, std::uint32_t i, std::uint32_t b) {
    return !p.sched || p.written[std::size_t(i) * p.field.w + b];
}

void run_staged(const Program& p, const std::vector<const std::uint8_t*>& host_in,
                const std::vector<std::uint8_t*>& host_out, std::uint64_t strip, std::uint64_t off,
                std::uint64_t win, std::uint64_t chunk, DeviceCtx& ctx) {
    const std::uint32_t w = p.field.w;
    const std::uint64_t in_strips = std::uint64_t(p.cols) * w;
    const std::size_t need = static_cast<std::size_t>(std::uint64_t(p.cols + p.rows) * w * chunk);
    for (Slot& s : ctx.slots) {
        if (s.hbytes < need) {
            if (s.hbuf) check_cuda(cudaFreeHost(s.hbuf), "cudaFreeHost");
            s.hbuf = nullptr;
            s.hbytes = 0;
            check_cuda(cudaHostAlloc(reinterpret_cast<void**>(&s.hbuf), need, cudaHostAllocDefault), "pinned staging");
            s.hbytes = need;
        }
        if (!s.done) check_cuda(cudaEventCreateWithFlags(&s.done, cudaEventDisableTiming), "event");
    }
    std::vector<std::pair<std::uint32_t, std::uint32_t>> out_strips; // (output, strip) stored
    for (std::uint32_t i = 0; i < p.rows; ++i)
        for (std::uint32_t b = 0; b < w; ++b)
            if (stores_strip(p, i, b)) out_strips.push_back({i, b});
    struct Pending {
        bool live = false;
        std::uint64_t c0 = 0, len = 0;
    } pend[kSlots];
    auto unpack = [&](int si) {
        Slot& s = ctx.slots[si];
        Pending& pd = pend[si];
        if (!pd.live) return;
        check_cuda(cudaEventSynchronize(s.done), "cudaEventSynchronize");
        const std::uint8_t* h_out = s.hbuf + in_strips * chunk;
        host_pool().run(out_strips.size(), [&](std::size_t q) {
            const auto [i, b] = out_strips[q];
            host_copy(host_out[i] + std::uint64_t(b) * strip + pd.c0, h_out + (std::uint64_t(i) * w + b) * chunk,
                      pd.len);
        });
        pd.live = false;
    };
    std::vector<const std::uint8_t*> din(p.cols);
    std::vector<std::uint8_t*> dout(p.rows);
    std::uint64_t c0 = off;
    try {
        for (int c = 0; c0 < off + win; ++c) {
            const std::uint64_t len = std::min(chunk, off + win - c0);
            const int si = c % kSlots;
            Slot& s = ctx.slots[si];
            unpack(si); // the slot's previous chunk is done (H2D, kernel, D2H)
            host_pool().run(in_strips, [&](std::size_t q) {
                const std::uint64_t j = q / w, b = q % w;
                host_copy(s.hbuf + q * chunk, host_in[j] + b * strip + c0, len);
            });
            check_cuda(cudaMemcpy2DAsync(s.buf, chunk, s.hbuf, chunk, len, in_strips, cudaMemcpyHostToDevice, s.stream),
                       "H2D");
            for (std::uint32_t j = 0; j < p.cols; ++j) din[j] = s.buf + std::uint64_t(j) * w * chunk;
            for (std::uint32_t i = 0; i < p.rows; ++i) dout[i] = s.buf + std::uint64_t(p.cols + i) * w * chunk;
            launch_program(p, din.data(), dout.data(), chunk, 0, len, s.stream);
            check_cuda(cudaMemcpy2DAsync(s.hbuf + in_strips * chunk, chunk, s.buf + in_strips * chunk, chunk, len,
                                         std::uint64_t(p.rows) * w, cudaMemcpyDeviceToHost, s.stream),
                       "D2H");
            check_cuda(cudaEventRecord(s.done, s.stream), "cudaEventRecord");
            pend[si] = {true, c0, len};
            c0 += len;
        }
        for (int si = 0; si < kSlots; ++si) unpack(si);
    } catch (...) {
        for (Slot& s : ctx.slots) (void)cudaStreamSynchronize(s.stream); // no copy may outlive the caller's buffers
        throw;
    }
}

} // namespace

void run_host_window(const Program& p, const std::vector<const std::uint8_t*>& host_in,
                     const std::vector<std::uint8_t*>& host_out, std::uint64_t strip, std::uint64_t off,
                     std::uint64_t win, int device) {
    const std::uint32_t w = p.field.w;
    if (host_in.size() != p.cols || host_out.size() != p.rows) raise(Errc::BufferShape, "symbol count mismatch");
    if (off + win > strip) raise(Errc::BufferShape, "column window out of range");
    if (p.rows == 0 || win == 0) return;
    DeviceCtx& ctx = ctx_for(device);
    std::lock_guard<std::mutex> lk(ctx.mu);
    check_cuda(cudaSetDevice(device), "cudaSetDevice");

    const std::uint64_t strips = std::uint64_t(p.cols + p.rows) * w;
    std::uint64_t chunk = g_chunk;
    if (chunk == 0) {
        static const char* env = std::getenv("PYRIT_B200_HOST_STAGE_MIB"); // tuning knob
        const std::uint64_t mib = env ? std::strtoull(env, nullptr, 10) : 192;
        chunk = ((mib ? mib : 192) << 20) / strips; // ~192 MiB of staging per slot
    }
    // calls get >= 16 chunks (64 KiB per strip at least) so the D2H of one
    // chunk overlaps the H2D of the next
    // (PYRIT_B200_HOST_MIN_CHUNKS, default 16: the first H2D and the last D2H
    // are the only copies nothing overlaps, so they should be small)
    static const std::uint64_t min_chunks = [] {
        const char* e = std::getenv("PYRIT_B200_HOST_MIN_CHUNKS");
        const long v = e ? std::strtol(e, nullptr, 10) : 16;
        return static_cast<std::uint64_t>(v > 0 ? v : 16);
    }();
    if (g_chunk == 0) chunk = std::min<std::uint64_t>(chunk, std::max<std::uint64_t>(64 * 1024, win / min_chunks));
    chunk = std::max<std::uint64_t>(chunk, 64 * 1024) & ~std::uint64_t(4095);
    if (win % 16 == 0) chunk = std::min(chunk, win);
    else chunk = std::min(chunk, win & ~std::uint64_t(15)); // tail chunk handled in byte mode
    if (chunk == 0) chunk = win;
    const std::size_t need = static_cast<std::size_t>(strips * chunk);
    for (Slot& s : ctx.slots) {
        if (!s.stream) check_cuda(cudaStreamCreateWithFlags(&s.stream, cudaStreamNonBlocking), "stream");
        if (s.bytes < need) {
            if (s.buf) check_cuda(cudaFree(s.buf), "cudaFree");
            s.buf = nullptr;
            s.bytes = 0;
            check_cuda(cudaMalloc(&s.buf, need), "cudaMalloc staging");
            s.bytes = need;
        }
    }
    // Pageable symbols (a reference SymbolBuffer is a std::vector): the
    // driver would stage every copy through its own small pinned buffer,
    // synchronously and on one thread (measured 8-10 GB/s).  Instead the host
    // pool packs each chunk's strips into a pinned mirror of the slot (and
    // unpacks the outputs) while the copy engines and SMs work on the other
    // slots: pack chunk c | H2D + kernel + D2H of c-1, c-2 | unpack c-3.
    bool pinned = true;
    for (const std::uint8_t* q : host_in) pinned = pinned && dma_capable(q);
    for (std::uint8_t* q : host_out) pinned = pinned && dma_capable(q);
    if (!pinned) {
        run_staged(p, host_in, host_out, strip, off, win, chunk, ctx);
        return;
    }
    // runs of symbols laid out back to back on the host (SymbolBuffer storage,
    // codec.hpp:24-73): one 2D copy moves the window of all their strips
    auto runs = [&](const auto& ptrs) {
        std::vector<std::pair<std::uint32_t, std::uint32_t>> out; // [first, end)
        for (std::uint32_t j = 0; j < ptrs.size(); ++j) {
            if (!out.empty() && ptrs[j] == ptrs[j - 1] + std::uint64_t(w) * strip) ++out.back().second;
            else out.push_back({j, j + 1});
        }
        return out;
    };
    const auto in_runs = runs(host_in);
    // outputs a schedule program writes only partly (Program::written): only
    // their written strips come back, the others stay as they are on the host
    std::vector<std::pair<std::uint32_t, std::uint32_t>> out_runs; // [first, end) of fully written outputs
    std::vector<std::pair<std::uint32_t, std::uint32_t>> partial;  // (output, strip)
    for (std::uint32_t i = 0; i < p.rows; ++i) {
        bool all = true;
        for (std::uint32_t b = 0; p.sched && b < w; ++b) all = all && p.written[std::size_t(i) * w + b];
        if (!all) {
            for (std::uint32_t b = 0; b < w; ++b)
                if (p.written[std::size_t(i) * w + b]) partial.push_back({i, b});
        } else if (!out_runs.empty() && out_runs.back().second == i &&
                   host_out[i] == host_out[i - 1] + std::uint64_t(w) * strip)
            ++out_runs.back().second;
        else
            out_runs.push_back({i, i + 1});
    }
    std::vector<const std::uint8_t*> din(p.cols);
    std::vector<std::uint8_t*> dout(p.rows);
    // PYRIT_B200_PIPE_TRACE=<file>: CUDA events around every chunk's H2D, kernel
    // and D2H, written as a timeline (ms from the first event) -- the copy-engine
    // overlap evidence nsys would give (nsys is not on these boxes)
    static const char* trace_path = std::getenv("PYRIT_B200_PIPE_TRACE");
    struct Ev {
        cudaEvent_t e[4];
        int slot;
        std::uint64_t bytes_in, bytes_out;
    };
    std::vector<Ev> trace;
    std::uint64_t c0 = off;
    try {
        for (int c = 0; c0 < off + win; ++c) {
            const std::uint64_t len = std::min(chunk, off + win - c0);
            Slot& s = ctx.slots[c % kSlots];
            for (std::uint32_t j = 0; j < p.cols; ++j) din[j] = s.buf + std::uint64_t(j) * w * chunk;
            for (std::uint32_t i = 0; i < p.rows; ++i) dout[i] = s.buf + std::uint64_t(p.cols + i) * w * chunk;
            Ev ev{};
            if (trace_path) {
                for (auto& e : ev.e) check_cuda(cudaEventCreate(&e), "trace event");
                ev.slot = c % kSlots;
                ev.bytes_in = std::uint64_t(p.cols) * w * len;
                ev.bytes_out = std::uint64_t(p.rows) * w * len;
                check_cuda(cudaEventRecord(ev.e[0], s.stream), "trace");
            }
            for (const auto& [j0, j1] : in_runs)
                check_cuda(cudaMemcpy2DAsync(const_cast<std::uint8_t*>(din[j0]), chunk, host_in[j0] + c0, strip, len,
                                             std::size_t(j1 - j0) * w, cudaMemcpyHostToDevice, s.stream),
                           "H2D");
            if (trace_path) check_cuda(cudaEventRecord(ev.e[1], s.stream), "trace");
            launch_program(p, din.data(), dout.data(), chunk, 0, len, s.stream);
            if (trace_path) check_cuda(cudaEventRecord(ev.e[2], s.stream), "trace");
            for (const auto& [i0, i1] : out_runs)
                check_cuda(cudaMemcpy2DAsync(host_out[i0] + c0, strip, dout[i0], chunk, len, std::size_t(i1 - i0) * w,
                                             cudaMemcpyDeviceToHost, s.stream),
                           "D2H");
            for (const auto& [i, b] : partial)
                check_cuda(cudaMemcpyAsync(host_out[i] + std::uint64_t(b) * strip + c0,
                                           dout[i] + std::uint64_t(b) * chunk, len, cudaMemcpyDeviceToHost, s.stream),
                           "D2H");
            if (trace_path) {
                check_cuda(cudaEventRecord(ev.e[3], s.stream), "trace");
                trace.push_back(ev);
            }
            c0 += len;
        }
        for (Slot& s : ctx.slots) check_cuda(cudaStreamSynchronize(s.stream), "cudaStreamSynchronize");
    } catch (...) {
        // no copy may outlive the caller's buffers (a later chunk's launch or copy failed)
        for (Slot& s : ctx.slots) (void)cudaStreamSynchronize(s.stream);
        throw;
    }
    if (trace_path && !trace.empty()) {
        if (FILE* f = std::fopen(trace_path, "a")) {
            std::fprintf(f, "{\"chunks\": [");
            for (std::size_t c = 0; c < trace.size(); ++c) {
                float t[4];
                for (int q = 0; q < 4; ++q) cudaEventElapsedTime(&t[q], trace[0].e[0], trace[c].e[q]);
                std::fprintf(f, "%s{\"slot\": %d, \"h2d\": [%.4f, %.4f], \"kernel\": [%.4f, %.4f], \"d2h\": [%.4f, %.4f], "
                                "\"h2d_bytes\": %llu, \"d2h_bytes\": %llu}",
                             c ? ", " : "", trace[c].slot, t[0], t[1], t[1], t[2], t[2], t[3],
                             static_cast<unsigned long long>(trace[c].bytes_in),
                             static_cast<unsigned long long>(trace[c].bytes_out));
            }
            std::fprintf(f, "]}\n");
            std::fclose(f);
        }
        for (Ev& ev : trace)
            for (auto& e : ev.e) cudaEventDestroy(e);
    }
}

} // namespace pyrit_b200
