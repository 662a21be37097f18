#include "container.hpp"

#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <sys/uio.h>
#include <unistd.h>

#include <algorithm>
#include <cerrno>
#include <condition_variable>
#include <functional>
#include <thread>
#include <climits>
#include <cstring>
#include <filesystem>
#include <future>
#include <map>
#include <memory>
#include <mutex>

#include "hostpool.hpp"
#include "plans.hpp"
#include "runtime.hpp"

namespace pyrit_b200 {

namespace {

constexpr std::uint8_t kMagic[4] = {'P', 'Y', 'R', 'T'};
std::uint64_t g_file_chunk = 0;

void put16(std::uint8_t* p, std::uint16_t v) {
    p[0] = static_cast<std::uint8_t>(v);
    p[1] = static_cast<std::uint8_t>(v >> 8);
}
void put32(std::uint8_t* p, std::uint32_t v) {
    for (int i = 0; i < 4; ++i) p[i] = static_cast<std::uint8_t>(v >> (8 * i));
}
void put64(std::uint8_t* p, std::uint64_t v) {
    for (int i = 0; i < 8; ++i) p[i] = static_cast<std::uint8_t>(v >> (8 * i));
}
std::uint16_t get16(const std::uint8_t* p) { return static_cast<std::uint16_t>(p[0] | (p[1] << 8)); }
std::uint32_t get32(const std::uint8_t* p) {
    std::uint32_t v = 0;
    for (int i = 0; i < 4; ++i) v |= static_cast<std::uint32_t>(p[i]) << (8 * i);
    return v;
}
std::uint64_t get64(const std::uint8_t* p) {
    std::uint64_t v = 0;
    for (int i = 0; i < 8; ++i) v |= static_cast<std::uint64_t>(p[i]) << (8 * i);
    return v;
}

// ---- POSIX file helpers (typed IoError on failure) ----------------------

struct Fd {
    int fd = -1;
    Fd() = default;
    explicit Fd(int f) : fd(f) {}
    Fd(const Fd&) = delete;
    Fd& operator=(const Fd&) = delete;
    Fd(Fd&& o) noexcept : fd(o.fd) { o.fd = -1; }
    Fd& operator=(Fd&& o) noexcept {
        std::swap(fd, o.fd);
        return *this;
    }
    ~Fd() {
        if (fd >= 0) ::close(fd);
    }
};

// reads up to len bytes at off; returns the count (short only at end of file)
std::size_t pread_full(int fd, std::uint8_t* dst, std::size_t len, std::uint64_t off, const std::string& path) {
    std::size_t got = 0;
    while (got < len) {
        const ssize_t n = ::pread(fd, dst + got, len - got, static_cast<off_t>(off + got));
        if (n < 0) {
            if (errno == EINTR) continue;
            raise(Errc::IoError, "read failed on " + path + ": " + std::strerror(errno));
        }
        if (n == 0) break;
        got += static_cast<std::size_t>(n);
    }
    return got;
}

void pwrite_full(int fd, const std::uint8_t* src, std::size_t len, std::uint64_t off, const std::string& path) {
    std::size_t put = 0;
    while (put < len) {
        const ssize_t n = ::pwrite(fd, src + put, len - put, static_cast<off_t>(off + put));
        if (n < 0 && errno == EINTR) continue;
        if (n <= 0) raise(Errc::IoError, "short write on " + path);
        put += static_cast<std::size_t>(n);
    }
}

// gathered write of (ptr, len) pieces placed back to back at off
void pwritev_full(int fd, std::vector<iovec>& iov, std::uint64_t off, const std::string& path) {
    std::size_t i = 0;
    while (i < iov.size()) {
        const int cnt = static_cast<int>(std::min<std::size_t>(iov.size() - i, IOV_MAX));
        ssize_t n = ::pwritev(fd, &iov[i], cnt, static_cast<off_t>(off));
        if (n < 0 && errno == EINTR) continue;
        if (n <= 0) raise(Errc::IoError, "short write on " + path);
        off += static_cast<std::uint64_t>(n);
        // consume n bytes of the iovec list (partial writes resume mid-piece)
        while (n > 0 && i < iov.size()) {
            if (static_cast<std::size_t>(n) >= iov[i].iov_len) {
                n -= static_cast<ssize_t>(iov[i].iov_len);
                ++i;
            } else {
                iov[i].iov_base = static_cast<char*>(iov[i].iov_base) + n;
                iov[i].iov_len -= static_cast<std::size_t>(n);
                n = 0;
            }
        }
        while (i < iov.size() && iov[i].iov_len == 0) ++i;
    }
}

// pread of [off, off+len) split over the pool; returns the bytes read
std::size_t pread_parallel(int fd, std::uint8_t* dst, std::size_t len, std::uint64_t off, const std::string& path) {
    constexpr std::size_t kPiece = 8u << 20;
    const std::size_t pieces = (len + kPiece - 1) / kPiece;
    std::vector<std::size_t> got(pieces, 0);
    host_pool().run(pieces, [&](std::size_t i) {
        const std::size_t b = i * kPiece, n = std::min(kPiece, len - b);
        got[i] = pread_full(fd, dst + b, n, off + b, path);
    });
    std::size_t total = 0;
    for (std::size_t i = 0; i < pieces; ++i) {
        total += got[i];
        if (got[i] < std::min(kPiece, len - i * kPiece)) break; // end of file
    }
    return total;
}

// A file region the host pool writes through a shared mapping: write()
// calls on one file serialise on its inode lock, stores into a mapping do
// not (decode_file's single output file).  The blocks are reserved first
// (fallocate), so a full disk is an error here and never a SIGBUS later;
// where a file cannot be reserved or mapped the caller keeps the pwrite
// path.  (For encode_file's shard files, measured: mapping them was slower
// than pwritev per shard -- 5.5 vs 6.4 GB/s for k4 r2 on tmpfs -- page
// faults cost more than the per-file write serialisation.)
struct FileMap {
    std::uint8_t* p = nullptr;
    std::size_t n = 0;
    FileMap() = default;
    FileMap(const FileMap&) = delete;
    FileMap& operator=(const FileMap&) = delete;
    ~FileMap() {
        if (p) ::munmap(p, n);
    }
    bool map(int fd, std::uint64_t bytes) {
        if (bytes == 0 || ::fallocate(fd, 0, 0, static_cast<off_t>(bytes)) != 0) return false;
        void* m = ::mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
        if (m == MAP_FAILED) return false;
        p = static_cast<std::uint8_t*>(m);
        n = bytes;
        return true;
    }
};

// ---- per-device staging: pinned host + device buffers, one stream per stage

constexpr int kStages = 3;

struct Stage {
    cudaStream_t stream = nullptr;
    std::uint8_t *h_in = nullptr, *h_out = nullptr, *d_in = nullptr, *d_out = nullptr;
    std::size_t in_cap = 0, out_cap = 0;
};

struct FileCtx {
    std::mutex mu;
    Stage st[kStages];
};

std::mutex g_ctx_mu;
std::map<int, std::unique_ptr<FileCtx>> g_ctx;

FileCtx& ctx_for(int device) {
    std::lock_guard<std::mutex> lk(g_ctx_mu);
    auto& c = g_ctx[device];
    if (!c) c = std::make_unique<FileCtx>();
    return *c;
}

void reserve(Stage& s, std::size_t in_bytes, std::size_t out_bytes) {
    if (!s.stream) check_cuda(cudaStreamCreateWithFlags(&s.stream, cudaStreamNonBlocking), "stream");
    if (s.in_cap < in_bytes) {
        if (s.h_in) check_cuda(cudaFreeHost(s.h_in), "cudaFreeHost");
        if (s.d_in) check_cuda(cudaFree(s.d_in), "cudaFree");
        s.h_in = s.d_in = nullptr;
        s.in_cap = 0;
        check_cuda(cudaHostAlloc(reinterpret_cast<void**>(&s.h_in), in_bytes, cudaHostAllocDefault), "pinned alloc");
        check_cuda(cudaMalloc(reinterpret_cast<void**>(&s.d_in), in_bytes), "device alloc");
        s.in_cap = in_bytes;
    }
    if (s.out_cap < out_bytes) {
        if (s.h_out) check_cuda(cudaFreeHost(s.h_out), "cudaFreeHost");
        if (s.d_out) check_cuda(cudaFree(s.d_out), "cudaFree");
        s.h_out = s.d_out = nullptr;
        s.out_cap = 0;
        check_cuda(cudaHostAlloc(reinterpret_cast<void**>(&s.h_out), out_bytes, cudaHostAllocDefault), "pinned alloc");
        check_cuda(cudaMalloc(reinterpret_cast<void**>(&s.d_out), out_bytes), "device alloc");
        s.out_cap = out_bytes;
    }
}

// stripes per pipeline chunk: ~64 MiB of source (or the whole file)
std::uint64_t batch_stripes(std::uint64_t stripe_bytes, std::uint64_t stripes) {
    const std::uint64_t chunk = g_file_chunk ? g_file_chunk : (std::uint64_t(64) << 20);
    return std::max<std::uint64_t>(1, std::min(stripes, chunk / stripe_bytes));
}

void validate_geometry(std::uint32_t k, std::uint32_t r, const Field& f, std::uint32_t symbol_size) {
    validate_field(f);
    if (k == 0) raise(Errc::InvalidArgument, "k must be at least 1"); // matrix.hpp:25-26
    if (std::uint64_t(k) + r > f.field_size()) raise(Errc::TooManySymbols, "k + r exceeds field size");
    if (symbol_size == 0 || symbol_size % f.w != 0 || symbol_size % 8 != 0) // container.hpp:171-172
        raise(Errc::BufferShape, "symbol size must be a positive multiple of w and of 8");
}

} // namespace

// ---- header --------------------------------------------------------------

std::uint32_t crc32(const std::uint8_t* bytes, std::size_t len) {
    static const auto table = [] {
        std::vector<std::uint32_t> t(256);
        for (std::uint32_t i = 0; i < 256; ++i) {
            std::uint32_t c = i;
            for (int b = 0; b < 8; ++b) c = (c >> 1) ^ ((c & 1u) ? 0xEDB88320u : 0u);
            t[i] = c;
        }
        return t;
    }();
    std::uint32_t c = 0xFFFFFFFFu;
    for (std::size_t i = 0; i < len; ++i) c = (c >> 8) ^ table[(c ^ bytes[i]) & 0xFFu];
    return c ^ 0xFFFFFFFFu;
}

bool ShardHeader::same_set(const ShardHeader& o) const {
    return version == o.version && field == o.field && transform == o.transform && k == o.k && r == o.r &&
           symbol_size == o.symbol_size && original_length == o.original_length;
}

std::uint64_t ShardHeader::stripe_count() const {
    const std::uint64_t stripe_bytes = std::uint64_t{k} * symbol_size;
    return stripe_bytes == 0 ? 0 : (original_length + stripe_bytes - 1) / stripe_bytes;
}

namespace {
const Field kFields[] = {
    Field{4, 5, FieldKind::Aop, 1, 4, 0x1F},       // 0: gf16_aop (field.hpp:38-40)
    Field{6, 9, FieldKind::Esp, 3, 2, 0x49},       // 1: gf64_esp (field.hpp:41-43)
    Field{8, 17, FieldKind::Aop, 1, 8, 0x139},     // 2: GF(2^8) in R_{2,17}
    Field{10, 11, FieldKind::Aop, 1, 10, 0x7FF},   // 3: GF(2^10) AOP
    Field{12, 13, FieldKind::Aop, 1, 12, 0x1FFF},  // 4: GF(2^12) AOP
};
} // namespace

std::uint8_t field_id(const Field& f) {
    for (std::uint8_t i = 0; i < sizeof kFields / sizeof kFields[0]; ++i)
        if (kFields[i] == f) return i;
    raise(Errc::InvalidArgument, "field has no shard-header id");
}

Field field_from_id(std::uint8_t id) {
    if (id < sizeof kFields / sizeof kFields[0]) return kFields[id];
    raise(Errc::BadHeader, "unknown field id " + std::to_string(id)); // field.hpp:58-62
}

void serialize_header(const ShardHeader& h, std::uint8_t out[kHeaderSize]) {
    std::memcpy(out, kMagic, 4);
    out[4] = h.version;
    out[5] = h.field;
    out[6] = h.transform;
    put16(out + 7, h.k);
    put16(out + 9, h.r);
    put16(out + 11, h.shard_index);
    put32(out + 13, h.symbol_size);
    put64(out + 17, h.original_length);
    put32(out + 25, crc32(out, 25));
}

// Strict parse in the reference's order: magic and version, then the
// checksum, then field semantics (container.hpp:132-161).
ShardHeader parse_header(const std::uint8_t* bytes, std::size_t len) {
    if (len < kHeaderSize) raise(Errc::BadHeader, "header truncated");
    if (std::memcmp(bytes, kMagic, 4) != 0) raise(Errc::BadHeader, "bad magic");
    if (bytes[4] != 1) raise(Errc::BadHeader, "unsupported version " + std::to_string(bytes[4]));
    if (get32(bytes + 25) != crc32(bytes, 25)) raise(Errc::ChecksumError, "header checksum mismatch");
    ShardHeader h;
    h.version = bytes[4];
    h.field = bytes[5];
    h.transform = bytes[6];
    h.k = get16(bytes + 7);
    h.r = get16(bytes + 9);
    h.shard_index = get16(bytes + 11);
    h.symbol_size = get32(bytes + 13);
    h.original_length = get64(bytes + 17);
    const Field f = field_from_id(h.field);
    if (h.transform > 1) raise(Errc::BadHeader, "unknown transform id " + std::to_string(h.transform)); // transform.hpp:26-29
    if (h.k == 0) raise(Errc::BadHeader, "k must be at least 1");
    if (static_cast<std::uint32_t>(h.k) + h.r > f.field_size()) raise(Errc::BadHeader, "k + r exceeds field size");
    if (h.shard_index >= static_cast<std::uint32_t>(h.k) + h.r) raise(Errc::BadHeader, "shard index out of range");
    if (h.symbol_size == 0 || h.symbol_size % f.w != 0 || h.symbol_size % 8 != 0)
        raise(Errc::BadHeader, "symbol size not a positive multiple of w and word width");
    return h;
}

std::string shard_path(const std::string& input, const std::string& out_dir, unsigned index) {
    char suffix[16];
    std::snprintf(suffix, sizeof suffix, ".s%03u", index);
    return (std::filesystem::path(out_dir) /
            (std::filesystem::path(input).filename().string() + suffix + ".pyrit"))
        .string();
}

void set_file_chunk(std::uint64_t bytes) { g_file_chunk = bytes; }

// ---- encode_file -----------------------------------------------------------
//
// Per chunk of B stripes (stripe = k symbols, file order): pread into a
// pinned stage, one H2D copy, ONE batched kernel launch that writes the r
// parity symbols of all B stripes straight into shard order (parity i of
// stripe b at out_i + b * symbol_size), one D2H copy; a writer task then
// gathers the data symbols (pwritev) and the parity runs into the shard
// files.  Stages rotate over three streams, so reading chunk c+1, the
// GPU work of chunk c and the writes of chunk c-1 overlap.

std::vector<std::string> encode_file(const std::string& input, const std::string& out_dir, std::uint32_t k,
                                     std::uint32_t r, const Field& f, TransformKind kind,
                                     std::uint32_t symbol_size, int device) {
    validate_geometry(k, r, f, symbol_size);
    const std::uint8_t fid = field_id(f);
    Fd in(::open(input.c_str(), O_RDONLY | O_CLOEXEC));
    if (in.fd < 0) raise(Errc::IoError, "cannot open " + input);
    struct stat sb{};
    if (::fstat(in.fd, &sb) != 0) raise(Errc::IoError, "cannot stat " + input);
    const std::uint64_t length = static_cast<std::uint64_t>(sb.st_size);
    std::error_code ec;
    std::filesystem::create_directories(out_dir, ec);

    const std::uint32_t total = k + r;
    std::vector<std::string> paths(total);
    std::vector<Fd> out(total);
    for (std::uint32_t i = 0; i < total; ++i) {
        paths[i] = shard_path(input, out_dir, i);
        out[i] = Fd(::open(paths[i].c_str(), O_WRONLY | O_CREAT | O_TRUNC | O_CLOEXEC, 0644));
        if (out[i].fd < 0) raise(Errc::IoError, "cannot create " + paths[i]);
        ShardHeader h;
        h.field = fid;
        h.transform = static_cast<std::uint8_t>(kind);
        h.k = static_cast<std::uint16_t>(k);
        h.r = static_cast<std::uint16_t>(r);
        h.shard_index = static_cast<std::uint16_t>(i);
        h.symbol_size = symbol_size;
        h.original_length = length;
        std::uint8_t hb[kHeaderSize];
        serialize_header(h, hb);
        pwrite_full(out[i].fd, hb, kHeaderSize, 0, paths[i]);
    }

    const std::uint64_t ss = symbol_size, stripe_bytes = std::uint64_t(k) * ss;
    const std::uint64_t stripes = length == 0 ? 0 : (length + stripe_bytes - 1) / stripe_bytes;
    if (stripes == 0) return paths;
    CodeParams cp{k, r, f, kind};
    std::shared_ptr<const Program> prog = r ? encode_program(cp) : nullptr;
    const std::uint64_t B = batch_stripes(stripe_bytes, stripes);

    FileCtx& ctx = ctx_for(device);
    std::lock_guard<std::mutex> lk(ctx.mu);
    check_cuda(cudaSetDevice(device), "cudaSetDevice");
    for (Stage& s : ctx.st) reserve(s, B * stripe_bytes, std::max<std::uint64_t>(B * r * ss, 1));
    std::future<void> pending[kStages];
    std::vector<const std::uint8_t*> din(k);
    std::vector<std::uint8_t*> dout(r);
    for (std::uint64_t s0 = 0, c = 0; s0 < stripes; s0 += B, ++c) {
        Stage& st = ctx.st[c % kStages];
        if (pending[c % kStages].valid()) pending[c % kStages].get();
        const std::uint64_t nb = std::min(B, stripes - s0);
        const std::uint64_t bytes = nb * stripe_bytes, at = s0 * stripe_bytes;
        const std::size_t got = pread_parallel(in.fd, st.h_in, static_cast<std::size_t>(std::min(bytes, length - at)),
                                               at, input);
        std::memset(st.h_in + got, 0, static_cast<std::size_t>(bytes - got)); // container.hpp:209-211
        if (prog) {
            check_cuda(cudaMemcpyAsync(st.d_in, st.h_in, bytes, cudaMemcpyHostToDevice, st.stream), "H2D");
            for (std::uint32_t j = 0; j < k; ++j) din[j] = st.d_in + j * ss;
            for (std::uint32_t i = 0; i < r; ++i) dout[i] = st.d_out + i * nb * ss;
            launch_batch(*prog, din.data(), dout.data(), ss / f.w, 0, ss / f.w, nb, stripe_bytes, ss, st.stream);
            check_cuda(cudaMemcpyAsync(st.h_out, st.d_out, nb * r * ss, cudaMemcpyDeviceToHost, st.stream), "D2H");
        }
        pending[c % kStages] = std::async(std::launch::async, [&, s0, nb, sp = &st] {
            check_cuda(cudaSetDevice(device), "cudaSetDevice");
            check_cuda(cudaStreamSynchronize(sp->stream), "cudaStreamSynchronize");
            const std::uint64_t at_shard = kHeaderSize + s0 * ss;
            host_pool().run(total, [&](std::size_t i) { // one shard file per task
                if (i < k) {
                    std::vector<iovec> iov(nb);
                    for (std::uint64_t b = 0; b < nb; ++b) iov[b] = {sp->h_in + b * stripe_bytes + i * ss, ss};
                    pwritev_full(out[i].fd, iov, at_shard, paths[i]);
                } else {
                    pwrite_full(out[i].fd, sp->h_out + (i - k) * nb * ss, nb * ss, at_shard, paths[i]);
                }
            });
        });
    }
    for (auto& p : pending)
        if (p.valid()) p.get();
    return paths;
}

// ---- decode_file -----------------------------------------------------------
//
// Validation follows the reference exactly (load each shard: header, then
// payload length; then set consistency; first occurrence of an index wins;
// at least k distinct shards).  The k survivors are taken lowest index
// first (codec.hpp:257-259) and only the erased DATA symbols are rebuilt --
// the output file holds data symbols only (container.hpp:291-296) -- by one
// batched launch per chunk that reads each survivor byte once.

void decode_file(const std::vector<std::string>& shard_paths, const std::string& output, int device) {
    if (shard_paths.empty()) raise(Errc::InsufficientShards, "no shards given");
    struct Loaded {
        ShardHeader h;
        Fd fd;
        std::string path;
        bool present = false;
    };
    std::vector<Loaded> byindex;
    ShardHeader ref;
    bool have_ref = false;
    for (const std::string& p : shard_paths) {
        Fd fd(::open(p.c_str(), O_RDONLY | O_CLOEXEC));
        if (fd.fd < 0) raise(Errc::IoError, "cannot open " + p);
        struct stat sb{};
        if (::fstat(fd.fd, &sb) != 0) raise(Errc::IoError, "cannot stat " + p);
        std::uint8_t hb[kHeaderSize];
        const std::size_t got = pread_full(fd.fd, hb, kHeaderSize, 0, p);
        const ShardHeader h = parse_header(hb, got);
        const std::uint64_t expect = h.stripe_count() * h.symbol_size;
        if (static_cast<std::uint64_t>(sb.st_size) != kHeaderSize + expect)
            raise(Errc::BadHeader, "shard payload truncated: " + p);
        if (!have_ref) {
            ref = h;
            have_ref = true;
            byindex.resize(static_cast<std::size_t>(ref.k) + ref.r);
        } else if (!h.same_set(ref)) {
            raise(Errc::HeaderMismatch, "shard from a different set: " + p);
        }
        Loaded& slot = byindex[h.shard_index];
        if (!slot.present) {
            slot.h = h;
            slot.fd = std::move(fd);
            slot.path = p;
            slot.present = true;
        }
    }
    const std::uint32_t k = ref.k, r = ref.r;
    const Field f = field_from_id(ref.field);
    std::vector<std::uint32_t> erased;
    for (std::uint32_t i = 0; i < k + r; ++i)
        if (!byindex[i].present) erased.push_back(i);
    if (k + r - erased.size() < k)
        raise(Errc::InsufficientShards,
              "have " + std::to_string(k + r - erased.size()) + " shards, need " + std::to_string(k));

    Fd out(::open(output.c_str(), O_RDWR | O_CREAT | O_TRUNC | O_CLOEXEC, 0644));
    if (out.fd < 0) raise(Errc::IoError, "cannot create " + output);
    // the output is one file: concurrent write() calls would serialise on its
    // inode lock, so the workers copy into a shared mapping instead (falls
    // back to pwritev where the file cannot be mapped)
    FileMap map;
    map.map(out.fd, ref.original_length);

    const std::uint64_t stripes = ref.stripe_count(), ss = ref.symbol_size, length = ref.original_length;
    const std::uint64_t stripe_bytes = std::uint64_t(k) * ss;
    if (stripes == 0) return;
    CodeParams cp{k, r, f, static_cast<TransformKind>(ref.transform)};
    const DecodeProgram dp = decode_program(cp, erased, /*data_only=*/true);
    // survivors (lowest index first) and where data symbol j comes from
    std::vector<std::uint32_t> surv = dp.repair.survivors;
    if (!dp.prog) { // no data erased: the data shards are the survivors
        surv.clear();
        for (std::uint32_t j = 0; j < k; ++j) surv.push_back(j);
    }
    std::vector<std::int64_t> from_in(k, -1), from_out(k, -1);
    for (std::size_t i = 0; i < surv.size(); ++i)
        if (surv[i] < k) from_in[surv[i]] = static_cast<std::int64_t>(i);
    for (std::size_t e = 0; e < dp.repair.outputs.size(); ++e) from_out[dp.repair.outputs[e]] = static_cast<std::int64_t>(e);
    const std::uint32_t ne = static_cast<std::uint32_t>(dp.repair.outputs.size());
    const std::uint64_t B = batch_stripes(stripe_bytes, stripes);

    FileCtx& ctx = ctx_for(device);
    std::lock_guard<std::mutex> lk(ctx.mu);
    check_cuda(cudaSetDevice(device), "cudaSetDevice");
    for (Stage& s : ctx.st) reserve(s, B * stripe_bytes, std::max<std::uint64_t>(B * ne * ss, 1));
    std::future<void> pending[kStages];
    std::vector<const std::uint8_t*> din(k);
    std::vector<std::uint8_t*> dout(ne);
    for (std::uint64_t s0 = 0, c = 0; s0 < stripes; s0 += B, ++c) {
        Stage& st = ctx.st[c % kStages];
        if (pending[c % kStages].valid()) pending[c % kStages].get();
        const std::uint64_t nb = std::min(B, stripes - s0);
        // survivor-major staging: survivor i's nb symbols are contiguous
        host_pool().run(surv.size(), [&](std::size_t i) {
            const Loaded& L = byindex[surv[i]];
            const std::size_t want = static_cast<std::size_t>(nb * ss);
            if (pread_full(L.fd.fd, st.h_in + i * nb * ss, want, kHeaderSize + s0 * ss, L.path) != want)
                raise(Errc::IoError, "short read on " + L.path);
        });
        if (dp.prog) {
            check_cuda(cudaMemcpyAsync(st.d_in, st.h_in, k * nb * ss, cudaMemcpyHostToDevice, st.stream), "H2D");
            for (std::uint32_t i = 0; i < k; ++i) din[i] = st.d_in + i * nb * ss;
            for (std::uint32_t e = 0; e < ne; ++e) dout[e] = st.d_out + e * nb * ss;
            launch_batch(*dp.prog, din.data(), dout.data(), ss / f.w, 0, ss / f.w, nb, ss, ss, st.stream);
            check_cuda(cudaMemcpyAsync(st.h_out, st.d_out, ne * nb * ss, cudaMemcpyDeviceToHost, st.stream), "D2H");
        }
        pending[c % kStages] = std::async(std::launch::async, [&, s0, nb, sp = &st] {
            check_cuda(cudaSetDevice(device), "cudaSetDevice");
            check_cuda(cudaStreamSynchronize(sp->stream), "cudaStreamSynchronize");
            // the output range of this chunk, written by several tasks (runs of stripes)
            const std::uint64_t pieces = std::min<std::uint64_t>(nb, 16);
            host_pool().run(pieces, [&](std::size_t q) {
                const std::uint64_t b0 = nb * q / pieces, b1 = nb * (q + 1) / pieces;
                const std::uint64_t at = (s0 + b0) * stripe_bytes;
                if (at >= length) return;
                std::vector<iovec> iov;
                iov.reserve((b1 - b0) * k);
                std::uint64_t remaining = std::min(length - at, (b1 - b0) * stripe_bytes);
                for (std::uint64_t b = b0; b < b1 && remaining; ++b)
                    for (std::uint32_t j = 0; j < k && remaining; ++j) {
                        const std::uint64_t take = std::min<std::uint64_t>(ss, remaining);
                        std::uint8_t* src = from_in[j] >= 0 ? sp->h_in + (from_in[j] * nb + b) * ss
                                                            : sp->h_out + (from_out[j] * nb + b) * ss;
                        iov.push_back({src, static_cast<std::size_t>(take)});
                        remaining -= take;
                    }
                if (map.p) {
                    std::uint64_t pos = at;
                    for (const iovec& v : iov) {
                        std::memcpy(map.p + pos, v.iov_base, v.iov_len);
                        pos += v.iov_len;
                    }
                } else {
                    pwritev_full(out.fd, iov, at, output);
                }
            });
        });
    }
    for (auto& p : pending)
        if (p.valid()) p.get();
}

} // namespace pyrit_b200
