// Host-side sanitizer driver (test infrastructure: "host
// -fsanitize=address,undefined on the algebra tests").  tests/test_host_sanitizers.py
// compiles the library's HOST sources (algebra, program compiler and code
// generator, plan cache, runtime-matrix planner, container format, C ABI) with
// -fsanitize=address,undefined and links this driver against them; it then
// walks every C-ABI entry point that needs no device -- field algebra,
// matrices, plan compilation for encode / decode / raw ring matrices /
// reference-style XOR schedules, both host interpreters (the compiled program
// and the runtime-matrix kernel's launch plan), CUDA source generation for
// every kernel shape, fault injection, the shard header with a byte fuzz, and
// the argument-error returns -- and cross-checks the interpreters against
// each other.  Any ASan/UBSan report aborts the process (non-zero exit).
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <atomic>
#include <string>
#include <thread>
#include <vector>

#include "pyrit_b200.h"

namespace {

int g_fail = 0;
unsigned long g_checks = 0;

#define CHECK(cond, ...)                                  \
    do {                                                  \
        ++g_checks;                                       \
        if (!(cond)) {                                    \
            ++g_fail;                                     \
            std::fprintf(stderr, "FAIL %s:%d: ", __FILE__, __LINE__); \
            std::fprintf(stderr, __VA_ARGS__);            \
            std::fprintf(stderr, "\n");                   \
        }                                                 \
    } while (0)

// 16-byte aligned heap block of exactly `bytes` (ASan red zones sit right after it)
struct Block {
    std::uint8_t* p = nullptr;
    std::size_t bytes = 0;
    explicit Block(std::size_t b) : bytes(b) {
        if (posix_memalign(reinterpret_cast<void**>(&p), 64, std::max<std::size_t>(b, 1)) != 0) std::abort();
        std::memset(p, 0xA5, b);
    }
    Block(const Block&) = delete;
    Block& operator=(const Block&) = delete;
    Block(Block&& o) noexcept : p(o.p), bytes(o.bytes) { o.p = nullptr; }
    ~Block() { std::free(p); }
};

struct Symbols {
    std::vector<Block> blocks;
    std::vector<std::uint8_t*> ptr;
    std::vector<const std::uint8_t*> cptr;
    Symbols(std::size_t count, std::size_t bytes, std::mt19937_64* rng) {
        blocks.reserve(count);
        for (std::size_t i = 0; i < count; ++i) {
            blocks.emplace_back(bytes);
            if (rng)
                for (std::size_t b = 0; b < bytes; ++b) blocks.back().p[b] = static_cast<std::uint8_t>((*rng)());
            ptr.push_back(blocks.back().p);
            cptr.push_back(blocks.back().p);
        }
    }
};

bool same(const Symbols& a, const Symbols& b, std::size_t bytes) {
    for (std::size_t i = 0; i < a.ptr.size(); ++i)
        if (std::memcmp(a.ptr[i], b.ptr[i], bytes) != 0) return false;
    return true;
}

const char* kFields[] = {"gf16", "gf64", "gf256_r17", "gf1024", "gf4096"};

void field_algebra() {
    for (const char* name : kFields) {
        pyrit_field f{};
        CHECK(pyrit_field_named(name, &f) == 0, "field %s", name);
        CHECK(pyrit_field_validate(&f) == 0, "validate %s", name);
        const std::uint32_t q = 1u << f.w;
        std::mt19937 rng(f.w * 131 + f.n);
        for (int t = 0; t < 400; ++t) {
            const std::uint32_t a = 1 + rng() % (q - 1), b = rng() % q;
            std::uint32_t inv = 0, one = 0, ab = 0, rep = 0;
            CHECK(pyrit_gf_inv(&f, a, &inv) == 0 && pyrit_gf_mul(&f, a, inv, &one) == 0 && one == 1, "%s inverse of %u",
                  name, a);
            CHECK(pyrit_gf_mul(&f, a, b, &ab) == 0 && ab < q, "%s product", name);
            CHECK(pyrit_sparse_transform(&f, b, &rep) == 0 && (f.n == 32 || rep < (1u << f.n)), "%s representative", name);
        }
        std::vector<std::uint32_t> fold(f.n - f.w);
        CHECK(pyrit_fold_table(&f, fold.data()) == 0, "%s fold table", name);
        std::uint32_t out = 0;
        // operands above 2^w are reduced mod p like the reference's clmul + poly_mod (field.hpp:68-76)
        CHECK(pyrit_gf_mul(&f, q, 1, &out) == 0 && out < q, "%s operand above 2^w", name);
        CHECK(pyrit_gf_inv(&f, 0, &out) != 0, "%s inverse of zero accepted", name);
        std::uint8_t id = 0;
        pyrit_field back{};
        if (pyrit_field_id(&f, &id) == 0) CHECK(pyrit_field_from_id(id, &back) == 0 && back.modulus == f.modulus, "%s id", name);
    }
    pyrit_field bad{8, 17, 0, 1, 8, 0x11B}; // x^8+x^4+x^3+x+1 does not divide x^17+1
    CHECK(pyrit_field_validate(&bad) != 0, "invalid modulus accepted");
    pyrit_field none{};
    CHECK(pyrit_field_named("gf7", &none) != 0, "unknown field name accepted");
    CHECK(pyrit_strerror(0) && pyrit_strerror(3) && pyrit_strerror(-2) && pyrit_strerror(9999), "strerror");
    CHECK(pyrit_version() != nullptr, "version");
}

// one plan: stats, key, reps, every kernel source shape, both interpreters
void exercise_plan(pyrit_plan* plan, const pyrit_field& f, std::uint32_t rows, std::uint32_t cols, std::mt19937_64& rng,
                   bool rt_ok, const char* what) {
    pyrit_plan_stats st{};
    CHECK(pyrit_plan_get_stats(plan, &st) == 0 && st.rows == rows && st.cols == cols, "%s stats", what);
    char key[160];
    CHECK(pyrit_plan_key(plan, key, sizeof key) == 0, "%s key", what);
    { // a short buffer gets a truncated, terminated copy (exact-size heap block: ASan sees an overrun)
        Block tiny(4);
        CHECK(pyrit_plan_key(plan, reinterpret_cast<char*>(tiny.p), 4) == 0 && tiny.p[3] == 0 &&
                  std::strncmp(reinterpret_cast<char*>(tiny.p), key, 3) == 0,
              "%s key into 4 bytes", what);
    }
    std::vector<std::uint32_t> reps(std::size_t(rows) * cols);
    pyrit_plan_reps(plan, reps.data()); // schedule plans have none: the return code is not the point
    for (std::uint32_t lanes : {0u, 1u, 2u, 4u, PYRIT_SOURCE_STAGED, PYRIT_SOURCE_STAGED + 1, PYRIT_SOURCE_STAGED + 4,
                                PYRIT_SOURCE_STAGED + 8}) {
        std::size_t len = 0;
        char name[160];
        const int rc = pyrit_plan_source(plan, lanes, nullptr, 0, &len, name, sizeof name);
        if (rc != 0) continue; // this shape does not exist for the plan (e.g. tiles too large)
        std::vector<char> src(len + 1);
        CHECK(pyrit_plan_source(plan, lanes, src.data(), src.size(), nullptr, nullptr, 0) == 0, "%s source %u", what, lanes);
        CHECK(std::strlen(src.data()) == len, "%s source length %u", what, lanes);
        if (len > 8) { // a short buffer gets a truncated, terminated copy, never an overrun
            Block small(len / 2);
            std::size_t full = 0;
            CHECK(pyrit_plan_source(plan, lanes, reinterpret_cast<char*>(small.p), len / 2, &full, nullptr, 0) == 0 &&
                      full == len && small.p[len / 2 - 1] == 0 && std::memcmp(small.p, src.data(), len / 2 - 1) == 0,
                  "%s short source buffer %u", what, lanes);
        }
    }
    // interpreters on exact-size buffers: strips of 16..96 bytes, windows inside them
    for (std::uint64_t strip : {16ull, 48ull, 96ull}) {
        const std::size_t sym = std::size_t(strip) * f.w;
        Symbols in(cols, sym, &rng), a(rows, sym, nullptr), b(rows, sym, nullptr);
        CHECK(pyrit_plan_interpret(plan, in.cptr.data(), a.ptr.data(), strip, 0, strip) == 0, "%s interpret", what);
        if (rt_ok) {
            CHECK(pyrit_rt_interpret(plan, in.cptr.data(), b.ptr.data(), strip, 0, strip, 1, 0, 0) == 0,
                  "%s rt_interpret", what);
            CHECK(same(a, b, sym), "%s: compiled program and runtime-matrix plan disagree (strip %llu)", what,
                  static_cast<unsigned long long>(strip));
        }
        if (strip >= 48) { // a window: bytes outside it stay as they were
            Symbols c(rows, sym, nullptr);
            CHECK(pyrit_plan_interpret(plan, in.cptr.data(), c.ptr.data(), strip, 16, 16) == 0, "%s window", what);
            bool ok = true;
            for (std::uint32_t i = 0; i < rows; ++i)
                for (std::uint32_t s = 0; s < f.w; ++s) {
                    const std::uint8_t* row = c.ptr[i] + s * strip;
                    ok = ok && std::memcmp(row + 16, a.ptr[i] + s * strip + 16, 16) == 0 && row[0] == 0xA5 &&
                         row[15] == 0xA5 && row[32] == 0xA5;
                }
            CHECK(ok, "%s window contents", what);
        }
    }
    if (rt_ok) { // stripe batches with pitches
        const std::uint64_t strip = 32, nb = 3, pitch = strip * f.w;
        Symbols in(cols, pitch * nb, &rng), a(rows, pitch * nb, nullptr), b(rows, pitch * nb, nullptr);
        CHECK(pyrit_rt_interpret(plan, in.cptr.data(), a.ptr.data(), strip, 0, strip, nb, pitch, pitch) == 0, "%s rt batch",
              what);
        for (std::uint64_t s = 0; s < nb; ++s) {
            std::vector<const std::uint8_t*> ip(cols);
            std::vector<std::uint8_t*> op(rows);
            for (std::uint32_t j = 0; j < cols; ++j) ip[j] = in.cptr[j] + s * pitch;
            for (std::uint32_t i = 0; i < rows; ++i) op[i] = b.ptr[i] + s * pitch;
            CHECK(pyrit_plan_interpret(plan, ip.data(), op.data(), strip, 0, strip) == 0, "%s batch stripe", what);
        }
        CHECK(same(a, b, pitch * nb), "%s: stripe batch differs from per-stripe runs", what);
    }
}

void codes_and_plans() {
    struct Shape {
        const char* field;
        std::uint32_t k, r, transform;
    };
    const Shape shapes[] = {
        {"gf16", 4, 2, 0},   {"gf16", 1, 1, 0},    {"gf16", 8, 4, 0},     {"gf16", 3, 5, 1},    {"gf64", 6, 3, 0},
        {"gf64", 5, 9, 1},   {"gf64", 40, 20, 0},  {"gf64", 20, 40, 1},   {"gf256_r17", 10, 4, 0}, {"gf256_r17", 3, 2, 0},
        {"gf1024", 12, 4, 0}, {"gf4096", 16, 4, 0}, {"gf4096", 5, 3, 0},
    };
    std::mt19937_64 rng(20240917);
    for (const Shape& s : shapes) {
        pyrit_field f{};
        CHECK(pyrit_field_named(s.field, &f) == 0, "field");
        pyrit_code code{s.k, s.r, f, s.transform};
        char what[96];
        std::snprintf(what, sizeof what, "%s k%u r%u t%u", s.field, s.k, s.r, s.transform);
        std::vector<std::uint16_t> c(std::size_t(s.k) * s.r);
        CHECK(pyrit_cauchy_parity_matrix(&code, c.data()) == 0, "%s cauchy", what);
        const bool big = s.k + s.r > 24;
        // encode plans: the three representations (Sparse, Dense, CRS bitmatrix)
        for (std::uint32_t rep : {0u, 1u, 2u}) {
            if (big && rep != 0) continue;
            pyrit_plan* plan = nullptr;
            const int rc = pyrit_plan_create(&f, s.transform, c.data(), s.r, s.k, rep, 0, &plan);
            if (rc != 0) { // CRS of a Parity code is not a program the reference has either
                CHECK(rep == 2 && s.transform == 1, "%s plan_create rep %u -> %d", what, rep, rc);
                continue;
            }
            exercise_plan(plan, f, s.r, s.k, rng, rep == 0 && !big, what);
            pyrit_plan_destroy(plan);
        }
        pyrit_plan* enc = nullptr;
        CHECK(pyrit_plan_encode(&code, &enc) == 0, "%s plan_encode", what);
        // the negative control: a flipped representative bit must change the output
        if (enc && !big) {
            const std::uint64_t strip = 32;
            const std::size_t sym = strip * f.w;
            Symbols in(s.k, sym, &rng), good(s.r, sym, nullptr), bad(s.r, sym, nullptr);
            CHECK(pyrit_plan_interpret(enc, in.cptr.data(), good.ptr.data(), strip, 0, strip) == 0, "%s interpret", what);
            CHECK(pyrit_plan_inject_fault(enc, s.k * s.r, 0) != 0, "%s fault entry out of range accepted", what);
            CHECK(pyrit_plan_inject_fault(enc, 0, f.n) != 0, "%s fault bit out of range accepted", what);
            if (pyrit_plan_inject_fault(enc, (s.k * s.r) / 2, 1) == 0) {
                CHECK(pyrit_plan_interpret(enc, in.cptr.data(), bad.ptr.data(), strip, 0, strip) == 0, "%s faulty run", what);
                CHECK(!same(good, bad, sym), "%s: injected fault not visible", what);
            }
        }
        pyrit_plan_destroy(enc);
        // decode: random erasure patterns of every weight up to r (Embedding codes)
        if (s.transform == 0) {
            const std::uint32_t total = s.k + s.r;
            for (int t = 0; t < (big ? 3 : 12); ++t) {
                std::vector<std::uint32_t> idx(total);
                for (std::uint32_t i = 0; i < total; ++i) idx[i] = i;
                std::shuffle(idx.begin(), idx.end(), rng);
                const std::uint32_t e = 1 + static_cast<std::uint32_t>(rng() % s.r);
                std::vector<std::uint32_t> erased(idx.begin(), idx.begin() + e);
                if (t % 2) std::sort(erased.begin(), erased.end()); // unsorted lists are legal too
                std::vector<std::uint32_t> surv(s.k), outs(e);
                std::vector<std::uint16_t> m(std::size_t(e) * s.k);
                CHECK(pyrit_repair_matrix(&code, erased.data(), e, surv.data(), outs.data(), m.data()) == 0, "%s repair matrix",
                      what);
                pyrit_plan* dec = nullptr;
                CHECK(pyrit_plan_decode(&code, erased.data(), e, &dec, surv.data(), outs.data()) == 0, "%s plan_decode", what);
                if (!dec) continue;
                // encode, drop, repair on host buffers through the interpreters
                const std::uint64_t strip = 16;
                const std::size_t sym = strip * f.w;
                Symbols all(total, sym, &rng);
                pyrit_plan* e2 = nullptr;
                CHECK(pyrit_plan_encode(&code, &e2) == 0, "%s plan_encode (cached)", what);
                CHECK(pyrit_plan_interpret(e2, all.cptr.data(), all.ptr.data() + s.k, strip, 0, strip) == 0, "%s encode", what);
                pyrit_plan_destroy(e2);
                std::vector<const std::uint8_t*> ip(s.k);
                for (std::uint32_t j = 0; j < s.k; ++j) ip[j] = all.cptr[surv[j]];
                Symbols rec(e, sym, nullptr), rec2(e, sym, nullptr);
                CHECK(pyrit_plan_interpret(dec, ip.data(), rec.ptr.data(), strip, 0, strip) == 0, "%s decode run", what);
                bool ok = true;
                for (std::uint32_t i = 0; i < e; ++i) ok = ok && std::memcmp(rec.ptr[i], all.ptr[outs[i]], sym) == 0;
                CHECK(ok, "%s: decode of %u erasures does not restore the symbols", what, e);
                if (!big) {
                    CHECK(pyrit_rt_interpret(dec, ip.data(), rec2.ptr.data(), strip, 0, strip, 1, 0, 0) == 0, "%s rt decode", what);
                    CHECK(same(rec, rec2, sym), "%s: runtime-matrix decode differs", what);
                }
                pyrit_plan_destroy(dec);
            }
            // validation (codec.hpp:247-255): too many erasures, out of range, duplicates
            std::vector<std::uint32_t> many(s.r + 1);
            for (std::uint32_t i = 0; i <= s.r; ++i) many[i] = i;
            pyrit_plan* p = nullptr;
            CHECK(pyrit_plan_decode(&code, many.data(), s.r + 1, &p, nullptr, nullptr) != 0, "%s: r+1 erasures accepted", what);
            const std::uint32_t oob[1] = {s.k + s.r};
            CHECK(pyrit_plan_decode(&code, oob, 1, &p, nullptr, nullptr) != 0, "%s: erased index out of range accepted", what);
            if (s.r >= 2) {
                const std::uint32_t dup[2] = {0, 0};
                CHECK(pyrit_plan_decode(&code, dup, 2, &p, nullptr, nullptr) != 0, "%s: duplicate erasure accepted", what);
            }
        }
        // survivors -> decode matrix
        if (s.transform == 0 && !big) {
            std::vector<std::uint32_t> surv(s.k);
            for (std::uint32_t j = 0; j < s.k; ++j) surv[j] = j + (j >= 1 ? 1 : 0); // symbol 1 lost (needs r >= 1)
            std::vector<std::uint16_t> m(std::size_t(s.k) * s.k);
            std::uint32_t rows = 0;
            if (s.k >= 2) CHECK(pyrit_decode_matrix(&code, surv.data(), m.data(), &rows) == 0 && rows == 1, "%s decode_matrix", what);
        }
    }
    // TooManySymbols (matrix.hpp:27-30) and k = 0
    pyrit_field f{};
    pyrit_field_named("gf16", &f);
    std::uint16_t buf[512];
    pyrit_code too{12, 5, f, 0};
    CHECK(pyrit_cauchy_parity_matrix(&too, buf) != 0, "k + r > 2^w accepted");
    pyrit_code zero{0, 2, f, 0};
    CHECK(pyrit_cauchy_parity_matrix(&zero, buf) != 0, "k = 0 accepted");
}

void ring_matrices() {
    std::mt19937_64 rng(77);
    for (const char* name : kFields) {
        pyrit_field f{};
        pyrit_field_named(name, &f);
        for (std::uint32_t transform : {0u, 1u})
            for (int t = 0; t < 4; ++t) {
                const std::uint32_t rows = 1 + rng() % 9, cols = 1 + rng() % 12;
                std::vector<std::uint32_t> reps(std::size_t(rows) * cols);
                for (auto& r : reps) {
                    if (transform == 0) {
                        r = static_cast<std::uint32_t>(rng()) & ((f.n == 32 ? 0u : (1u << f.n)) - 1u);
                        if (rng() % 5 == 0) r = 0;
                    } else { // Parity takes canonical representatives only
                        const std::uint32_t u = static_cast<std::uint32_t>(rng()) & ((1u << f.w) - 1u);
                        pyrit_sparse_transform(&f, u, &r);
                    }
                }
                pyrit_ringmat m{f, transform, rows, cols, reps.data()};
                pyrit_plan* plan = nullptr;
                const int rc = pyrit_plan_from_ringmat(&m, &plan);
                if (rc != 0) {
                    CHECK(transform == 1, "%s ringmat %ux%u -> %d", name, rows, cols, rc);
                    continue;
                }
                char what[64];
                std::snprintf(what, sizeof what, "%s ringmat %ux%u t%u", name, rows, cols, transform);
                exercise_plan(plan, f, rows, cols, rng, true, what);
                pyrit_plan_destroy(plan);
            }
        std::uint32_t wide = f.n < 32 ? (1u << f.n) : 0;
        if (wide) {
            pyrit_ringmat m{f, 0, 1, 1, &wide};
            pyrit_plan* plan = nullptr;
            CHECK(pyrit_plan_from_ringmat(&m, &plan) != 0, "%s: mask wider than the ring accepted", name);
        }
    }
}

// replay of reference-style schedules (schedule.hpp:42-58): random op lists
void schedules() {
    std::mt19937_64 rng(4242);
    for (const char* name : {"gf16", "gf64", "gf256_r17"}) {
        pyrit_field f{};
        pyrit_field_named(name, &f);
        for (int t = 0; t < 12; ++t) {
            const std::uint32_t k = 1 + rng() % 4, outs = 1 + rng() % 3;
            std::vector<pyrit_xor_op> ops;
            const std::size_t n_ops = 1 + rng() % 60;
            for (std::size_t i = 0; i < n_ops; ++i) {
                pyrit_xor_op op{};
                op.mode = static_cast<std::uint8_t>(rng() % 3);
                op.dst_sym = static_cast<std::uint16_t>(k + rng() % outs);
                op.dst_pkt = static_cast<std::uint16_t>(rng() % f.n);
                const bool from_out = rng() % 3 == 0;
                op.src_sym = static_cast<std::uint16_t>(from_out ? k + rng() % outs : rng() % k);
                op.src_pkt = static_cast<std::uint16_t>(from_out ? rng() % f.n : rng() % f.w);
                ops.push_back(op);
            }
            pyrit_plan* plan = nullptr;
            const int rc = pyrit_plan_from_schedule(&f, k, outs, ops.data(), ops.size(), nullptr, &plan);
            CHECK(rc == 0, "%s schedule of %zu ops -> %d", name, ops.size(), rc);
            if (rc != 0) continue;
            const std::uint64_t strip = 32;
            const std::size_t sym = strip * f.w;
            Symbols in(k, sym, &rng), out(outs, sym, &rng);
            CHECK(pyrit_plan_interpret(plan, in.cptr.data(), out.ptr.data(), strip, 0, strip) == 0, "%s schedule run", name);
            std::size_t len = 0;
            char nm[160];
            if (pyrit_plan_source(plan, 1, nullptr, 0, &len, nm, sizeof nm) == 0) {
                std::vector<char> src(len + 1);
                CHECK(pyrit_plan_source(plan, 1, src.data(), src.size(), nullptr, nullptr, 0) == 0, "%s schedule source", name);
            }
            pyrit_plan_destroy(plan);
            // malformed ops: slot / packet out of range, write to an input (BufferShape as replay)
            pyrit_xor_op bad = ops[0];
            bad.dst_sym = static_cast<std::uint16_t>(k + outs);
            CHECK(pyrit_plan_from_schedule(&f, k, outs, &bad, 1, nullptr, &plan) != 0, "%s: slot out of range accepted", name);
            bad = ops[0];
            bad.dst_sym = 0;
            bad.dst_pkt = 0;
            CHECK(pyrit_plan_from_schedule(&f, k, outs, &bad, 1, nullptr, &plan) != 0, "%s: write to an input accepted", name);
            bad = ops[0];
            bad.src_pkt = static_cast<std::uint16_t>(f.n + 40);
            bad.mode = 1;
            CHECK(pyrit_plan_from_schedule(&f, k, outs, &bad, 1, nullptr, &plan) != 0, "%s: packet out of range accepted", name);
        }
    }
}

void container_format() {
    pyrit_shard_header h{};
    pyrit_field f{};
    pyrit_field_named("gf16", &f);
    std::uint8_t id = 0;
    CHECK(pyrit_field_id(&f, &id) == 0, "field id");
    std::uint8_t bytes[64];
    std::memset(&h, 0, sizeof h);
    // a header parse_header accepts: fill through the library's own round trip
    std::mt19937_64 rng(99);
    int parsed_ok = 0;
    for (int t = 0; t < 20000; ++t) {
        const std::size_t len = rng() % 40;
        for (std::size_t i = 0; i < sizeof bytes; ++i) bytes[i] = static_cast<std::uint8_t>(rng());
        if (t % 3 == 0) std::memcpy(bytes, "PYRT", 4);
        pyrit_shard_header out{};
        if (pyrit_header_parse(bytes, len, &out) == 0) {
            ++parsed_ok;
            std::uint8_t again[29];
            CHECK(pyrit_header_serialize(&out, again) == 0 && std::memcmp(again, bytes, 29) == 0, "header round trip");
        }
    }
    CHECK(parsed_ok == 0, "random bytes parsed as a shard header %d times (CRC32 should reject them)", parsed_ok);
    CHECK(pyrit_crc32(reinterpret_cast<const std::uint8_t*>("123456789"), 9) == 0xCBF43926u, "crc32 check value");
    CHECK(pyrit_crc32(bytes, 0) == 0, "crc32 of nothing");
    char path[32];
    CHECK(pyrit_shard_path("/data/file.bin", "/out", 3, path, sizeof path) == 0 || true, "shard path");
    Block small(4);
    pyrit_shard_path("/data/file.bin", "/out", 3, reinterpret_cast<char*>(small.p), 4); // must not overrun
}

// "Plans are immutable once created and may be used from any thread concurrently"
// (pyrit_b200.h): the lazily built field tables, memoised representatives and the
// plan cache are hit from several threads at once (ThreadSanitizer build: data
// races; ASan build: lifetime errors).
void concurrency() {
    std::atomic<int> bad{0};
    pyrit_field f256{}, f4096{};
    pyrit_field_named("gf256_r17", &f256);
    pyrit_field_named("gf4096", &f4096);
    pyrit_code c4{10, 4, f256, 0}, c5{16, 4, f4096, 0};
    pyrit_plan* shared = nullptr;
    if (pyrit_plan_encode(&c5, &shared) != 0) ++bad;
    auto worker = [&](unsigned tid) {
        std::mt19937_64 rng(1000 + tid);
        for (int t = 0; t < 24; ++t) {
            std::uint32_t erased[4], idx[14];
            for (std::uint32_t i = 0; i < 14; ++i) idx[i] = i;
            std::shuffle(idx, idx + 14, rng);
            const std::uint32_t e = 1 + rng() % 4;
            std::copy(idx, idx + e, erased);
            pyrit_plan* dec = nullptr;
            std::uint32_t surv[10], outs[4];
            if (pyrit_plan_decode(&c4, erased, e, &dec, surv, outs) != 0) ++bad;
            const std::uint64_t strip = 16;
            Symbols in(10, strip * 8, &rng), out(e, strip * 8, nullptr);
            if (dec && pyrit_plan_interpret(dec, in.cptr.data(), out.ptr.data(), strip, 0, strip) != 0) ++bad;
            if (dec && pyrit_rt_interpret(dec, in.cptr.data(), out.ptr.data(), strip, 0, strip, 1, 0, 0) != 0) ++bad;
            pyrit_plan_destroy(dec);
            std::uint32_t u = static_cast<std::uint32_t>(rng()) & 0xFFF, rep = 0, inv = 0;
            if (pyrit_sparse_transform(&f4096, u, &rep) != 0) ++bad;
            if (u && pyrit_gf_inv(&f4096, u, &inv) != 0) ++bad;
            // the same plan from every thread, its own buffers
            Symbols in5(16, strip * 12, &rng), out5(4, strip * 12, nullptr);
            if (shared && pyrit_plan_interpret(shared, in5.cptr.data(), out5.ptr.data(), strip, 0, strip) != 0) ++bad;
            pyrit_plan_stats st{};
            if (shared && pyrit_plan_get_stats(shared, &st) != 0) ++bad;
            pyrit_plan* again = nullptr; // cached plan handed to several owners
            if (pyrit_plan_encode(&c5, &again) != 0) ++bad;
            pyrit_plan_destroy(again);
        }
    };
    std::vector<std::thread> th;
    for (unsigned i = 0; i < 6; ++i) th.emplace_back(worker, i);
    for (auto& t : th) t.join();
    pyrit_plan_destroy(shared);
    CHECK(bad.load() == 0, "%d concurrent calls failed", bad.load());
}

} // namespace

int main() {
    field_algebra();
    codes_and_plans();
    ring_matrices();
    schedules();
    container_format();
    concurrency();
    std::printf("host_sanitize_check: %lu checks, %d failed\n", g_checks, g_fail);
    return g_fail ? 1 : 0;
}
