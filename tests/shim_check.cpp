// shim_check.cpp -- TEST INFRASTRUCTURE: exercises include/pyrit_b200_shim.hpp
// exactly the way a reference user would (reference SymbolBuffer/CodeSpec,
// reference encode()/decode() beside the GPU versions).  Built by
// oracle/Makefile (target `shim`) against the unmodified reference headers
// into oracle/_ref/shim_check; run on a GPU box by tests/test_gpu_shim.py.
#include <cstdio>
#include <cstring>
#include <random>

#include <fstream>

#include "pyrit/codec.hpp"
#include "pyrit/container.hpp"
#include "pyrit_b200_shim.hpp"

using namespace pyrit;

static bool same(const SymbolBuffer& a, const SymbolBuffer& b) {
    return a.symbols() == b.symbols() && a.symbol_size() == b.symbol_size() &&
           std::memcmp(a.symbol(0), b.symbol(0), a.symbols() * a.symbol_size()) == 0;
}

static void fill(SymbolBuffer& buf, std::uint64_t seed) {
    std::mt19937_64 rng(seed);
    for (unsigned s = 0; s < buf.symbols(); ++s)
        for (std::size_t i = 0; i < buf.symbol_size(); ++i) buf.symbol(s)[i] = static_cast<std::uint8_t>(rng());
}

int main() {
    int failures = 0;
    struct Case {
        const char* name;
        FieldSpec f;
        unsigned k, r;
        std::size_t symbol_size;
        bool ring_ok; // the reference's own ring encode() is valid for this field
    };
    const Case cases[] = {
        {"gf16 k4 r2 (BASELINE config 1 shape)", FieldSpec::gf16_aop(), 4, 2, 4 * 4096, true},
        {"gf64 esp k6 r3", FieldSpec::gf64_esp(), 6, 3, 24 * 1000, true},
        {"gf1024 k12 r4 (config 3 shape)", FieldSpec{10, 11, FieldKind::Aop, 1, 10, 0x7FF}, 12, 4, 160 * 512, true},
        {"gf4096 k16 r4 (config 5 shape)", FieldSpec{12, 13, FieldKind::Aop, 1, 12, 0x1FFF}, 16, 4, 192 * 512, true},
        {"gf256/R17 k10 r4 (configs 2/4)", FieldSpec{8, 17, FieldKind::Aop, 1, 8, 0x139}, 10, 4, 8 * 8192, false},
    };
    for (const Case& c : cases) {
        const CodeSpec code{c.k, c.r, c.f, TransformKind::Embedding};
        SymbolBuffer data(c.k, c.symbol_size, c.f);
        fill(data, c.k * 1000 + c.r);
        const SymbolBuffer want = c.ring_ok ? encode(data, code, 4) : encode_crs(data, code, 4);
        const SymbolBuffer got = pyrit::cuda::encode(data, code);
        // the reference's own argument lists: (data, code, threads) -- threads is a host-thread count,
        // not a device; and an explicit device
        const bool enc_ok = same(got, want) && same(pyrit::cuda::encode_crs(data, code), want) &&
                            same(pyrit::cuda::encode(data, code, 4u), want) &&
                            same(pyrit::cuda::encode(data, code, pyrit::cuda::Device{0}), want);
        // decode: erase r symbols (data and parity mixed), repair in place
        SymbolBuffer full(c.k + c.r, c.symbol_size, c.f);
        std::memcpy(full.symbol(0), data.symbol(0), c.k * c.symbol_size);
        std::memcpy(full.symbol(c.k), want.symbol(0), c.r * c.symbol_size);
        SymbolBuffer work = full;
        std::vector<unsigned> erased;
        for (unsigned i = 0; i < c.r; ++i) erased.push_back((i * 5 + 1) % (c.k + c.r));
        for (unsigned e : erased) std::memset(work.symbol(e), 0xAA, c.symbol_size);
        pyrit::cuda::decode(work, erased, code, 8u);
        const bool dec_ok = same(work, full);
        std::printf("%-40s encode %s decode %s\n", c.name, enc_ok ? "OK" : "MISMATCH", dec_ok ? "OK" : "MISMATCH");
        failures += !enc_ok + !dec_ok;
    }
    // operator level: the reference's own schedules replayed by pyrit::cuda::parallel_replay
    {
        struct SCase {
            const char* name;
            FieldSpec f;
            unsigned k, r;
            TransformKind kind;
            int which; // 0 sparse ring, 1 dense ring, 2 CRS
        };
        const SCase sc[] = {
            {"gf16 k4 r2 sparse", FieldSpec::gf16_aop(), 4, 2, TransformKind::Embedding, 0},
            {"gf16 k4 r2 dense", FieldSpec::gf16_aop(), 4, 2, TransformKind::Embedding, 1},
            {"gf64 k5 r3 crs", FieldSpec::gf64_esp(), 5, 3, TransformKind::Embedding, 2},
            {"gf64 k3 r5 parity", FieldSpec::gf64_esp(), 3, 5, TransformKind::Parity, 0},
            {"gf4096 k16 r4 sparse", FieldSpec{12, 13, FieldKind::Aop, 1, 12, 0x1FFF}, 16, 4, TransformKind::Embedding, 0},
        };
        for (const SCase& c : sc) {
            const CodeSpec code{c.k, c.r, c.f, c.kind};
            const FieldMatrix m = cauchy_parity_matrix(code);
            const XorSchedule sched = c.which == 2 ? compile_crs_schedule(m)
                                                   : compile_schedule(m, c.kind, c.which ? RingRep::Dense : RingRep::Sparse);
            const std::size_t ss = std::size_t(c.f.w) * 8 * 777;
            SymbolBuffer in(c.k + 2, ss, c.f);
            fill(in, 77 + c.k);
            std::vector<unsigned> in_map, out_map;
            for (unsigned j = 0; j < c.k; ++j) in_map.push_back(c.k + 1 - j); // a permutation into k + 2 symbols
            for (unsigned i = 0; i < c.r; ++i) out_map.push_back(c.r - 1 - i);
            SymbolBuffer want(c.r, ss, c.f), got(c.r, ss, c.f);
            fill(want, 9);
            std::memcpy(got.symbol(0), want.symbol(0), c.r * ss);
            parallel_replay(sched, in, in_map, want, out_map, 4);
            pyrit::cuda::parallel_replay(sched, in, in_map, got, out_map, 4u);
            bool ok = same(got, want);
            // window only (replay) and in place in one buffer, decode()-style
            SymbolBuffer both(c.k + c.r, ss, c.f), both_ref(c.k + c.r, ss, c.f);
            fill(both, 5);
            std::memcpy(both_ref.symbol(0), both.symbol(0), (c.k + c.r) * ss);
            std::vector<unsigned> im(c.k), om(c.r);
            for (unsigned j = 0; j < c.k; ++j) im[j] = j;
            for (unsigned i = 0; i < c.r; ++i) om[i] = c.k + i;
            Workspace ws(sched, 64);
            replay(sched, both_ref, im, both_ref, om, ws, 128, 64);
            Workspace ws_gpu(sched, 64);
            pyrit::cuda::replay(sched, both, im, both, om, ws_gpu, 128, 64); // codec.hpp:118 argument list
            ok = ok && same(both, both_ref);
            std::printf("parallel_replay %-28s %s\n", c.name, ok ? "OK" : "MISMATCH");
            failures += !ok;
        }
    }
    // error behaviour mirrors the reference
    try {
        const CodeSpec code{4, 2, FieldSpec::gf16_aop(), TransformKind::Embedding};
        SymbolBuffer full(6, 16, FieldSpec::gf16_aop());
        pyrit::cuda::decode(full, {0, 1, 2}, code);
        std::printf("InsufficientShards not raised\n");
        ++failures;
    } catch (const Error& e) {
        std::printf("decode 3 erasures with r=2 -> Errc %d (%s)\n", static_cast<int>(e.code()), e.what());
        failures += e.code() != Errc::InsufficientShards;
    }
    // file codec: reference encode_file vs the GPU's, decoded crosswise
    {
        namespace fs = std::filesystem;
        const fs::path dir = fs::temp_directory_path() / ("pyrit_shim_" + std::to_string(std::random_device{}()));
        fs::create_directories(dir);
        std::vector<std::uint8_t> payload(123457);
        std::mt19937_64 rng(5);
        for (auto& b : payload) b = static_cast<std::uint8_t>(rng());
        std::ofstream(dir / "in.bin", std::ios::binary)
            .write(reinterpret_cast<const char*>(payload.data()), static_cast<std::streamsize>(payload.size()));
        auto slurp = [](const fs::path& p) {
            std::ifstream in(p, std::ios::binary);
            return std::vector<std::uint8_t>(std::istreambuf_iterator<char>(in), {});
        };
        const CodeSpec fcodes[] = {{4, 2, FieldSpec::gf16_aop(), TransformKind::Embedding},
                                   {3, 6, FieldSpec::gf64_esp(), TransformKind::Parity}};
        for (const CodeSpec& code : fcodes) {
            const std::uint32_t ss = code.field.w == 4 ? 128 : 48;
            const auto ref = encode_file(dir / "in.bin", dir / "ref", code, ss);
            const auto gpu = pyrit::cuda::encode_file(dir / "in.bin", dir / "gpu", code, ss);
            bool same_files = ref.size() == gpu.size();
            for (std::size_t i = 0; same_files && i < ref.size(); ++i) same_files = slurp(ref[i]) == slurp(gpu[i]);
            std::vector<fs::path> surv(gpu.begin() + code.r, gpu.end());
            decode_file(surv, dir / "ref_out.bin"); // reference decodes GPU shards
            std::vector<fs::path> surv_ref(ref.begin() + 1, ref.begin() + 1 + code.k);
            pyrit::cuda::decode_file(surv_ref, dir / "gpu_out.bin"); // GPU decodes reference shards
            const bool rt = slurp(dir / "ref_out.bin") == payload && slurp(dir / "gpu_out.bin") == payload;
            std::printf("encode_file/decode_file w=%u k%u r%u: shards %s, round trips %s\n", code.field.w, code.k,
                        code.r, same_files ? "IDENTICAL" : "DIFFER", rt ? "OK" : "MISMATCH");
            failures += !same_files + !rt;
        }
        fs::remove_all(dir);
    }
    std::printf(failures ? "SHIM CHECK FAILED\n" : "SHIM CHECK PASSED\n");
    return failures ? 1 : 0;
}
