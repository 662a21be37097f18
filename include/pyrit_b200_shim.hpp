// pyrit_b200_shim.hpp -- drop-in GPU replacements for the reference codec's
// top-level calls, written against the reference's OWN types.
//
//   pyrit::encode(data, code, threads)          codec.hpp:212-220
//     -> pyrit::cuda::encode(data, code, device)
//   pyrit::decode(symbols, erased, code, threads) codec.hpp:241-284
//     -> pyrit::cuda::decode(symbols, erased, code, device)
//   pyrit::encode_file(input, out_dir, code, symbol_size) container.hpp:168-222
//     -> pyrit::cuda::encode_file(input, out_dir, code, symbol_size, device)
//   pyrit::decode_file(shard_paths, output)      container.hpp:249-299
//     -> pyrit::cuda::decode_file(shard_paths, output, device)
//
// Include after the reference headers (it needs SymbolBuffer, CodeSpec,
// Error from proj/include/pyrit/) and link libpyrit_b200.so.  Validation and
// error behaviour follow the reference: shape errors throw pyrit::Error with
// the same Errc (BufferShape, InvalidArgument, InsufficientShards,
// TooManySymbols); device failures throw std::runtime_error.  Results are
// byte-identical to the reference's embedding-transform encode/decode (and,
// for fields the reference cannot represent, e.g. GF(2^8) in R_{2,17}, to its
// field oracle oracle_apply / encode_crs).
#pragma once

#include <filesystem>
#include <stdexcept>
#include <string>
#include <vector>

#include "pyrit/codec.hpp"
#include "pyrit_b200.h"

namespace pyrit::cuda {

inline pyrit_code to_c(const CodeSpec& code) {
    pyrit_code c{};
    c.k = code.k;
    c.r = code.r;
    c.field.w = code.field.w;
    c.field.n = code.field.n;
    c.field.kind = code.field.kind == FieldKind::Esp ? 1u : 0u;
    c.field.s = code.field.s;
    c.field.r_esp = code.field.r_esp;
    c.field.modulus = code.field.modulus;
    c.transform = static_cast<std::uint32_t>(code.transform);
    return c;
}

// 1 + Errc -> pyrit::Error (errors.hpp:12-39); negative -> device failure
inline void check(int rc) {
    if (rc == 0) return;
    if (rc >= 1 && rc <= 11) throw Error(static_cast<Errc>(rc - 1), pyrit_strerror(rc));
    throw std::runtime_error(std::string("pyrit_b200: ") + pyrit_strerror(rc));
}

// codec.hpp:212 encode(): parity = C * data, on the GPU (host buffers in,
// host buffers out; H2D, fused ring kernel and D2H are pipelined inside).
inline SymbolBuffer encode(const SymbolBuffer& data, const CodeSpec& code, int device = 0) {
    check_data_shape(data, code); // codec.hpp:205-209, the reference's own validation
    SymbolBuffer parity(code.r, data.symbol_size(), code.field);
    const pyrit_code c = to_c(code);
    if (code.r) check(pyrit_encode_host(&c, data.symbol(0), parity.symbol(0), data.symbol_size(), device));
    return parity;
}

// codec.hpp:223 encode_crs(): the bitmatrix baseline codec on the GPU, same
// parity bytes as encode() (host buffers, like encode above).
inline SymbolBuffer encode_crs(const SymbolBuffer& data, const CodeSpec& code, int device = 0) {
    check_data_shape(data, code);
    SymbolBuffer parity(code.r, data.symbol_size(), code.field);
    const pyrit_code c = to_c(code);
    if (code.r) check(pyrit_encode_crs_host(&c, data.symbol(0), parity.symbol(0), data.symbol_size(), device));
    return parity;
}

// codec.hpp:241 decode(): in-place repair of the listed symbols from any k
// survivors (lowest index first), one fused pass on the GPU.
inline void decode(SymbolBuffer& symbols, const std::vector<unsigned>& erased, const CodeSpec& code,
                   int device = 0) {
    validate_code(code);
    if (!(symbols.spec() == code.field) || symbols.symbols() != code.k + code.r)
        raise(Errc::BufferShape, "symbol buffer does not match the code");
    const pyrit_code c = to_c(code);
    std::vector<std::uint32_t> er(erased.begin(), erased.end());
    check(pyrit_decode_host(&c, symbols.symbol(0), er.data(), static_cast<std::uint32_t>(er.size()),
                            symbols.symbol_size(), device));
}

// container.hpp:168 encode_file(): same shard files (names, 29-byte headers,
// stripe layout) as the reference; stripes go through the GPU in batches.
inline std::vector<std::filesystem::path> encode_file(const std::filesystem::path& input,
                                                      const std::filesystem::path& out_dir, const CodeSpec& code,
                                                      std::uint32_t symbol_size, int device = 0) {
    const pyrit_code c = to_c(code);
    check(pyrit_encode_file(&c, input.c_str(), out_dir.c_str(), symbol_size, device));
    std::vector<std::filesystem::path> paths;
    char buf[4096];
    for (unsigned i = 0; i < code.k + code.r; ++i) {
        check(pyrit_shard_path(input.c_str(), out_dir.c_str(), i, buf, sizeof buf));
        paths.emplace_back(buf);
    }
    return paths;
}

// container.hpp:249 decode_file(): rebuild the original file from any k shards.
inline void decode_file(const std::vector<std::filesystem::path>& shard_paths, const std::filesystem::path& output,
                        int device = 0) {
    std::vector<const char*> ps;
    for (const auto& p : shard_paths) ps.push_back(p.c_str());
    check(pyrit_decode_file(ps.data(), static_cast<std::uint32_t>(ps.size()), output.c_str(), device));
}

} // namespace pyrit::cuda
