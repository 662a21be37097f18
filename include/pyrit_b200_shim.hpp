// pyrit_b200_shim.hpp -- drop-in GPU replacements for the reference codec's
// top-level calls, written against the reference's OWN types.
//
//   pyrit::encode(data, code, threads)          codec.hpp:212-220
//     -> pyrit::cuda::encode(data, code, threads)   (or (data, code, Device{id}))
//   pyrit::decode(symbols, erased, code, threads) codec.hpp:241-284
//     -> pyrit::cuda::decode(symbols, erased, code, threads)
//   pyrit::encode_file(input, out_dir, code, symbol_size) container.hpp:168-222
//     -> pyrit::cuda::encode_file(input, out_dir, code, symbol_size)
//   pyrit::decode_file(shard_paths, output)      container.hpp:249-299
//     -> pyrit::cuda::decode_file(shard_paths, output)
//   pyrit::parallel_replay(sched, in, in_map, out, out_map, threads)  codec.hpp:176-193
//     -> pyrit::cuda::parallel_replay(sched, in, in_map, out, out_map, threads)
//   pyrit::replay(sched, in, in_map, out, out_map, ws, offset, len)   codec.hpp:118-157
//     -> pyrit::cuda::replay(sched, in, in_map, out, out_map, ws, offset, len)
// Same arguments with the same meaning: switching is a namespace change.  The
// device is pyrit::cuda::set_device(id) (default 0) or a trailing Device{id}.
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

#include <algorithm>
#include <cstddef>
#include <filesystem>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "pyrit/codec.hpp"
#include "pyrit_b200.h"

namespace pyrit::cuda {

// Device selection.  The drop-ins keep the reference's signatures exactly --
// including the trailing `unsigned threads` of encode/decode/parallel_replay,
// which the GPU path accepts and ignores -- so the device comes from
// set_device() (per host thread, default 0) or from an explicit Device{id}
// argument in the overloads that take one.
struct Device {
    int id = 0;
};
inline int& current_device() {
    static thread_local int d = 0;
    return d;
}
inline void set_device(int id) { current_device() = id; }

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
inline SymbolBuffer encode(const SymbolBuffer& data, const CodeSpec& code, Device device) {
    check_data_shape(data, code); // codec.hpp:205-209, the reference's own validation
    SymbolBuffer parity(code.r, data.symbol_size(), code.field);
    const pyrit_code c = to_c(code);
    if (code.r) check(pyrit_encode_host(&c, data.symbol(0), parity.symbol(0), data.symbol_size(), device.id));
    return parity;
}
inline SymbolBuffer encode(const SymbolBuffer& data, const CodeSpec& code, unsigned /*threads*/ = 1) {
    return encode(data, code, Device{current_device()});
}

// codec.hpp:223 encode_crs(): the bitmatrix baseline codec on the GPU, same
// parity bytes as encode() (host buffers, like encode above).
inline SymbolBuffer encode_crs(const SymbolBuffer& data, const CodeSpec& code, Device device) {
    check_data_shape(data, code);
    SymbolBuffer parity(code.r, data.symbol_size(), code.field);
    const pyrit_code c = to_c(code);
    if (code.r) check(pyrit_encode_crs_host(&c, data.symbol(0), parity.symbol(0), data.symbol_size(), device.id));
    return parity;
}
inline SymbolBuffer encode_crs(const SymbolBuffer& data, const CodeSpec& code, unsigned /*threads*/ = 1) {
    return encode_crs(data, code, Device{current_device()});
}

// codec.hpp:241 decode(): in-place repair of the listed symbols from any k
// survivors (lowest index first), one fused pass on the GPU.
inline void decode(SymbolBuffer& symbols, const std::vector<unsigned>& erased, const CodeSpec& code,
                   Device device) {
    validate_code(code);
    if (!(symbols.spec() == code.field) || symbols.symbols() != code.k + code.r)
        raise(Errc::BufferShape, "symbol buffer does not match the code");
    const pyrit_code c = to_c(code);
    std::vector<std::uint32_t> er(erased.begin(), erased.end());
    check(pyrit_decode_host(&c, symbols.symbol(0), er.data(), static_cast<std::uint32_t>(er.size()),
                            symbols.symbol_size(), device.id));
}
inline void decode(SymbolBuffer& symbols, const std::vector<unsigned>& erased, const CodeSpec& code,
                   unsigned /*threads*/ = 1) {
    decode(symbols, erased, code, Device{current_device()});
}

// container.hpp:168 encode_file(): same shard files (names, 29-byte headers,
// stripe layout) as the reference; stripes go through the GPU in batches.
inline std::vector<std::filesystem::path> encode_file(const std::filesystem::path& input,
                                                      const std::filesystem::path& out_dir, const CodeSpec& code,
                                                      std::uint32_t symbol_size, Device device = Device{current_device()}) {
    const pyrit_code c = to_c(code);
    check(pyrit_encode_file(&c, input.c_str(), out_dir.c_str(), symbol_size, device.id));
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
                        Device device = Device{current_device()}) {
    std::vector<const char*> ps;
    for (const auto& p : shard_paths) ps.push_back(p.c_str());
    check(pyrit_decode_file(ps.data(), static_cast<std::uint32_t>(ps.size()), output.c_str(), device.id));
}

// The operator level: any XorSchedule (compile_schedule, compile_crs_schedule
// or hand-built) compiled into one fused kernel and replayed over host
// SymbolBuffers (H2D, kernel, D2H inside).  The reference's XorOp is passed
// as is (same layout as pyrit_xor_op).  Scratch packets start zeroed, as the
// fresh Workspace of parallel_replay; slots that name the same symbol of
// the same buffer share storage, as in the reference's op-by-op replay.
static_assert(sizeof(XorOp) == sizeof(pyrit_xor_op) && offsetof(XorOp, mode) == offsetof(pyrit_xor_op, mode),
              "XorOp layout");

inline void replay(const XorSchedule& sched, const SymbolBuffer& in, std::span<const unsigned> in_map,
                   SymbolBuffer& out, std::span<const unsigned> out_map, std::size_t offset, std::size_t len,
                   Device device) {
    // codec.hpp:122-127, the reference's own checks
    if (in_map.size() != sched.k || out_map.size() != sched.outputs)
        raise(Errc::BufferShape, "replay: slot map sizes do not match schedule");
    if (!(in.spec() == sched.spec) || !(out.spec() == sched.spec)) raise(Errc::BufferShape, "replay: field mismatch");
    if (in.packet_size() != out.packet_size() || offset + len > in.packet_size())
        raise(Errc::BufferShape, "replay: column window out of range");
    for (unsigned j : in_map)
        if (j >= in.symbols()) raise(Errc::BufferShape, "replay: input slot maps outside the buffer");
    for (unsigned i : out_map)
        if (i >= out.symbols()) raise(Errc::BufferShape, "replay: output slot maps outside the buffer");
    std::vector<XorOp> ops(sched.pre);
    ops.insert(ops.end(), sched.core.begin(), sched.core.end());
    ops.insert(ops.end(), sched.post.begin(), sched.post.end());
    std::vector<const std::uint8_t*> ip;
    std::vector<std::uint8_t*> op;
    for (unsigned j : in_map) ip.push_back(in.symbol(j));
    for (unsigned i : out_map) op.push_back(out.symbol(i));
    std::vector<std::uint32_t> labels; // slots naming the same symbol share storage
    std::vector<const std::uint8_t*> addr(ip.begin(), ip.end());
    addr.insert(addr.end(), op.begin(), op.end());
    for (const std::uint8_t* a : addr)
        labels.push_back(static_cast<std::uint32_t>(std::find(addr.begin(), addr.end(), a) - addr.begin()));
    pyrit_field f{};
    f.w = sched.spec.w;
    f.n = sched.spec.n;
    f.kind = sched.spec.kind == FieldKind::Esp ? 1u : 0u;
    f.s = sched.spec.s;
    f.r_esp = sched.spec.r_esp;
    f.modulus = sched.spec.modulus;
    pyrit_plan* plan = nullptr;
    check(pyrit_plan_from_schedule(&f, sched.k, sched.outputs, reinterpret_cast<const pyrit_xor_op*>(ops.data()),
                                   ops.size(), labels.data(), &plan));
    const int rc = pyrit_apply_host(plan, ip.data(), op.data(), in.packet_size(), offset, len, device.id);
    pyrit_plan_destroy(plan);
    check(rc);
}

// codec.hpp:118 signature: the Workspace is accepted for drop-in compatibility;
// on the GPU the scratch packets live in registers and start at zero for every
// call (the reference's schedules never read scratch before writing it)
inline void replay(const XorSchedule& sched, const SymbolBuffer& in, std::span<const unsigned> in_map,
                   SymbolBuffer& out, std::span<const unsigned> out_map, Workspace& /*ws*/, std::size_t offset,
                   std::size_t len) {
    replay(sched, in, in_map, out, out_map, offset, len, Device{current_device()});
}

// codec.hpp:176 signature (threads: the reference's host threads, unused here)
inline void parallel_replay(const XorSchedule& sched, const SymbolBuffer& in, std::span<const unsigned> in_map,
                            SymbolBuffer& out, std::span<const unsigned> out_map, unsigned /*threads*/ = 1) {
    replay(sched, in, in_map, out, out_map, 0, in.packet_size(), Device{current_device()});
}
inline void parallel_replay(const XorSchedule& sched, const SymbolBuffer& in, std::span<const unsigned> in_map,
                            SymbolBuffer& out, std::span<const unsigned> out_map, Device device) {
    replay(sched, in, in_map, out, out_map, 0, in.packet_size(), device);
}

} // namespace pyrit::cuda
