// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// Exposes the UNMODIFIED reference library (header-only C++20, compiled in
// place from /root/reference/proj/include by oracle/Makefile; nothing is
// copied into this repository) through a small extern "C" surface so the
// Python tests can pin the C oracle against it and bench.py can time the
// reference's own CPU path.  Output: oracle/_ref/libpyrit_ref.so.
//
// Every function forwards to the reference symbol named in its comment;
// pyrit::Error is mapped to 1 + Errc (errors.hpp:12-24).
#include <cstdint>
#include <cstring>
#include <memory>
#include <vector>

#include "pyrit/bench.hpp"
#include "pyrit/codec.hpp"
#include "pyrit/container.hpp"
#include "pyrit/matrix.hpp"
#include "pyrit/schedule.hpp"

using namespace pyrit;

#define REF_EXPORT extern "C" __attribute__((visibility("default")))

namespace {

FieldSpec make_field(unsigned w, unsigned n, unsigned kind, unsigned s, unsigned r_esp,
                     std::uint32_t modulus) {
    return FieldSpec{w, n, kind ? FieldKind::Esp : FieldKind::Aop, s, r_esp, modulus};
}

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const Error& e) {
        return 1 + static_cast<int>(e.code());
    } catch (...) {
        return 100;
    }
}

FieldMatrix make_matrix(const FieldSpec& spec, unsigned rows, unsigned cols, const std::uint16_t* m) {
    FieldMatrix fm(rows, cols, spec);
    for (unsigned i = 0; i < rows * cols; ++i) fm.e[i] = m[i];
    return fm;
}

} // namespace

// field.hpp:68 gf_mul / :168 gf_inv
REF_EXPORT std::uint32_t ref_gf_mul(std::uint32_t a, std::uint32_t b, unsigned w, unsigned n,
                                    std::uint32_t modulus) {
    return gf_mul(static_cast<FieldElem>(a), static_cast<FieldElem>(b),
                  make_field(w, n, 0, 1, w, modulus));
}
REF_EXPORT std::uint32_t ref_gf_inv(std::uint32_t a, unsigned w, unsigned n, std::uint32_t modulus) {
    std::uint32_t out = 0;
    guarded([&] { out = gf_inv(static_cast<FieldElem>(a), make_field(w, n, 0, 1, w, modulus)); });
    return out;
}

// ring.hpp:24 ring_mul, :77 sparse_transform, transform.hpp:39 phi_E_inv
REF_EXPORT std::uint32_t ref_ring_mul(std::uint32_t a, std::uint32_t b, unsigned w, unsigned n,
                                      std::uint32_t modulus) {
    return ring_mul(static_cast<RingElem>(a), static_cast<RingElem>(b),
                    make_field(w, n, 0, 1, w, modulus));
}
REF_EXPORT std::uint32_t ref_sparse_transform(std::uint32_t u, unsigned w, unsigned n, unsigned kind,
                                              unsigned s, unsigned r_esp, std::uint32_t modulus) {
    return sparse_transform(static_cast<FieldElem>(u), make_field(w, n, kind, s, r_esp, modulus));
}
REF_EXPORT std::uint32_t ref_phi_E_inv(std::uint32_t a, unsigned w, unsigned n, unsigned kind,
                                       unsigned s, unsigned r_esp, std::uint32_t modulus) {
    return phi_E_inv(static_cast<RingElem>(a), make_field(w, n, kind, s, r_esp, modulus));
}

// matrix.hpp:54 cauchy_parity_matrix
REF_EXPORT int ref_cauchy(unsigned k, unsigned r, unsigned w, unsigned n, std::uint32_t modulus,
                          std::uint16_t* out) {
    return guarded([&] {
        const FieldMatrix c = cauchy_parity_matrix(k, r, make_field(w, n, 0, 1, w, modulus));
        std::memcpy(out, c.e.data(), c.e.size() * sizeof(std::uint16_t));
    });
}

// matrix.hpp:96 invert
REF_EXPORT int ref_invert(unsigned dim, unsigned w, unsigned n, std::uint32_t modulus,
                          const std::uint16_t* in, std::uint16_t* out) {
    return guarded([&] {
        const FieldMatrix inv = invert(make_matrix(make_field(w, n, 0, 1, w, modulus), dim, dim, in));
        std::memcpy(out, inv.e.data(), inv.e.size() * sizeof(std::uint16_t));
    });
}

// matrix.hpp:193 decode_matrix
REF_EXPORT int ref_decode_matrix(unsigned k, unsigned r, unsigned w, unsigned n, std::uint32_t modulus,
                                 const std::uint32_t* survivors, std::uint16_t* out,
                                 unsigned* rows_out) {
    return guarded([&] {
        const FieldSpec spec = make_field(w, n, 0, 1, w, modulus);
        const CodeSpec code{k, r, spec, TransformKind::Embedding};
        const FieldMatrix c = cauchy_parity_matrix(k, r, spec);
        std::vector<unsigned> surv(survivors, survivors + k);
        const FieldMatrix dm = decode_matrix(code, c, surv);
        std::memcpy(out, dm.e.data(), dm.e.size() * sizeof(std::uint16_t));
        *rows_out = static_cast<unsigned>(dm.rows);
    });
}

// schedule.hpp:94 compile_schedule / :168 compile_crs_schedule + :216 schedule_stats
// crs: 0 ring schedule (rep: 0 Sparse, 1 Dense), 1 CRS bitmatrix schedule.
// stats: [copy, xor, zero, total, matrix_ones, pre, core, post]
REF_EXPORT int ref_schedule_stats(unsigned w, unsigned n, unsigned kind, unsigned s, unsigned r_esp,
                                  std::uint32_t modulus, unsigned rows, unsigned cols,
                                  const std::uint16_t* m, unsigned transform, unsigned crs,
                                  unsigned rep, std::uint64_t* stats) {
    return guarded([&] {
        const FieldMatrix fm = make_matrix(make_field(w, n, kind, s, r_esp, modulus), rows, cols, m);
        const XorSchedule sched =
            crs ? compile_crs_schedule(fm)
                : compile_schedule(fm, static_cast<TransformKind>(transform),
                                   rep ? RingRep::Dense : RingRep::Sparse);
        const ScheduleStats st = schedule_stats(sched);
        stats[0] = st.copy_ops;
        stats[1] = st.xor_ops;
        stats[2] = st.zero_ops;
        stats[3] = st.total_region_ops;
        stats[4] = st.matrix_ones;
        stats[5] = sched.pre.size();
        stats[6] = sched.core.size();
        stats[7] = sched.post.size();
    });
}

// schedule.hpp:94 compile_schedule / :168 compile_crs_schedule: the op list
// itself (pre, core, post concatenated, XorOp layout); *n_ops = total, ops
// may be null (count only).  Returns BufferShape + 1 when cap is too small.
REF_EXPORT int ref_schedule_ops(unsigned w, unsigned n, unsigned kind, unsigned s, unsigned r_esp,
                                std::uint32_t modulus, unsigned rows, unsigned cols, const std::uint16_t* m,
                                unsigned transform, unsigned crs, unsigned rep, XorOp* ops, std::uint64_t cap,
                                std::uint64_t* n_ops) {
    return guarded([&] {
        const FieldMatrix fm = make_matrix(make_field(w, n, kind, s, r_esp, modulus), rows, cols, m);
        const XorSchedule sched =
            crs ? compile_crs_schedule(fm)
                : compile_schedule(fm, static_cast<TransformKind>(transform),
                                   rep ? RingRep::Dense : RingRep::Sparse);
        std::vector<XorOp> all(sched.pre);
        all.insert(all.end(), sched.core.begin(), sched.core.end());
        all.insert(all.end(), sched.post.begin(), sched.post.end());
        *n_ops = all.size();
        if (ops) {
            if (all.size() > cap) raise(Errc::BufferShape, "op buffer too small");
            std::memcpy(ops, all.data(), all.size() * sizeof(XorOp));
        }
    });
}

// codec.hpp:176 parallel_replay of an arbitrary op list (all in core).
// in: n_in symbols, out: n_out symbols (symbol_size bytes each, contiguous);
// same_buffer: in and out are ONE SymbolBuffer (decode()'s in-place replay),
// held in `out` (n_out symbols).
REF_EXPORT int ref_replay_ops(unsigned w, unsigned n, unsigned kind, unsigned s, unsigned r_esp,
                              std::uint32_t modulus, unsigned k, unsigned outputs, const XorOp* ops,
                              std::uint64_t n_ops, const std::uint8_t* in, unsigned n_in, const unsigned* in_map,
                              std::uint8_t* out, unsigned n_out, const unsigned* out_map,
                              std::uint64_t symbol_size, unsigned same_buffer, unsigned threads) {
    return guarded([&] {
        const FieldSpec spec = make_field(w, n, kind, s, r_esp, modulus);
        XorSchedule sched;
        sched.spec = spec;
        sched.k = k;
        sched.outputs = outputs;
        sched.core.assign(ops, ops + n_ops);
        SymbolBuffer ob(n_out, symbol_size, spec);
        std::memcpy(ob.symbol(0), out, std::size_t(n_out) * symbol_size);
        const std::vector<unsigned> im(in_map, in_map + k), om(out_map, out_map + outputs);
        if (same_buffer) {
            parallel_replay(sched, ob, im, ob, om, threads);
        } else {
            SymbolBuffer ib(n_in, symbol_size, spec);
            std::memcpy(ib.symbol(0), in, std::size_t(n_in) * symbol_size);
            parallel_replay(sched, ib, im, ob, om, threads);
        }
        std::memcpy(out, ob.symbol(0), std::size_t(n_out) * symbol_size);
    });
}

// codec.hpp:444 oracle_apply over whole symbols (data: cols symbols contiguous)
REF_EXPORT int ref_oracle_apply(unsigned w, unsigned n, unsigned kind, unsigned s, unsigned r_esp,
                                std::uint32_t modulus, unsigned transform, unsigned rows,
                                unsigned cols, const std::uint16_t* m, const std::uint8_t* data,
                                std::uint64_t symbol_size, std::uint8_t* out) {
    return guarded([&] {
        const FieldSpec spec = make_field(w, n, kind, s, r_esp, modulus);
        SymbolBuffer in(cols, symbol_size, spec);
        std::memcpy(in.symbol(0), data, cols * symbol_size);
        const SymbolBuffer o = oracle_apply(make_matrix(spec, rows, cols, m),
                                            static_cast<TransformKind>(transform), in);
        std::memcpy(out, o.symbol(0), rows * symbol_size);
    });
}

// codec.hpp:212 encode (ring) and :480 encode_crs, whole symbols
REF_EXPORT int ref_encode(unsigned w, unsigned n, unsigned kind, unsigned s, unsigned r_esp,
                          std::uint32_t modulus, unsigned k, unsigned r, unsigned transform,
                          unsigned crs, const std::uint8_t* data, std::uint64_t symbol_size,
                          std::uint8_t* parity, unsigned threads) {
    return guarded([&] {
        const FieldSpec spec = make_field(w, n, kind, s, r_esp, modulus);
        const CodeSpec code{k, r, spec, static_cast<TransformKind>(transform)};
        SymbolBuffer in(k, symbol_size, spec);
        std::memcpy(in.symbol(0), data, k * symbol_size);
        const SymbolBuffer p = crs ? encode_crs(in, code, threads) : encode(in, code, threads);
        std::memcpy(parity, p.symbol(0), r * symbol_size);
    });
}

// codec.hpp:241 decode, in place over k + r contiguous symbols
REF_EXPORT int ref_decode(unsigned w, unsigned n, unsigned kind, unsigned s, unsigned r_esp,
                          std::uint32_t modulus, unsigned k, unsigned r, unsigned transform,
                          std::uint8_t* symbols, std::uint64_t symbol_size, const unsigned* erased,
                          unsigned n_erased, unsigned threads) {
    return guarded([&] {
        const FieldSpec spec = make_field(w, n, kind, s, r_esp, modulus);
        const CodeSpec code{k, r, spec, static_cast<TransformKind>(transform)};
        SymbolBuffer buf(k + r, symbol_size, spec);
        std::memcpy(buf.symbol(0), symbols, (k + r) * symbol_size);
        decode(buf, std::vector<unsigned>(erased, erased + n_erased), code, threads);
        std::memcpy(symbols, buf.symbol(0), (k + r) * symbol_size);
    });
}

// ---------------------------------------------------------------------------
// Precompiled plans for timing the reference CPU path the way bench.hpp:146-208
// does (schedule compiled once, buffers preallocated, parallel_replay timed).
// mode 0: encode with the ring schedule (compile_schedule, schedule.hpp:94)
// mode 1: encode with the CRS schedule  (compile_crs_schedule, schedule.hpp:168)
// mode 2: decode (codec.hpp:241-284 restated with CRS schedules): erased data
//         via decode_matrix, then erased parity re-encoded from data.
// mode 3: decode, same two passes with ring schedules (the reference's own
//         decode(); valid for the AOP/ESP fields only).
// mode | 0x10: the code uses the Parity transform (ring schedules only).
struct RefPlan {
    FieldSpec spec;
    CodeSpec code;
    unsigned mode;
    std::unique_ptr<SymbolBuffer> symbols; // k data then r parity
    XorSchedule sched_a, sched_b;
    std::vector<unsigned> in_a, out_a, in_b, out_b;
    bool has_a = false, has_b = false;
};

REF_EXPORT void* ref_plan_create(unsigned w, unsigned n, unsigned kind, unsigned s, unsigned r_esp,
                                 std::uint32_t modulus, unsigned k, unsigned r, unsigned mode,
                                 std::uint64_t symbol_size, const unsigned* erased,
                                 unsigned n_erased) {
    RefPlan* p = nullptr;
    const int rc = guarded([&] {
        auto plan = std::make_unique<RefPlan>(RefPlan{make_field(w, n, kind, s, r_esp, modulus),
                                                      CodeSpec{}, mode, nullptr, {}, {}, {}, {},
                                                      {}, {}, false, false});
        const TransformKind kind = (mode & 0x10) ? TransformKind::Parity : TransformKind::Embedding;
        mode &= 0xF;
        plan->mode = mode;
        plan->code = CodeSpec{k, r, plan->spec, kind};
        plan->symbols = std::make_unique<SymbolBuffer>(k + r, symbol_size, plan->spec);
        const FieldMatrix c = cauchy_parity_matrix(plan->code);
        auto compile = [&](const FieldMatrix& m, bool crs) {
            return crs ? compile_crs_schedule(m) : compile_schedule(m, kind);
        };
        if (mode <= 1) {
            plan->sched_a = compile(c, mode == 1);
            plan->in_a = detail::iota_map(k);
            plan->out_a = detail::iota_map(r, k);
            plan->has_a = true;
        } else {
            const bool crs = mode == 2;
            std::vector<bool> gone(k + r, false);
            for (unsigned i = 0; i < n_erased; ++i) gone[erased[i]] = true;
            std::vector<unsigned> surv, ed, ep;
            for (unsigned i = 0; i < k + r && surv.size() < k; ++i)
                if (!gone[i]) surv.push_back(i);
            for (unsigned i = 0; i < k + r; ++i)
                if (gone[i]) (i < k ? ed : ep).push_back(i);
            if (!ed.empty()) {
                plan->sched_a = compile(decode_matrix(plan->code, c, surv), crs);
                plan->in_a = surv;
                plan->out_a = ed;
                plan->has_a = true;
            }
            if (!ep.empty()) {
                FieldMatrix rows(ep.size(), k, plan->spec);
                for (std::size_t i = 0; i < ep.size(); ++i)
                    for (unsigned j = 0; j < k; ++j) rows.at(i, j) = c.at(ep[i] - k, j);
                plan->sched_b = compile(rows, crs);
                plan->in_b = detail::iota_map(k);
                plan->out_b = ep;
                plan->has_b = true;
            }
        }
        p = plan.release();
    });
    return rc == 0 ? p : nullptr;
}

REF_EXPORT std::uint8_t* ref_plan_symbol(void* plan, unsigned sym) {
    return static_cast<RefPlan*>(plan)->symbols->symbol(sym);
}

REF_EXPORT int ref_plan_run(void* plan, unsigned threads) {
    RefPlan* p = static_cast<RefPlan*>(plan);
    return guarded([&] {
        if (p->has_a)
            parallel_replay(p->sched_a, *p->symbols, p->in_a, *p->symbols, p->out_a, threads);
        if (p->has_b)
            parallel_replay(p->sched_b, *p->symbols, p->in_b, *p->symbols, p->out_b, threads);
    });
}

REF_EXPORT void ref_plan_destroy(void* plan) { delete static_cast<RefPlan*>(plan); }

// ---------------------------------------------------------------------------
// Shard container and file codec (container.hpp), for pinning the GPU file
// path byte for byte.  The reference's field_id() records any AOP field as
// 0 (field.hpp:54-56), so only gf16_aop / gf64_esp shard sets round-trip.

// container.hpp:114-127 serialize_header
REF_EXPORT int ref_serialize_header(unsigned field, unsigned transform, unsigned k, unsigned r, unsigned index,
                                    std::uint32_t symbol_size, std::uint64_t length, std::uint8_t* out) {
    return guarded([&] {
        ShardHeader h;
        h.field = static_cast<std::uint8_t>(field);
        h.transform = static_cast<std::uint8_t>(transform);
        h.k = static_cast<std::uint16_t>(k);
        h.r = static_cast<std::uint16_t>(r);
        h.shard_index = static_cast<std::uint16_t>(index);
        h.symbol_size = symbol_size;
        h.original_length = length;
        const auto b = serialize_header(h);
        std::memcpy(out, b.data(), b.size());
    });
}

// container.hpp:132-161 parse_header; fields out[0..7] =
// version, field, transform, k, r, shard_index, symbol_size, original_length
REF_EXPORT int ref_parse_header(const std::uint8_t* bytes, std::uint64_t len, std::uint64_t* out) {
    return guarded([&] {
        const ShardHeader h = parse_header(std::span<const std::uint8_t>(bytes, len));
        const std::uint64_t v[8] = {h.version, h.field, h.transform, h.k, h.r, h.shard_index, h.symbol_size,
                                    h.original_length};
        std::memcpy(out, v, sizeof v);
    });
}

// container.hpp:41-55
REF_EXPORT std::uint32_t ref_crc32(const std::uint8_t* bytes, std::uint64_t len) {
    return crc32(std::span<const std::uint8_t>(bytes, len));
}

// container.hpp:168-222 encode_file
REF_EXPORT int ref_encode_file(const char* input, const char* out_dir, unsigned w, unsigned n, unsigned kind,
                               unsigned s, unsigned r_esp, std::uint32_t modulus, unsigned k, unsigned r,
                               unsigned transform, std::uint32_t symbol_size) {
    return guarded([&] {
        const CodeSpec code{k, r, make_field(w, n, kind, s, r_esp, modulus), static_cast<TransformKind>(transform)};
        encode_file(input, out_dir, code, symbol_size);
    });
}

// container.hpp:249-299 decode_file
REF_EXPORT int ref_decode_file(const char* const* paths, unsigned n_paths, const char* output) {
    return guarded([&] {
        std::vector<std::filesystem::path> ps;
        for (unsigned i = 0; i < n_paths; ++i) ps.emplace_back(paths[i]);
        decode_file(ps, output);
    });
}

// bench.hpp:111-208: BenchRunner::run_point, the reference's own benchmark
// cell (one stripe, column windows over `workers` threads with a barrier
// per iteration, auto-calibrated to target_seconds).  GB/s in the
// reference's (k + r) * size convention.  codec 0 pyrit, 1 crs, 2 table;
// op 0 encode, 1 decode.  Valid only where TableCodec is (w <= 6).
REF_EXPORT double ref_bench_point(unsigned w, unsigned n, unsigned kind, unsigned s, unsigned r_esp,
                                  std::uint32_t modulus, unsigned k, unsigned r, unsigned transform, unsigned codec,
                                  unsigned op, std::uint64_t size, unsigned workers, double target_seconds) {
    double out = -1.0;
    guarded([&] {
        const CodeSpec code{k, r, make_field(w, n, kind, s, r_esp, modulus), static_cast<TransformKind>(transform)};
        BenchRunner runner(code, size);
        out = runner.run_point(static_cast<CodecKind>(codec), op ? BenchOp::Decode : BenchOp::Encode, workers, 0,
                               target_seconds);
    });
    return out;
}
