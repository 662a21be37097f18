// extern "C" boundary (include/pyrit_b200.h).  Every entry point catches
// and maps errors to return codes; nothing throws across the ABI.
#include "../../include/pyrit_b200.h"

#include <cstdlib>
#include <cstring>
#include <list>
#include <memory>
#include <mutex>
#include <sstream>
#include <unordered_map>

#include "algebra.hpp"
#include "kernels.hpp"
#include "pipeline.hpp"
#include "plans.hpp"
#include "container.hpp"
#include "program.hpp"
#include "runtime.hpp"

using namespace pyrit_b200;

struct pyrit_plan {
    Program prog;
    // plans from a schedule (pyrit_plan_from_schedule): kernel input q reads
    // slot src_slot[q] (>= 0 input slot, < 0 output slot -1-q's prior
    // contents), kernel output r is output slot dst_slot[r]
    bool sched = false;
    std::uint32_t k = 0, outputs = 0;
    std::vector<std::int32_t> src_slot;
    std::vector<std::uint32_t> dst_slot;
};

namespace {

// slot-indexed pointer arrays -> the kernel's input/output arrays
void kernel_ptrs(const pyrit_plan* plan, const uint8_t* const* in, uint8_t* const* out,
                 std::vector<const uint8_t*>& kin, std::vector<uint8_t*>& kout) {
    kin.clear();
    kout.clear();
    for (std::int32_t s : plan->src_slot) {
        const uint8_t* p = s >= 0 ? in[s] : out[-1 - s];
        if (!p) raise(Errc::InvalidArgument, "null symbol pointer");
        kin.push_back(p);
    }
    for (std::uint32_t i : plan->dst_slot) {
        if (!out[i]) raise(Errc::InvalidArgument, "null symbol pointer");
        kout.push_back(out[i]);
    }
}

} // namespace

namespace {

thread_local std::string g_last_error;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const Error& e) {
        g_last_error = e.what();
        return 1 + static_cast<int>(e.code());
    } catch (const CudaFailure& e) {
        g_last_error = e.what();
        return e.code();
    } catch (const std::bad_alloc&) {
        g_last_error = "out of host memory";
        return -2;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return -3;
    }
}

Field to_field(const pyrit_field* f) {
    if (!f) raise(Errc::InvalidArgument, "null field");
    Field x;
    x.w = f->w;
    x.n = f->n;
    x.kind = static_cast<FieldKind>(f->kind);
    x.s = f->s;
    x.r_esp = f->r_esp;
    x.modulus = f->modulus;
    validate_field(x);
    return x;
}

void check_code(const pyrit_code* c) {
    if (!c) raise(Errc::InvalidArgument, "null code");
    if (c->k == 0) raise(Errc::InvalidArgument, "k must be at least 1");          // matrix.hpp:25-26
    if (c->transform > 1) raise(Errc::InvalidArgument, "unknown transform");
    const Field f = to_field(&c->field);
    if (c->k + c->r > f.field_size()) raise(Errc::TooManySymbols, "k + r exceeds field size"); // :274-277
}

std::uint64_t strip_of(const pyrit_code* c, std::uint64_t symbol_size) {
    // SymbolBuffer shape rule, codec.hpp:28-30
    if (symbol_size == 0 || symbol_size % c->field.w != 0 || symbol_size % 8 != 0)
        raise(Errc::BufferShape, "symbol size must be a positive multiple of w and of the word width");
    return symbol_size / c->field.w;
}

CodeParams params_of(const pyrit_code* c) {
    CodeParams p;
    p.k = c->k;
    p.r = c->r;
    p.field = to_field(&c->field);
    p.kind = static_cast<TransformKind>(c->transform);
    return p;
}

std::shared_ptr<const Program> encode_program(const pyrit_code* c) { return encode_program(params_of(c)); }

DecodeProgram decode_program(const pyrit_code* c, const std::vector<std::uint32_t>& erased) {
    return decode_program(params_of(c), erased);
}

} // namespace

extern "C" {

const char* pyrit_version(void) { return "pyrit_b200 0.1 (sm_100a, generated ring programs)"; }

const char* pyrit_strerror(int code) {
    static const char* errc[] = {"ok",
                                 "ZeroInverse: multiplicative inverse of 0 requested",
                                 "Singular: matrix inversion hit a zero pivot",
                                 "TooManySymbols: k + r exceeds the field size",
                                 "BufferShape: symbol buffer does not match the code geometry",
                                 "TransformMismatch",
                                 "InsufficientShards: fewer than k usable shards",
                                 "HeaderMismatch",
                                 "ChecksumError",
                                 "BadHeader",
                                 "IoError",
                                 "InvalidArgument: bad API parameter"};
    if (code >= 0 && code <= 11) return errc[code];
    if (!g_last_error.empty()) return g_last_error.c_str();
    if (code <= -2000) return "CUDA driver error";
    if (code <= -1000) return "NVRTC error";
    return "CUDA runtime error";
}

int pyrit_field_named(const char* name, pyrit_field* out) {
    return guarded([&] {
        if (!name || !out) raise(Errc::InvalidArgument, "null argument");
        const std::string n = name;
        if (n == "gf16") *out = pyrit_field{4, 5, 0, 1, 4, 0x1F};          // field.hpp:38-40
        else if (n == "gf64") *out = pyrit_field{6, 9, 1, 3, 2, 0x49};     // field.hpp:41-43
        else if (n == "gf256_r17") *out = pyrit_field{8, 17, 0, 1, 8, 0x139};
        else if (n == "gf1024") *out = pyrit_field{10, 11, 0, 1, 10, 0x7FF};
        else if (n == "gf4096") *out = pyrit_field{12, 13, 0, 1, 12, 0x1FFF};
        else raise(Errc::InvalidArgument, "unknown field name " + n);
    });
}

int pyrit_field_validate(const pyrit_field* f) {
    return guarded([&] { to_field(f); });
}

int pyrit_gf_mul(const pyrit_field* f, uint32_t a, uint32_t b, uint32_t* out) {
    return guarded([&] {
        if (!out) raise(Errc::InvalidArgument, "null argument");
        *out = gf_mul(a, b, to_field(f));
    });
}

int pyrit_gf_inv(const pyrit_field* f, uint32_t a, uint32_t* out) {
    return guarded([&] {
        if (!out) raise(Errc::InvalidArgument, "null argument");
        *out = gf_inv(a, to_field(f));
    });
}

int pyrit_sparse_transform(const pyrit_field* f, uint32_t u, uint32_t* rep) {
    return guarded([&] {
        const Field x = to_field(f);
        if (!rep) raise(Errc::InvalidArgument, "null argument");
        if (u >= x.field_size()) raise(Errc::InvalidArgument, "element outside the field");
        *rep = sparse_transform(u, x);
    });
}

int pyrit_fold_table(const pyrit_field* f, uint32_t* fold) {
    return guarded([&] {
        const auto t = fold_table(to_field(f));
        if (!fold) raise(Errc::InvalidArgument, "null argument");
        std::memcpy(fold, t.data(), t.size() * sizeof(uint32_t));
    });
}

int pyrit_cauchy_parity_matrix(const pyrit_code* code, uint16_t* out) {
    return guarded([&] {
        check_code(code);
        if (!out) raise(Errc::InvalidArgument, "null argument");
        const Matrix m = cauchy_parity_matrix(code->k, code->r, to_field(&code->field));
        std::memcpy(out, m.e.data(), m.e.size() * sizeof(uint16_t));
    });
}

int pyrit_decode_matrix(const pyrit_code* code, const uint32_t* survivors, uint16_t* out, uint32_t* rows) {
    return guarded([&] {
        check_code(code);
        if (!survivors || !out || !rows) raise(Errc::InvalidArgument, "null argument");
        const Field f = to_field(&code->field);
        const Matrix c = cauchy_parity_matrix(code->k, code->r, f);
        const Matrix dm =
            decode_matrix(code->k, code->r, f, c, std::vector<uint32_t>(survivors, survivors + code->k));
        std::memcpy(out, dm.e.data(), dm.e.size() * sizeof(uint16_t));
        *rows = dm.rows;
    });
}

int pyrit_repair_matrix(const pyrit_code* code, const uint32_t* erased, uint32_t n_erased, uint32_t* survivors,
                        uint32_t* outputs, uint16_t* matrix) {
    return guarded([&] {
        check_code(code);
        if ((!erased && n_erased) || !survivors || (n_erased && (!outputs || !matrix)))
            raise(Errc::InvalidArgument, "null argument");
        const RepairPlan rp = repair_matrix(code->k, code->r, to_field(&code->field),
                                            std::vector<uint32_t>(erased, erased + n_erased));
        std::memcpy(survivors, rp.survivors.data(), rp.survivors.size() * sizeof(uint32_t));
        std::memcpy(outputs, rp.outputs.data(), rp.outputs.size() * sizeof(uint32_t));
        std::memcpy(matrix, rp.m.e.data(), rp.m.e.size() * sizeof(uint16_t));
    });
}

int pyrit_plan_create(const pyrit_field* f, uint32_t transform, const uint16_t* matrix, uint32_t rows,
                      uint32_t cols, uint32_t rep, uint32_t group, pyrit_plan** out) {
    return guarded([&] {
        if (!out || (!matrix && rows != 0 && cols != 0)) raise(Errc::InvalidArgument, "null argument");
        if (transform > 1) raise(Errc::InvalidArgument, "unknown transform");
        Matrix m(rows, cols);
        std::memcpy(m.e.data(), matrix, std::size_t(rows) * cols * sizeof(uint16_t));
        CompileOptions opt;
        opt.group = group;
        if (rep > 2) raise(Errc::InvalidArgument, "rep must be 0 (sparse ring), 1 (dense ring) or 2 (CRS bitmatrix)");
        opt.dense = rep == 1;
        opt.crs = rep == 2;
        auto plan = std::make_unique<pyrit_plan>();
        plan->prog = compile_program(to_field(f), static_cast<TransformKind>(transform), m, opt);
        *out = plan.release();
    });
}

int pyrit_plan_from_ringmat(const pyrit_ringmat* m, pyrit_plan** out) {
    return guarded([&] {
        if (!m || !out || (!m->reps && m->rows && m->cols)) raise(Errc::InvalidArgument, "null argument");
        if (m->transform > 1) raise(Errc::InvalidArgument, "unknown transform");
        auto plan = std::make_unique<pyrit_plan>();
        plan->prog = ring_program(to_field(&m->field), static_cast<TransformKind>(m->transform), m->reps, m->rows,
                                  m->cols);
        *out = plan.release();
    });
}

int pyrit_cu_apply_ringmat(const pyrit_ringmat* m, const uint8_t* const* in, uint8_t* const* out,
                           uint64_t strip_bytes, uint64_t off, uint64_t len, void* stream) {
    return guarded([&] {
        if (!m || !in || !out || (!m->reps && m->rows && m->cols)) raise(Errc::InvalidArgument, "null argument");
        if (m->transform > 1) raise(Errc::InvalidArgument, "unknown transform");
        auto p = ringmat_program(to_field(&m->field), static_cast<TransformKind>(m->transform), m->reps, m->rows,
                                 m->cols);
        launch_program(*p, in, out, strip_bytes, off, len, static_cast<cudaStream_t>(stream));
    });
}

int pyrit_plan_from_schedule(const pyrit_field* f, uint32_t k, uint32_t outputs, const pyrit_xor_op* ops,
                             size_t n_ops, const uint32_t* labels, pyrit_plan** out) {
    return guarded([&] {
        if (!out || (!ops && n_ops)) raise(Errc::InvalidArgument, "null argument");
        std::vector<ScheduleOp> v(n_ops);
        for (size_t i = 0; i < n_ops; ++i)
            v[i] = ScheduleOp{ops[i].src_sym, ops[i].src_pkt, ops[i].dst_sym, ops[i].dst_pkt, ops[i].mode};
        std::vector<uint32_t> lab;
        if (labels) lab.assign(labels, labels + std::size_t(k) + outputs);
        ScheduleProgram sp = compile_schedule_program(to_field(f), k, outputs, v, lab, CompileOptions{});
        auto plan = std::make_unique<pyrit_plan>();
        plan->prog = std::move(sp.prog);
        plan->sched = true;
        plan->k = k;
        plan->outputs = outputs;
        plan->src_slot = std::move(sp.src_slot);
        plan->dst_slot = std::move(sp.dst_slot);
        *out = plan.release();
    });
}

int pyrit_plan_encode(const pyrit_code* code, pyrit_plan** out) {
    return guarded([&] {
        check_code(code);
        auto plan = std::make_unique<pyrit_plan>();
        plan->prog = *encode_program(code);
        *out = plan.release();
    });
}

int pyrit_plan_decode(const pyrit_code* code, const uint32_t* erased, uint32_t n_erased, pyrit_plan** out,
                      uint32_t* survivors, uint32_t* outputs) {
    return guarded([&] {
        check_code(code);
        const DecodeProgram d = decode_program(code, std::vector<uint32_t>(erased, erased + n_erased));
        if (!d.prog) raise(Errc::InvalidArgument, "nothing erased");
        auto plan = std::make_unique<pyrit_plan>();
        plan->prog = *d.prog;
        if (survivors) std::memcpy(survivors, d.repair.survivors.data(), d.repair.survivors.size() * sizeof(uint32_t));
        if (outputs) std::memcpy(outputs, d.repair.outputs.data(), d.repair.outputs.size() * sizeof(uint32_t));
        *out = plan.release();
    });
}

int pyrit_plan_get_stats(const pyrit_plan* plan, pyrit_plan_stats* out) {
    return guarded([&] {
        if (!plan || !out) raise(Errc::InvalidArgument, "null argument");
        const Program& fp = full_program(plan->prog);
        const auto& s = fp.stats;
        out->rows = fp.rows;
        out->cols = fp.cols;
        out->matrix_ones = s.matrix_ones;
        out->ref_region_ops = s.ref_region_ops;
        out->naive_xors = s.naive_xors;
        out->xors = s.xors;
        out->loads = s.loads;
        out->stores = s.stores;
        out->group = fp.group;
        out->parts = static_cast<uint32_t>(fp.parts.size());
        out->part_xors = 0;
        for (const Program& q : fp.parts) out->part_xors += q.stats.xors;
    });
}

int pyrit_plan_key(const pyrit_plan* plan, char* buf, size_t cap) {
    return guarded([&] {
        if (!plan || !buf || !cap) raise(Errc::InvalidArgument, "null argument");
        const std::string k = plan_key(plan->prog);
        const size_t n = std::min(cap - 1, k.size());
        std::memcpy(buf, k.data(), n);
        buf[n] = 0;
    });
}

int pyrit_plan_inject_fault(pyrit_plan* plan, uint32_t entry, uint32_t bit) {
    return guarded([&] {
        if (!plan) raise(Errc::InvalidArgument, "null plan");
        const Program& fp = full_program(plan->prog);
        if (plan->sched || fp.crs) raise(Errc::InvalidArgument, "fault injection applies to ring programs");
        if (entry >= fp.reps.size() || bit >= fp.field.n) raise(Errc::InvalidArgument, "no such representative bit");
        std::vector<uint32_t> reps = fp.reps;
        reps[entry] ^= 1u << bit;
        Matrix m(fp.rows, fp.cols);
        m.e = fp.matrix;
        CompileOptions opt;
        opt.reps = &reps;
        plan->prog = compile_program(fp.field, fp.kind, m, opt);
    });
}

int pyrit_plan_reps(const pyrit_plan* plan, uint32_t* reps) {
    return guarded([&] {
        if (!plan || !reps) raise(Errc::InvalidArgument, "null argument");
        std::memcpy(reps, plan->prog.reps.data(), plan->prog.reps.size() * sizeof(uint32_t));
    });
}

int pyrit_plan_source(const pyrit_plan* plan, uint32_t lanes, char* buf, size_t cap, size_t* len, char* name,
                      size_t name_cap) {
    return guarded([&] {
        if (!plan) raise(Errc::InvalidArgument, "null plan");
        const bool staged = lanes == PYRIT_SOURCE_STAGED || lanes == PYRIT_SOURCE_STAGED + 1 ||
                            lanes == PYRIT_SOURCE_STAGED + 4 || lanes == PYRIT_SOURCE_STAGED + 8;
        if (lanes != 0 && lanes != 1 && lanes != 2 && lanes != 4 && !staged) raise(Errc::InvalidArgument, "bad lanes");
        const Program& fp = full_program(plan->prog);
        KernelShape ks = direct_shape(fp, staged ? 1 : lanes);
        if (staged) {
            ks = staged_shape(fp, 227 * 1024);
            if (!ks.staged) raise(Errc::BufferShape, "program tiles do not fit in shared memory");
            ks.chunk = lanes <= PYRIT_SOURCE_STAGED + 1 ? 16 : lanes - PYRIT_SOURCE_STAGED;
            if (ks.chunk != 16) ks.copy = 1; // TMA needs 16-byte alignment
            ks.tmap4 = lanes == PYRIT_SOURCE_STAGED + 1 && ks.copy == 2 ? 1u : 0u;
            if (const char* env = std::getenv("PYRIT_B200_WS")) ks.ws = std::atoi(env) ? 1u : 0u;
            if (const char* env = std::getenv("PYRIT_B200_COPY")) { // same producer the runtime would pick
                const int c = std::atoi(env);
                ks.copy = c == 2 ? 2u : c ? 1u : 0u;
            }
        }
        const std::string src = generate_cuda(fp, ks);
        const std::string nm = kernel_name(fp, ks);
        if (len) *len = src.size();
        if (buf && cap) {
            const size_t n = std::min(cap - 1, src.size());
            std::memcpy(buf, src.data(), n);
            buf[n] = 0;
        }
        if (name && name_cap) {
            const size_t n = std::min(name_cap - 1, nm.size());
            std::memcpy(name, nm.data(), n);
            name[n] = 0;
        }
    });
}

int pyrit_plan_interpret(const pyrit_plan* plan, const uint8_t* const* in, uint8_t* const* out,
                         uint64_t strip_bytes, uint64_t off, uint64_t len) {
    return guarded([&] {
        if (!plan || !in || !out) raise(Errc::InvalidArgument, "null argument");
        if (off + len > strip_bytes) raise(Errc::BufferShape, "column window out of range");
        if (plan->sched) {
            if (plan->dst_slot.empty()) return;
            std::vector<const uint8_t*> kin;
            std::vector<uint8_t*> kout;
            kernel_ptrs(plan, in, out, kin, kout);
            // prior contents of output slots the schedule reads: snapshot the
            // window first (the interpreter stores as it goes)
            std::vector<std::vector<uint8_t>> snap;
            for (std::size_t q = 0; q < kin.size(); ++q)
                if (plan->src_slot[q] < 0) {
                    snap.emplace_back(kin[q], kin[q] + std::size_t(plan->prog.field.w) * strip_bytes);
                    kin[q] = snap.back().data();
                }
            interpret_program(plan->prog, kin.data(), kout.data(), strip_bytes, off, len);
            return;
        }
        // PYRIT_B200_INTERPRET_GENERIC=1: evaluate the generic kernel's bitmatrix
        // (Program::field_masks) instead, so CPU tests pin what it computes
        const Program& fp = full_program(plan->prog);
        const char* gen_env = std::getenv("PYRIT_B200_INTERPRET_GENERIC");
        if (gen_env && std::atoi(gen_env)) {
            const Program& p = fp;
            if (p.field_masks.empty()) raise(Errc::InvalidArgument, "no generic bitmatrix for this program");
            const std::uint32_t w = p.field.w;
            for (std::uint32_t i = 0; i < p.rows; ++i)
                for (std::uint32_t b = 0; b < w; ++b) {
                    std::uint8_t* d = out[i] + std::uint64_t(b) * strip_bytes + off;
                    std::memset(d, 0, len);
                    for (std::uint32_t j = 0; j < p.cols; ++j)
                        for (std::uint32_t c = 0; c < w; ++c)
                            if ((p.field_masks[(std::size_t(i) * w + b) * p.cols + j] >> c) & 1u) {
                                const std::uint8_t* src = in[j] + std::uint64_t(c) * strip_bytes + off;
                                for (std::uint64_t q = 0; q < len; ++q) d[q] ^= src[q];
                            }
                }
            return;
        }
        // PYRIT_B200_INTERPRET_PARTS=1: run the output parts the staged and
        // split kernels execute (rows part_row0[r] ..) instead of the whole
        // program, so CPU tests cover the part programs too
        const char* parts_env = std::getenv("PYRIT_B200_INTERPRET_PARTS");
        if (parts_env && std::atoi(parts_env) && !fp.parts.empty()) {
            for (std::size_t r = 0; r < fp.parts.size(); ++r)
                interpret_program(fp.parts[r], in, out + fp.part_row0[r], strip_bytes, off, len);
            return;
        }
        interpret_program(fp, in, out, strip_bytes, off, len);
    });
}

void pyrit_plan_destroy(pyrit_plan* plan) { delete plan; }

int pyrit_cu_apply(const pyrit_plan* plan, const uint8_t* const* in, uint8_t* const* out, uint64_t strip_bytes,
                   uint64_t off, uint64_t len, void* stream) {
    return guarded([&] {
        if (!plan || !in || !out) raise(Errc::InvalidArgument, "null argument");
        if (plan->sched) {
            if (plan->dst_slot.empty()) return; // the schedule writes nothing
            std::vector<const uint8_t*> kin;
            std::vector<uint8_t*> kout;
            kernel_ptrs(plan, in, out, kin, kout);
            launch_program(plan->prog, kin.data(), kout.data(), strip_bytes, off, len, static_cast<cudaStream_t>(stream));
            return;
        }
        launch_program(plan->prog, in, out, strip_bytes, off, len, static_cast<cudaStream_t>(stream));
    });
}

int pyrit_cu_prepare(const pyrit_plan* plan) {
    return guarded([&] {
        if (!plan) raise(Errc::InvalidArgument, "null plan");
        prepare_program(full_program(plan->prog), preferred_lanes());
    });
}

int pyrit_cu_encode(const pyrit_code* code, const uint8_t* const* data, uint8_t* const* parity,
                    uint64_t symbol_size, void* stream) {
    return guarded([&] {
        check_code(code);
        const std::uint64_t strip = strip_of(code, symbol_size);
        if (!data || (!parity && code->r)) raise(Errc::InvalidArgument, "null symbol array");
        if (code->r == 0) return;
        auto p = encode_program(code);
        launch_program(*p, data, parity, strip, 0, strip, static_cast<cudaStream_t>(stream));
    });
}

int pyrit_cu_encode_crs(const pyrit_code* code, const uint8_t* const* data, uint8_t* const* parity,
                        uint64_t symbol_size, void* stream) {
    return guarded([&] {
        check_code(code);
        const std::uint64_t strip = strip_of(code, symbol_size);
        if (!data || (!parity && code->r)) raise(Errc::InvalidArgument, "null symbol array");
        if (code->r == 0) return;
        CodeParams cp = params_of(code);
        cp.kind = TransformKind::Embedding; // encode_crs ignores the transform (codec.hpp:223-231)
        cp.crs = true;
        auto p = encode_program(cp);
        launch_program(*p, data, parity, strip, 0, strip, static_cast<cudaStream_t>(stream));
    });
}

int pyrit_cu_decode(const pyrit_code* code, uint8_t* const* symbols, const uint32_t* erased, uint32_t n_erased,
                    uint64_t symbol_size, void* stream) {
    return guarded([&] {
        check_code(code);
        const std::uint64_t strip = strip_of(code, symbol_size);
        if (!symbols || (!erased && n_erased)) raise(Errc::InvalidArgument, "null argument");
        const DecodeProgram d = decode_program(code, std::vector<uint32_t>(erased, erased + n_erased));
        if (!d.prog) return;
        std::vector<const uint8_t*> in;
        std::vector<uint8_t*> out;
        for (uint32_t s : d.repair.survivors) in.push_back(symbols[s]);
        for (uint32_t o : d.repair.outputs) out.push_back(symbols[o]);
        launch_program(*d.prog, in.data(), out.data(), strip, 0, strip, static_cast<cudaStream_t>(stream));
    });
}

int pyrit_rt_interpret(const pyrit_plan* plan, const uint8_t* const* in, uint8_t* const* out, uint64_t strip_bytes,
                       uint64_t off, uint64_t len, uint64_t stripes, uint64_t in_pitch, uint64_t out_pitch) {
    return guarded([&] {
        if (!plan || !in || !out) raise(Errc::InvalidArgument, "null argument");
        if (plan->sched) raise(Errc::InvalidArgument, "replayed schedules do not run on the runtime-matrix kernel");
        if (off + len > strip_bytes) raise(Errc::BufferShape, "column window out of range");
        if (len == 0 || stripes == 0 || plan->prog.rows == 0) return;
        interpret_ring_rt(plan->prog, in, out, strip_bytes, off, len, stripes, in_pitch, out_pitch);
    });
}

int pyrit_numa_bind_thread(int device) { return numa_bind_thread(device); }
int pyrit_bind_thread_cpulist(const char* cpulist) { return bind_thread_cpulist(cpulist); }

int pyrit_rt_plan_info(const pyrit_plan* plan, uint32_t info[4]) {
    return guarded([&] {
        if (!plan || !info) raise(Errc::InvalidArgument, "null argument");
        if (plan->sched) raise(Errc::InvalidArgument, "replayed schedules do not run on the runtime-matrix kernel");
        ring_rt_plan_info(plan->prog, info);
    });
}

int pyrit_cu_apply_batch(const pyrit_plan* plan, const uint8_t* const* in, uint8_t* const* out,
                         uint64_t strip_bytes, uint64_t off, uint64_t len, uint64_t stripes, uint64_t in_pitch,
                         uint64_t out_pitch, void* stream) {
    return guarded([&] {
        if (!plan || !in || !out) raise(Errc::InvalidArgument, "null argument");
        if (plan->sched) {
            if (plan->dst_slot.empty()) return;
            for (std::int32_t s : plan->src_slot)
                if (s < 0 && in_pitch != out_pitch)
                    raise(Errc::InvalidArgument, "schedule reads an output slot: in_pitch must equal out_pitch");
            std::vector<const uint8_t*> kin;
            std::vector<uint8_t*> kout;
            kernel_ptrs(plan, in, out, kin, kout);
            launch_batch(plan->prog, kin.data(), kout.data(), strip_bytes, off, len, stripes, in_pitch, out_pitch,
                         static_cast<cudaStream_t>(stream));
            return;
        }
        launch_batch(plan->prog, in, out, strip_bytes, off, len, stripes, in_pitch, out_pitch,
                     static_cast<cudaStream_t>(stream));
    });
}

int pyrit_cu_encode_batch(const pyrit_code* code, const uint8_t* const* data, uint8_t* const* parity,
                          uint64_t symbol_size, uint64_t stripes, uint64_t data_pitch, uint64_t parity_pitch,
                          void* stream) {
    return guarded([&] {
        check_code(code);
        const std::uint64_t strip = strip_of(code, symbol_size);
        if (!data || (!parity && code->r)) raise(Errc::InvalidArgument, "null symbol array");
        if (code->r == 0) return;
        auto p = encode_program(code);
        launch_batch(*p, data, parity, strip, 0, strip, stripes, data_pitch, parity_pitch,
                     static_cast<cudaStream_t>(stream));
    });
}

int pyrit_cu_decode_batch(const pyrit_code* code, uint8_t* const* symbols, const uint32_t* erased,
                          uint32_t n_erased, uint64_t symbol_size, uint64_t stripes, uint64_t pitch, void* stream) {
    return guarded([&] {
        check_code(code);
        const std::uint64_t strip = strip_of(code, symbol_size);
        if (!symbols || (!erased && n_erased)) raise(Errc::InvalidArgument, "null argument");
        const DecodeProgram d = decode_program(code, std::vector<uint32_t>(erased, erased + n_erased));
        if (!d.prog) return;
        std::vector<const uint8_t*> in;
        std::vector<uint8_t*> out;
        for (uint32_t s : d.repair.survivors) in.push_back(symbols[s]);
        for (uint32_t o : d.repair.outputs) out.push_back(symbols[o]);
        launch_batch(*d.prog, in.data(), out.data(), strip, 0, strip, stripes, pitch, pitch,
                     static_cast<cudaStream_t>(stream));
    });
}

int pyrit_encode_host(const pyrit_code* code, const uint8_t* data, uint8_t* parity, uint64_t symbol_size,
                      int device) {
    return guarded([&] {
        check_code(code);
        const std::uint64_t strip = strip_of(code, symbol_size);
        if (!data || (!parity && code->r)) raise(Errc::InvalidArgument, "null buffer");
        if (code->r == 0) return;
        auto p = encode_program(code);
        std::vector<const uint8_t*> in;
        std::vector<uint8_t*> out;
        for (uint32_t j = 0; j < code->k; ++j) in.push_back(data + std::uint64_t(j) * symbol_size);
        for (uint32_t i = 0; i < code->r; ++i) out.push_back(parity + std::uint64_t(i) * symbol_size);
        run_host(*p, in, out, strip, device);
    });
}

int pyrit_apply_host(const pyrit_plan* plan, const uint8_t* const* in, uint8_t* const* out, uint64_t strip_bytes,
                     uint64_t off, uint64_t len, int device) {
    return guarded([&] {
        if (!plan || !in || !out) raise(Errc::InvalidArgument, "null argument");
        if (off + len > strip_bytes) raise(Errc::BufferShape, "column window out of range");
        std::vector<const uint8_t*> kin;
        std::vector<uint8_t*> kout;
        if (plan->sched) {
            if (plan->dst_slot.empty()) return;
            kernel_ptrs(plan, in, out, kin, kout);
        } else {
            kin.assign(in, in + plan->prog.cols);
            kout.assign(out, out + plan->prog.rows);
            for (const uint8_t* p : kin)
                if (!p) raise(Errc::InvalidArgument, "null symbol pointer");
            for (uint8_t* p : kout)
                if (!p) raise(Errc::InvalidArgument, "null symbol pointer");
        }
        run_host_window(plan->prog, kin, kout, strip_bytes, off, len, device);
    });
}

int pyrit_encode_host_devices(const pyrit_code* code, const uint8_t* data, uint8_t* parity, uint64_t symbol_size,
                              const int* devices, uint32_t n_devices) {
    return guarded([&] {
        check_code(code);
        const std::uint64_t strip = strip_of(code, symbol_size);
        if (!data || (!parity && code->r) || !devices || !n_devices) raise(Errc::InvalidArgument, "null argument");
        if (code->r == 0) return;
        auto p = encode_program(code);
        std::vector<const uint8_t*> in;
        std::vector<uint8_t*> out;
        for (uint32_t j = 0; j < code->k; ++j) in.push_back(data + std::uint64_t(j) * symbol_size);
        for (uint32_t i = 0; i < code->r; ++i) out.push_back(parity + std::uint64_t(i) * symbol_size);
        run_host_devices(*p, in, out, strip, std::vector<int>(devices, devices + n_devices));
    });
}

int pyrit_decode_host_devices(const pyrit_code* code, uint8_t* symbols, const uint32_t* erased, uint32_t n_erased,
                              uint64_t symbol_size, const int* devices, uint32_t n_devices) {
    return guarded([&] {
        check_code(code);
        const std::uint64_t strip = strip_of(code, symbol_size);
        if (!symbols || (!erased && n_erased) || !devices || !n_devices) raise(Errc::InvalidArgument, "null argument");
        const DecodeProgram d = decode_program(code, std::vector<uint32_t>(erased, erased + n_erased));
        if (!d.prog) return;
        std::vector<const uint8_t*> in;
        std::vector<uint8_t*> out;
        for (uint32_t s : d.repair.survivors) in.push_back(symbols + std::uint64_t(s) * symbol_size);
        for (uint32_t o : d.repair.outputs) out.push_back(symbols + std::uint64_t(o) * symbol_size);
        run_host_devices(*d.prog, in, out, strip, std::vector<int>(devices, devices + n_devices));
    });
}

int pyrit_encode_crs_host(const pyrit_code* code, const uint8_t* data, uint8_t* parity, uint64_t symbol_size,
                          int device) {
    return guarded([&] {
        check_code(code);
        const std::uint64_t strip = strip_of(code, symbol_size);
        if (!data || (!parity && code->r)) raise(Errc::InvalidArgument, "null buffer");
        if (code->r == 0) return;
        CodeParams cp = params_of(code);
        cp.kind = TransformKind::Embedding;
        cp.crs = true;
        auto p = encode_program(cp);
        std::vector<const uint8_t*> in;
        std::vector<uint8_t*> out;
        for (uint32_t j = 0; j < code->k; ++j) in.push_back(data + std::uint64_t(j) * symbol_size);
        for (uint32_t i = 0; i < code->r; ++i) out.push_back(parity + std::uint64_t(i) * symbol_size);
        run_host(*p, in, out, strip, device);
    });
}

int pyrit_decode_host(const pyrit_code* code, uint8_t* symbols, const uint32_t* erased, uint32_t n_erased,
                      uint64_t symbol_size, int device) {
    return guarded([&] {
        check_code(code);
        const std::uint64_t strip = strip_of(code, symbol_size);
        if (!symbols || (!erased && n_erased)) raise(Errc::InvalidArgument, "null argument");
        const DecodeProgram d = decode_program(code, std::vector<uint32_t>(erased, erased + n_erased));
        if (!d.prog) return;
        std::vector<const uint8_t*> in;
        std::vector<uint8_t*> out;
        for (uint32_t s : d.repair.survivors) in.push_back(symbols + std::uint64_t(s) * symbol_size);
        for (uint32_t o : d.repair.outputs) out.push_back(symbols + std::uint64_t(o) * symbol_size);
        run_host(*d.prog, in, out, strip, device);
    });
}

int pyrit_set_host_chunk(uint64_t strip_chunk_bytes) {
    return guarded([&] {
        if (strip_chunk_bytes % 16) raise(Errc::InvalidArgument, "chunk must be a multiple of 16 bytes");
        set_host_chunk(strip_chunk_bytes);
    });
}

uint32_t pyrit_crc32(const uint8_t* bytes, size_t len) { return bytes || !len ? crc32(bytes, len) : 0u; }

int pyrit_header_serialize(const pyrit_shard_header* h, uint8_t* out) {
    return guarded([&] {
        if (!h || !out) raise(Errc::InvalidArgument, "null argument");
        ShardHeader x;
        x.version = h->version;
        x.field = h->field;
        x.transform = h->transform;
        x.k = h->k;
        x.r = h->r;
        x.shard_index = h->shard_index;
        x.symbol_size = h->symbol_size;
        x.original_length = h->original_length;
        serialize_header(x, out);
    });
}

int pyrit_header_parse(const uint8_t* bytes, size_t len, pyrit_shard_header* out) {
    return guarded([&] {
        if ((!bytes && len) || !out) raise(Errc::InvalidArgument, "null argument");
        const ShardHeader h = parse_header(bytes, len);
        *out = pyrit_shard_header{h.version, h.field, h.transform, h.k, h.r, h.shard_index, h.symbol_size,
                                  h.original_length};
    });
}

int pyrit_field_id(const pyrit_field* f, uint8_t* id) {
    return guarded([&] {
        if (!id) raise(Errc::InvalidArgument, "null argument");
        *id = field_id(to_field(f));
    });
}

int pyrit_field_from_id(uint8_t id, pyrit_field* out) {
    return guarded([&] {
        if (!out) raise(Errc::InvalidArgument, "null argument");
        const Field f = field_from_id(id);
        *out = pyrit_field{f.w, f.n, static_cast<uint32_t>(f.kind), f.s, f.r_esp, f.modulus};
    });
}

int pyrit_shard_path(const char* input, const char* out_dir, uint32_t index, char* buf, size_t cap) {
    return guarded([&] {
        if (!input || !out_dir || !buf) raise(Errc::InvalidArgument, "null argument");
        const std::string p = shard_path(input, out_dir, index);
        if (p.size() + 1 > cap) raise(Errc::InvalidArgument, "path buffer too small");
        std::memcpy(buf, p.c_str(), p.size() + 1);
    });
}

int pyrit_encode_file(const pyrit_code* code, const char* input, const char* out_dir, uint32_t symbol_size,
                      int device) {
    return guarded([&] {
        if (!code || !input || !out_dir) raise(Errc::InvalidArgument, "null argument");
        if (code->transform > 1) raise(Errc::InvalidArgument, "unknown transform");
        encode_file(input, out_dir, code->k, code->r, to_field(&code->field),
                    static_cast<TransformKind>(code->transform), symbol_size, device);
    });
}

int pyrit_decode_file(const char* const* shard_paths, uint32_t n_paths, const char* output, int device) {
    return guarded([&] {
        if ((!shard_paths && n_paths) || !output) raise(Errc::InvalidArgument, "null argument");
        std::vector<std::string> paths;
        for (uint32_t i = 0; i < n_paths; ++i) {
            if (!shard_paths[i]) raise(Errc::InvalidArgument, "null shard path");
            paths.emplace_back(shard_paths[i]);
        }
        decode_file(paths, output, device);
    });
}

int pyrit_set_file_chunk(uint64_t bytes) {
    return guarded([&] { set_file_chunk(bytes); });
}

int pyrit_cu_fill(uint64_t seed, uint64_t frag, uint8_t* dst, uint64_t begin, uint64_t len, uint64_t valid,
                  void* stream) {
    return guarded([&] {
        if (!dst && len) raise(Errc::InvalidArgument, "null buffer");
        if (begin % 8 || reinterpret_cast<std::uintptr_t>(dst) % 8)
            raise(Errc::InvalidArgument, "fill needs 8-byte aligned begin and destination");
        check_cuda(launch_fill(seed, frag, dst, begin, len, valid, static_cast<cudaStream_t>(stream)), "fill");
    });
}

int pyrit_cu_digest(const uint8_t* src, uint64_t len, uint64_t word_offset, uint64_t* out, void* stream) {
    return guarded([&] {
        if ((!src && len) || !out) raise(Errc::InvalidArgument, "null buffer");
        if (reinterpret_cast<std::uintptr_t>(src) % 8) raise(Errc::InvalidArgument, "digest needs 8-byte alignment");
        check_cuda(launch_digest(src, len, word_offset, out, static_cast<cudaStream_t>(stream)), "digest");
    });
}

int pyrit_set_lanes(uint32_t lanes) {
    return guarded([&] { set_preferred_lanes(lanes); });
}

int pyrit_set_kernel_mode(int mode) {
    return guarded([&] { set_kernel_mode(mode); });
}

int pyrit_set_kernel_dir(const char* dir) {
    return guarded([&] { set_kernel_dir(dir ? dir : ""); });
}

int pyrit_cu_last_launch(char* kernel, size_t cap, uint32_t* blocks, uint32_t* threads) {
    return guarded([&] {
        const LaunchInfo li = last_launch();
        if (kernel && cap) {
            const size_t n = std::min(cap - 1, li.kernel.size());
            std::memcpy(kernel, li.kernel.data(), n);
            kernel[n] = 0;
        }
        if (blocks) *blocks = li.blocks;
        if (threads) *threads = li.threads;
    });
}

int pyrit_jit_wait(void) {
    return guarded([&] { jit_wait(); });
}

int pyrit_jit_info(char* buf, size_t cap) {
    return guarded([&] {
        if (!buf || !cap) raise(Errc::InvalidArgument, "null buffer");
        const std::string s = jit_info();
        const size_t n = std::min(cap - 1, s.size());
        std::memcpy(buf, s.data(), n);
        buf[n] = 0;
    });
}

uint64_t pyrit_jit_compiles(void) { return jit_compiles(); }
int pyrit_jit_time(double* last_ms, double* total_ms) {
    jit_time(last_ms, total_ms);
    return 0;
}
uint64_t pyrit_kernel_launches(void) { return kernel_launches(); }

int pyrit_warmup(int device) {
    return guarded([&] {
        check_cuda(cudaSetDevice(device), "cudaSetDevice");
        check_cuda(warm_ring_rt(), "runtime-matrix kernel modules");
    });
}

} // extern "C"
