#include "program.hpp"

#include <algorithm>
#include <bit>
#include <cstdio>
#include <cstring>
#include <sstream>

namespace pyrit_b200 {

std::uint64_t fnv1a(const std::string& s) {
    std::uint64_t h = 1469598103934665603ull;
    for (unsigned char c : s) {
        h ^= c;
        h *= 1099511628211ull;
    }
    return h;
}

namespace {

constexpr std::uint32_t kNone = 0xFFFFFFFFu;

// Greedy pair elimination over XOR targets.  Each target is a set of
// variable ids; the most frequent pair (ties: smallest ids) becomes a new
// temporary t = a ^ b substituted into every target holding both, until
// no pair is shared.  Emits the temporaries into `code`.
void share_pairs(std::vector<std::vector<std::uint32_t>>& targets, std::uint32_t& nvars,
                 std::vector<Instr>& code) {
    for (;;) {
        std::vector<std::uint32_t> ids;
        for (auto& t : targets) ids.insert(ids.end(), t.begin(), t.end());
        std::sort(ids.begin(), ids.end());
        ids.erase(std::unique(ids.begin(), ids.end()), ids.end());
        const std::size_t v = ids.size();
        if (v < 2) return;
        std::vector<std::uint16_t> count(v * v, 0);
        std::vector<std::uint32_t> local;
        for (auto& t : targets) {
            local.clear();
            for (std::uint32_t x : t)
                local.push_back(static_cast<std::uint32_t>(std::lower_bound(ids.begin(), ids.end(), x) - ids.begin()));
            std::sort(local.begin(), local.end());
            for (std::size_t a = 0; a < local.size(); ++a)
                for (std::size_t b = a + 1; b < local.size(); ++b) ++count[local[a] * v + local[b]];
        }
        std::size_t best = 0;
        std::uint16_t best_c = 1;
        for (std::size_t i = 0; i < v * v; ++i)
            if (count[i] > best_c) {
                best_c = count[i];
                best = i;
            }
        if (best_c < 2) return;
        const std::uint32_t a = ids[best / v], b = ids[best % v];
        const std::uint32_t t = nvars++;
        code.push_back(Instr{Instr::Xor, t, 0, 0, {a, b}});
        for (auto& tg : targets) {
            auto ia = std::find(tg.begin(), tg.end(), a);
            auto ib = std::find(tg.begin(), tg.end(), b);
            if (ia == tg.end() || ib == tg.end()) continue;
            tg.erase(std::remove_if(tg.begin(), tg.end(), [&](std::uint32_t x) { return x == a || x == b; }),
                     tg.end());
            tg.push_back(t);
        }
    }
}

void toggle(std::vector<std::uint32_t>& set, std::uint32_t x) {
    auto it = std::find(set.begin(), set.end(), x);
    if (it == set.end()) set.push_back(x);
    else set.erase(it);
}

} // namespace

Program compile_program(const Field& f, TransformKind kind, const Matrix& m, const CompileOptions& opt) {
    validate_field(f);
    if (m.cols == 0) raise(Errc::InvalidArgument, "matrix has no columns");
    Program p;
    p.field = f;
    p.kind = kind;
    p.rows = m.rows;
    p.cols = m.cols;
    const std::uint32_t w = f.w, n = f.n, k = m.cols, e = m.rows;
    p.group = opt.group ? opt.group : std::max<std::uint32_t>(1, 24 / w);
    p.group = std::min(p.group, k);
    p.fold = fold_table(f);
    p.reps.resize(std::size_t(e) * k);
    for (std::size_t i = 0; i < p.reps.size(); ++i) {
        if (m.e[i] >= f.field_size()) raise(Errc::InvalidArgument, "matrix entry outside the field");
        p.reps[i] = opt.dense ? dense_transform(m.e[i], f) : sparse_transform(m.e[i], f);
        p.stats.matrix_ones += std::uint64_t(std::popcount(p.reps[i])) * w;
    }

    const bool emb = kind == TransformKind::Embedding;
    const std::uint32_t out_rows = emb ? n : w; // schedule.hpp:132

    // reference op count (compile_schedule), generalized post phase
    {
        std::uint64_t ops = 0;
        if (!emb)
            for (std::uint32_t t = 0; t < n - w; ++t)
                for (std::uint32_t i = t; i < w; i += f.s) ops += k;
        for (std::uint32_t i = 0; i < e; ++i)
            for (std::uint32_t t = 0; t < out_rows; ++t) {
                std::uint64_t row = 0;
                for (std::uint32_t j = 0; j < k; ++j)
                    for (std::uint32_t sh = 0; sh < n; ++sh)
                        if ((p.reps[i * k + j] >> sh) & 1u) {
                            const std::uint32_t src = (t + n - sh) % n;
                            if (emb && src >= w) continue;
                            ++row;
                        }
                ops += row;
                if (!row && t < w) ++ops;
            }
        if (emb)
            for (std::uint32_t fv : p.fold) ops += std::uint64_t(std::popcount(fv)) * e;
        p.stats.ref_region_ops = ops;
    }

    // strips of input j that ring position src reads (Parity: the
    // pre-phase column parities, schedule.hpp:115-130, substituted)
    auto strips_of = [&](std::uint32_t src) {
        std::vector<std::uint32_t> out;
        if (src < w) out.push_back(src);
        else if (!emb)
            for (std::uint32_t i = src - w; i < w; i += f.s) out.push_back(i);
        return out;
    };

    std::uint32_t nvars = 0;
    std::vector<std::uint32_t> acc(std::size_t(e) * out_rows, kNone);
    std::vector<std::vector<Instr>> loads, compute;
    for (std::uint32_t g0 = 0; g0 < k; g0 += p.group) {
        const std::uint32_t g1 = std::min(k, g0 + p.group);
        std::vector<Instr> ld, cp;
        std::vector<std::uint32_t> var_of(std::size_t(g1 - g0) * w);
        for (std::uint32_t j = g0; j < g1; ++j)
            for (std::uint32_t s = 0; s < w; ++s) {
                var_of[(j - g0) * w + s] = nvars;
                ld.push_back(Instr{Instr::Load, nvars++, j, s, {}});
            }
        std::vector<std::vector<std::uint32_t>> targets(std::size_t(e) * out_rows);
        for (std::uint32_t i = 0; i < e; ++i)
            for (std::uint32_t t = 0; t < out_rows; ++t) {
                auto& tg = targets[i * out_rows + t];
                for (std::uint32_t j = g0; j < g1; ++j)
                    for (std::uint32_t sh = 0; sh < n; ++sh)
                        if ((p.reps[i * k + j] >> sh) & 1u)
                            for (std::uint32_t s : strips_of((t + n - sh) % n)) toggle(tg, var_of[(j - g0) * w + s]);
                std::sort(tg.begin(), tg.end());
                p.stats.naive_xors += tg.size(); // one XOR per term into the row...
            }
        if (opt.cse) share_pairs(targets, nvars, cp);
        for (std::size_t r = 0; r < targets.size(); ++r) {
            auto& tg = targets[r];
            if (tg.empty()) continue;
            if (acc[r] == kNone && tg.size() == 1) {
                acc[r] = tg[0];
                continue;
            }
            Instr x{Instr::Xor, nvars++, 0, 0, {}};
            if (acc[r] != kNone) x.src.push_back(acc[r]);
            x.src.insert(x.src.end(), tg.begin(), tg.end());
            acc[r] = x.dst;
            cp.push_back(std::move(x));
        }
        loads.push_back(std::move(ld));
        compute.push_back(std::move(cp));
    }
    // ...minus the first write of every row (a copy, not an XOR)
    for (std::uint32_t r = 0; r < acc.size(); ++r)
        if (acc[r] != kNone) --p.stats.naive_xors;

    // order: prefetch group g+1's strips before computing group g
    for (std::size_t g = 0; g < loads.size(); ++g) {
        if (g == 0) p.code.insert(p.code.end(), loads[0].begin(), loads[0].end());
        if (g + 1 < loads.size()) p.code.insert(p.code.end(), loads[g + 1].begin(), loads[g + 1].end());
        p.code.insert(p.code.end(), compute[g].begin(), compute[g].end());
    }

    // inverse transform and stores
    for (std::uint32_t i = 0; i < e; ++i) {
        std::vector<std::vector<std::uint32_t>> targets(w);
        for (std::uint32_t b = 0; b < w; ++b) {
            if (acc[i * out_rows + b] != kNone) targets[b].push_back(acc[i * out_rows + b]);
            if (emb)
                for (std::uint32_t t = w; t < n; ++t)
                    if (((p.fold[t - w] >> b) & 1u) && acc[i * out_rows + t] != kNone) {
                        targets[b].push_back(acc[i * out_rows + t]);
                        ++p.stats.naive_xors;
                    }
            if (!targets[b].empty() && acc[i * out_rows + b] == kNone) --p.stats.naive_xors;
        }
        if (opt.cse) share_pairs(targets, nvars, p.code);
        for (std::uint32_t b = 0; b < w; ++b) p.code.push_back(Instr{Instr::Store, 0, i, b, targets[b]});
    }
    p.nvars = nvars;
    for (const Instr& in : p.code) {
        if (in.op == Instr::Load) ++p.stats.loads;
        if (in.op == Instr::Store) ++p.stats.stores;
        if (in.op != Instr::Load && in.src.size() > 1) p.stats.xors += in.src.size() - 1;
    }
    p.stats.vars = nvars;
    return p;
}

void interpret_program(const Program& p, const std::uint8_t* const* in, std::uint8_t* const* out,
                       std::uint64_t strip, std::uint64_t off, std::uint64_t len) {
    constexpr std::uint64_t kBlock = 512;
    std::vector<std::uint8_t> vars(std::size_t(p.nvars) * kBlock);
    for (std::uint64_t pos = off; pos < off + len; pos += kBlock) {
        const std::uint64_t b = std::min<std::uint64_t>(kBlock, off + len - pos);
        for (const Instr& ins : p.code) {
            if (ins.op == Instr::Load) {
                std::memcpy(&vars[std::size_t(ins.dst) * kBlock], in[ins.sym] + ins.strip * strip + pos, b);
                continue;
            }
            std::uint8_t* d = ins.op == Instr::Xor ? &vars[std::size_t(ins.dst) * kBlock]
                                                   : out[ins.sym] + ins.strip * strip + pos;
            if (ins.src.empty()) {
                std::memset(d, 0, b);
                continue;
            }
            std::vector<std::uint8_t> acc(vars.begin() + std::size_t(ins.src[0]) * kBlock,
                                          vars.begin() + std::size_t(ins.src[0]) * kBlock + b);
            for (std::size_t s = 1; s < ins.src.size(); ++s) {
                const std::uint8_t* x = &vars[std::size_t(ins.src[s]) * kBlock];
                for (std::uint64_t q = 0; q < b; ++q) acc[q] ^= x[q];
            }
            std::memcpy(d, acc.data(), b);
        }
    }
}

std::string kernel_name(const Program& p, const KernelShape& ks) {
    std::ostringstream fp;
    fp << p.field.w << ',' << p.field.n << ',' << p.field.modulus << ',' << int(p.kind) << ',' << p.rows << ','
       << p.cols << ',' << p.group << ',' << ks.lanes << ',' << ks.threads << ',' << ks.min_blocks << ':';
    for (std::uint32_t r : p.reps) fp << r << ',';
    char name[96];
    std::snprintf(name, sizeof name, "pyrit_ring_k%u_e%u_w%u_n%u_L%u_%016llx", p.cols, p.rows, p.field.w,
                  p.field.n, ks.lanes, static_cast<unsigned long long>(fnv1a(fp.str())));
    return name;
}

std::string generate_cuda(const Program& p, const KernelShape& ks) {
    const std::uint32_t L = ks.lanes == 0 ? 1 : ks.lanes;
    const bool bytes = ks.lanes == 0;
    const std::uint32_t V = bytes ? 1 : 4 * L; // bytes per thread per strip
    std::ostringstream o;
    o << "// generated by pyrit_b200 program compiler: field w=" << p.field.w << " n=" << p.field.n << " p=0x"
      << std::hex << p.field.modulus << std::dec << ", " << p.rows << "x" << p.cols << " ring matrix, "
      << p.stats.xors << " XORs (naive ring program " << p.stats.naive_xors << ", reference schedule "
      << p.stats.ref_region_ops << " region ops)\n";
    o << "typedef unsigned int u32; typedef unsigned long long u64; typedef unsigned char u8;\n";
    o << "struct Args { const u8* in[" << p.cols << "]; u8* out[" << p.rows << "]; u64 S; u64 off; u64 nwords; };\n";
    // loads: read-only, no L1 allocation (streamed once); stores: evict-first
    if (bytes) {
        o << "#define LD(v, p) asm(\"ld.global.nc.L1::no_allocate.u8 %0, [%1];\" : \"=r\"(v) : \"l\"(p))\n";
        o << "#define ST(p, v) asm volatile(\"st.global.cs.u8 [%0], %1;\" :: \"l\"(p), \"r\"(v) : \"memory\")\n";
    } else if (L == 1) {
        o << "#define LD(v, p) asm(\"ld.global.nc.L1::no_allocate.b32 %0, [%1];\" : \"=r\"(v##_0) : \"l\"(p))\n";
        o << "#define ST(p, v) asm volatile(\"st.global.cs.b32 [%0], %1;\" :: \"l\"(p), \"r\"(v##_0) : \"memory\")\n";
    } else if (L == 2) {
        o << "#define LD(v, p) asm(\"ld.global.nc.L1::no_allocate.v2.b32 {%0, %1}, [%2];\" : \"=r\"(v##_0), "
             "\"=r\"(v##_1) : \"l\"(p))\n";
        o << "#define ST(p, v) asm volatile(\"st.global.cs.v2.b32 [%0], {%1, %2};\" :: \"l\"(p), \"r\"(v##_0), "
             "\"r\"(v##_1) : \"memory\")\n";
    } else {
        o << "#define LD(v, p) asm(\"ld.global.nc.L1::no_allocate.v4.b32 {%0, %1, %2, %3}, [%4];\" : "
             "\"=r\"(v##_0), \"=r\"(v##_1), \"=r\"(v##_2), \"=r\"(v##_3) : \"l\"(p))\n";
        o << "#define ST(p, v) asm volatile(\"st.global.cs.v4.b32 [%0], {%1, %2, %3, %4};\" :: \"l\"(p), "
             "\"r\"(v##_0), \"r\"(v##_1), \"r\"(v##_2), \"r\"(v##_3) : \"memory\")\n";
    }
    const std::string name = kernel_name(p, ks);
    o << "extern \"C\" __global__ void __launch_bounds__(" << ks.threads << ", " << ks.min_blocks << ") " << name
      << "(const Args a)\n{\n";
    o << "  const u64 S = a.S;\n";
    o << "  const u64 stride = (u64)gridDim.x * " << ks.threads << "u;\n";
    o << "  for (u64 c = (u64)blockIdx.x * " << ks.threads << "u + threadIdx.x; c < a.nwords; c += stride) {\n";
    o << "    const u64 o = a.off + c * " << V << "u;\n";
    auto var = [&](std::uint32_t v, std::uint32_t l) {
        std::string s = "v" + std::to_string(v);
        if (!bytes) s += "_" + std::to_string(l);
        return s;
    };
    std::vector<bool> frag_ptr(p.cols, false), out_ptr(p.rows, false);
    for (const Instr& ins : p.code) {
        if (ins.op == Instr::Load) {
            if (!frag_ptr[ins.sym]) {
                o << "    const u8* i" << ins.sym << " = a.in[" << ins.sym << "] + o;\n";
                frag_ptr[ins.sym] = true;
            }
            o << "    u32 ";
            for (std::uint32_t l = 0; l < L; ++l) o << (l ? ", " : "") << var(ins.dst, l);
            o << "; LD(v" << ins.dst << ", i" << ins.sym;
            if (ins.strip) o << " + " << ins.strip << "u * S";
            o << ");\n";
        } else if (ins.op == Instr::Xor) {
            for (std::uint32_t l = 0; l < L; ++l) {
                o << "    const u32 " << var(ins.dst, l) << " = ";
                for (std::size_t s = 0; s < ins.src.size(); ++s) o << (s ? " ^ " : "") << var(ins.src[s], l);
                o << ";\n";
            }
        } else {
            if (!out_ptr[ins.sym]) {
                o << "    u8* q" << ins.sym << " = a.out[" << ins.sym << "] + o;\n";
                out_ptr[ins.sym] = true;
            }
            o << "    { u32 ";
            for (std::uint32_t l = 0; l < L; ++l) {
                o << (l ? ", " : "") << "x" << (bytes ? "" : "_" + std::to_string(l)) << " = ";
                if (ins.src.empty()) o << "0u";
                for (std::size_t s = 0; s < ins.src.size(); ++s) o << (s ? " ^ " : "") << var(ins.src[s], l);
            }
            o << "; ST(q" << ins.sym;
            if (ins.strip) o << " + " << ins.strip << "u * S";
            o << ", x); }\n";
        }
    }
    o << "  }\n}\n";
    return o.str();
}

} // namespace pyrit_b200
