#include "program.hpp"

#include <algorithm>
#include <bit>
#include <cstdio>
#include <dlfcn.h>

#include <cstdlib>
#include <cstring>
#include <mutex>
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
// bump whenever generated code changes for the same program (prebuilt cubins are keyed by name)
constexpr int kGeneratorVersion = 15;

// Greedy pair elimination over XOR targets.  Each target is a set of
// variable ids; the most frequent pair (ties: smallest ids) becomes a new
// temporary t = a ^ b substituted into every target holding both, until
// no pair is shared.  Emits the temporaries into `code`.
void share_pairs(std::vector<std::vector<std::uint32_t>>& targets, std::uint32_t& nvars,
                 std::vector<Instr>& code, std::uint32_t max_temps = 0) {
    for (std::uint32_t made = 0; !max_temps || made < max_temps; ++made) {
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

// Reorder so that every pair temporary (the first `ntemps` instructions,
// as emitted by share_pairs) is defined right before its first use; keeps
// the live range of shared sub-sums short.
void lazy_order(std::vector<Instr>& code, std::size_t ntemps) {
    std::vector<Instr> out;
    out.reserve(code.size());
    std::vector<std::size_t> def_of;
    std::uint32_t lo = 0xFFFFFFFFu, hi = 0;
    for (std::size_t i = 0; i < ntemps; ++i) {
        lo = std::min(lo, code[i].dst);
        hi = std::max(hi, code[i].dst + 1);
    }
    if (ntemps) def_of.assign(hi - lo, SIZE_MAX);
    for (std::size_t i = 0; i < ntemps; ++i) def_of[code[i].dst - lo] = i;
    std::vector<bool> done(ntemps, false);
    std::vector<std::size_t> stack;
    auto emit_deps = [&](const Instr& ins, auto&& self) -> void {
        for (std::uint32_t v : ins.src)
            if (ntemps && v >= lo && v < hi && def_of[v - lo] != SIZE_MAX && !done[def_of[v - lo]]) {
                const std::size_t d = def_of[v - lo];
                done[d] = true;
                self(code[d], self);
                out.push_back(code[d]);
            }
    };
    for (std::size_t i = ntemps; i < code.size(); ++i) {
        emit_deps(code[i], emit_deps);
        out.push_back(code[i]);
    }
    for (std::size_t i = 0; i < ntemps; ++i)
        if (!done[i]) out.push_back(code[i]);
    code.swap(out);
}

} // namespace

std::string plan_key(const Program& p) {
    std::ostringstream fp;
    fp << p.field.w << ',' << p.field.n << ',' << p.field.modulus << ',' << int(p.kind) << ',' << p.rows << ','
       << p.cols << ':';
    for (std::uint32_t r : p.reps) fp << r << ',';
    if (p.sched) { // schedule programs: the linear map itself
        for (std::uint32_t b : p.bits) fp << 'b' << b;
        for (std::uint8_t x : p.written) fp << int(x);
    } else if (p.crs) // bitmatrix programs depend on the matrix itself, not on representatives
        for (std::uint16_t x : p.matrix) fp << 'c' << x;
    char key[64];
    std::snprintf(key, sizeof key, "w%un%u_%ux%u%s_%016llx", p.field.w, p.field.n, p.rows, p.cols,
                  p.sched ? "sch" : p.crs ? "crs" : "",
                  static_cast<unsigned long long>(fnv1a(fp.str())));
    return key;
}

namespace {
std::mutex g_tuned_mu;
std::string g_tuned_path;
std::vector<TunedEntry> g_tuned;
bool g_tuned_loaded = false;

std::string library_dir() {
    Dl_info info{};
    if (dladdr(reinterpret_cast<void*>(&library_dir), &info) && info.dli_fname) {
        std::string so = info.dli_fname;
        const auto slash = so.rfind('/');
        return slash == std::string::npos ? std::string(".") : so.substr(0, slash);
    }
    return ".";
}
} // namespace

void set_tuned_path(const std::string& path) {
    std::lock_guard<std::mutex> lk(g_tuned_mu);
    g_tuned_path = path;
    g_tuned_loaded = false;
}

const TunedEntry* find_tuned(const std::string& key) {
    std::lock_guard<std::mutex> lk(g_tuned_mu);
    if (!g_tuned_loaded) {
        g_tuned_loaded = true;
        g_tuned.clear();
        std::string path = g_tuned_path.empty() ? library_dir() + "/tuned.tsv" : g_tuned_path;
        if (const char* env = std::getenv("PYRIT_B200_TUNED")) path = env;
        if (!path.empty())
            if (FILE* fh = std::fopen(path.c_str(), "r")) {
                char line[512];
                while (std::fgets(line, sizeof line, fh)) {
                    if (line[0] == '#' || line[0] == '\n') continue;
                    char k[128];
                    unsigned parts = 0, pg = 0, threads = 0, producer = 0;
                    int cse = -1;
                    const int got =
                        std::sscanf(line, "%127s %u %u %d %u %u", k, &parts, &pg, &cse, &threads, &producer);
                    if (got >= 4)
                        g_tuned.push_back(TunedEntry{k, parts, pg, cse, got >= 5 ? threads : 0u, got >= 6 ? producer : 0u});
                }
                std::fclose(fh);
            }
    }
    // the table is only written at load time; later lookups are read-only
    for (const TunedEntry& t : g_tuned)
        if (t.key == key) return &t;
    return nullptr;
}

namespace {

void hash_instrs(std::uint64_t& h, const std::vector<Instr>& v) {
    auto mix = [&](std::uint64_t x) {
        for (int b = 0; b < 8; ++b) {
            h ^= (x >> (8 * b)) & 0xFF;
            h *= 1099511628211ull;
        }
    };
    mix(v.size());
    for (const Instr& in : v) {
        mix((std::uint64_t(in.op) << 56) ^ (std::uint64_t(in.dst) << 24) ^ (std::uint64_t(in.sym) << 8) ^ in.strip);
        mix(in.src.size());
        for (std::uint32_t x : in.src) mix(x);
    }
}

std::uint64_t ir_hash_of(const Program& p) {
    std::uint64_t h = 1469598103934665603ull;
    hash_instrs(h, p.code);
    for (const Program& q : p.parts) {
        for (const auto& g : q.group_loads) hash_instrs(h, g);
        for (const auto& g : q.group_compute) hash_instrs(h, g);
        hash_instrs(h, q.tail);
    }
    return h;
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
    p.cse = opt.cse;
    p.crs = opt.crs || opt.bits;
    // (p.cse is revised below for very large programs: greedy pair sharing is
    // superlinear in the terms per fragment group)
    p.sched = opt.bits != nullptr;
    p.matrix = m.e;
    p.fold = fold_table(f);
    p.reps.resize(std::size_t(e) * k);
    for (std::size_t i = 0; i < p.reps.size(); ++i) {
        if (m.e[i] >= f.field_size()) raise(Errc::InvalidArgument, "matrix entry outside the field");
        p.reps[i] = opt.reps ? (*opt.reps)[i] & f.ring_mask()
                    : opt.dense ? dense_transform(m.e[i], f) : sparse_transform(m.e[i], f);
        p.stats.matrix_ones += std::uint64_t(std::popcount(p.reps[i])) * w;
    }
    // CRS: the w x w bitmatrix of every entry (field_to_bitmatrix, field.hpp:198-207):
    // column c = coefficients of entry * x^c; rows[b] = mask of input strips feeding output strip b
    std::vector<std::uint32_t> bits;
    if (opt.bits) { // explicit linear map (compile_schedule_program)
        if (opt.bits->size() != std::size_t(e) * k * w || !opt.written || opt.written->size() != std::size_t(e) * w)
            raise(Errc::InvalidArgument, "bit matrix shape");
        bits = *opt.bits;
        p.bits = bits;
        p.written = *opt.written;
        p.stats.matrix_ones = 0;
        for (std::uint32_t b : bits) p.stats.matrix_ones += std::popcount(b);
    } else if (opt.crs) {
        if (kind != TransformKind::Embedding) raise(Errc::InvalidArgument, "CRS programs are plain field codes");
        bits.assign(std::size_t(e) * k * w, 0);
        p.stats.matrix_ones = 0;
        for (std::size_t idx = 0; idx < std::size_t(e) * k; ++idx)
            for (std::uint32_t c = 0; c < w; ++c) {
                const std::uint32_t prod = gf_mul(m.e[idx], 1u << c, f);
                for (std::uint32_t b = 0; b < w; ++b)
                    if ((prod >> b) & 1u) {
                        bits[idx * w + b] |= 1u << c;
                        ++p.stats.matrix_ones;
                    }
            }
    }

    // Pair sharing costs time superlinear in the program size and its
    // temporaries only serve the unsplit kernels; very large codes (more than
    // ~200k ring-matrix ones, e.g. k = 100, r = 50 over GF(2^12)) run split
    // into output parts, which do not share pairs, so skip it there.
    if (p.stats.matrix_ones > 200000) p.cse = false;
    const bool emb = kind == TransformKind::Embedding;
    const bool crs = p.crs;
    const std::uint32_t out_rows = emb && !crs ? n : w; // schedule.hpp:132 (CRS: w bit rows)

    // reference op count (compile_schedule), generalized post phase
    {
        std::uint64_t ops = 0;
        if (crs && !p.sched) // compile_crs_schedule (schedule.hpp:186-201): one op per bitmatrix one, Zero for empty rows
            for (std::uint32_t i = 0; i < e; ++i)
                for (std::uint32_t b = 0; b < w; ++b) {
                    std::uint64_t row = 0;
                    for (std::uint32_t j = 0; j < k; ++j) row += std::popcount(bits[(std::size_t(i) * k + j) * w + b]);
                    ops += row ? row : 1;
                }
        if (!emb && !crs)
            for (std::uint32_t t = 0; t < n - w; ++t)
                for (std::uint32_t i = t; i < w; i += f.s) ops += k;
        for (std::uint32_t i = 0; i < (crs ? 0u : e); ++i)
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
        if (emb && !crs)
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
                    if (crs) {
                        const std::uint32_t row = bits[(std::size_t(i) * k + j) * w + t];
                        for (std::uint32_t c = 0; c < w; ++c)
                            if ((row >> c) & 1u) toggle(tg, var_of[(j - g0) * w + c]);
                    } else {
                        for (std::uint32_t sh = 0; sh < n; ++sh)
                            if ((p.reps[i * k + j] >> sh) & 1u)
                                for (std::uint32_t s : strips_of((t + n - sh) % n)) toggle(tg, var_of[(j - g0) * w + s]);
                    }
                std::sort(tg.begin(), tg.end());
                p.stats.naive_xors += tg.size(); // one XOR per term into the row...
            }
        if (p.cse) {
            // pair sharing over windows of cse_window consecutive targets (ring
            // rows, output by output); 0 = the whole group.  Small windows keep
            // shared temporaries short-lived (register pressure)
            const std::size_t win = opt.cse_window ? opt.cse_window : targets.size();
            for (std::size_t w0 = 0; w0 < targets.size(); w0 += win) {
                const std::size_t w1 = std::min(targets.size(), w0 + win);
                std::vector<std::vector<std::uint32_t>> sub(targets.begin() + w0, targets.begin() + w1);
                share_pairs(sub, nvars, cp, opt.max_temps);
                std::copy(sub.begin(), sub.end(), targets.begin() + w0);
            }
        }
        const std::size_t ntemps = cp.size();
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
        lazy_order(cp, ntemps);
        loads.push_back(std::move(ld));
        compute.push_back(std::move(cp));
    }
    // ...minus the first write of every row (a copy, not an XOR)
    for (std::uint32_t r = 0; r < acc.size(); ++r)
        if (acc[r] != kNone) --p.stats.naive_xors;

    // order: prefetch group g+1's strips before computing group g
    for (std::size_t g = 0; g < loads.size(); ++g) {
        if (g == 0) p.code.insert(p.code.end(), loads[0].begin(), loads[0].end());
        // (direct mode) issue the next group's HBM loads before this group's XORs
        if (g + 1 < loads.size()) p.code.insert(p.code.end(), loads[g + 1].begin(), loads[g + 1].end());
        p.code.insert(p.code.end(), compute[g].begin(), compute[g].end());
    }

    // inverse transform and stores
    for (std::uint32_t i = 0; i < e; ++i) {
        std::vector<std::vector<std::uint32_t>> targets(w);
        for (std::uint32_t b = 0; b < w; ++b) {
            // toggle, not append: two ring rows can be the same variable (a row
            // that is a single input strip aliases the load), and x ^ x = 0
            if (acc[i * out_rows + b] != kNone) toggle(targets[b], acc[i * out_rows + b]);
            if (emb && !crs)
                for (std::uint32_t t = w; t < n; ++t)
                    if (((p.fold[t - w] >> b) & 1u) && acc[i * out_rows + t] != kNone) {
                        toggle(targets[b], acc[i * out_rows + t]);
                        ++p.stats.naive_xors;
                    }
            if (!targets[b].empty() && acc[i * out_rows + b] == kNone) --p.stats.naive_xors;
        }
        std::vector<Instr> fold;
        if (p.cse) share_pairs(targets, nvars, fold);
        const std::size_t ntemps = fold.size();
        for (std::uint32_t b = 0; b < w; ++b)
            if (!p.sched || p.written[std::size_t(i) * w + b]) fold.push_back(Instr{Instr::Store, 0, i, b, targets[b]});
        lazy_order(fold, ntemps);
        p.code.insert(p.code.end(), fold.begin(), fold.end());
        p.tail.insert(p.tail.end(), fold.begin(), fold.end());
    }
    p.group_loads = std::move(loads);
    p.group_compute = std::move(compute);
    p.nvars = nvars;
    for (const Instr& in : p.code) {
        if (in.op == Instr::Load) ++p.stats.loads;
        if (in.op == Instr::Store) ++p.stats.stores;
        if (in.op != Instr::Load && in.src.size() > 1) p.stats.xors += in.src.size() - 1;
    }
    p.stats.vars = nvars;

    // Output parts of the staged kernel (see KernelShape).  Knobs, in order
    // of precedence: CompileOptions, PYRIT_B200_PARTS / _PART_GROUP /
    // _PART_CSE / _THREADS, the measured tuning table (tuned.tsv next to the
    // library), and the heuristic: the fewest parts that keep <= 64 ring-row
    // accumulators per thread; fragment groups of about 48 strips; no pair
    // sharing (its temporaries lengthen live ranges and spill); 512 threads
    // per CTA when a part's live words (accumulators + one group's strips)
    // fit the 128 registers that allows, else 256.
    if (opt.parts != 1 && e > 0) {
        const auto env_u = [](const char* name) -> int {
            const char* v = std::getenv(name);
            return v ? std::atoi(v) : -1;
        };
        const TunedEntry* tuned = find_tuned(plan_key(p));
        p.staged_threads = opt.staged_threads;
        if (!p.staged_threads && env_u("PYRIT_B200_THREADS") > 0)
            p.staged_threads = static_cast<std::uint32_t>(env_u("PYRIT_B200_THREADS"));
        if (!p.staged_threads && tuned) p.staged_threads = tuned->threads;
        if (tuned) p.staged_producer = tuned->producer;
        std::uint32_t R = opt.parts;
        if (!R && env_u("PYRIT_B200_PARTS") > 0) R = static_cast<std::uint32_t>(env_u("PYRIT_B200_PARTS"));
        if (!R && tuned) R = tuned->parts;
        const std::uint32_t acc_rows = emb && !crs ? n : w; // accumulators per output row
        // Heuristic (measured on the BASELINE codes and the paper's (60,40) /
        // (60,20) GF(2^6) codes, profiles/r01_s2): the fewest parts -- every
        // part re-reads all input strips from shared memory -- that keep
        // <= 128 accumulators per thread; 512-thread CTAs when a part's
        // accumulators are few (<= 64), else 256 (255 registers); and the
        // largest fragment group whose slot still lets 3 slots fit in shared
        // memory, since every (tile, group) unit costs a barrier round trip.
        if (!R) { // a power of two (it must divide the CTA) no larger than e
            R = 1;
            while (2 * R <= e && (e + R - 1) / R * acc_rows > 128) R *= 2;
        }
        R = std::max<std::uint32_t>(1, std::min(R, e));
        const std::uint32_t acc = (e + R - 1) / R * acc_rows;
        if (!p.staged_threads) p.staged_threads = acc <= 64 ? 512 : 256;
        std::uint32_t pg = opt.part_group;
        if (!pg && env_u("PYRIT_B200_PART_GROUP") > 0) pg = static_cast<std::uint32_t>(env_u("PYRIT_B200_PART_GROUP"));
        if (!pg && tuned) pg = tuned->part_group;
        if (!pg) {
            const std::uint32_t tile = 4 * (p.staged_threads / R);
            pg = std::max<std::uint32_t>(1, (226u * 1024 / 3) / (w * tile));
            pg = std::min(pg, std::max<std::uint32_t>(1, 160 / w));
        }
        pg = std::max<std::uint32_t>(1, std::min(pg, k));
        int pcse = env_u("PYRIT_B200_PART_CSE");
        if (pcse < 0 && tuned) pcse = tuned->part_cse;
        // Parity transform: every input's column parities (ring positions
        // >= w) are XORs of its data strips, so expanded ring rows repeat the
        // same pairs; sharing them within one output's rows (short-lived
        // temporaries) pays: (60,20) GF(2^6) parity code 1.57x
        // (profiles/r01_s3/cse/); for the embedding codes it does not
        const bool parity = !emb && !crs;
        if (pcse < 0) pcse = parity ? 1 : 0;
        const bool parity_cse = parity && pcse;
        auto build_parts = [&](bool cse) {
            p.parts.clear();
            p.part_row0.clear();
            for (std::uint32_t r = 0, row0 = 0; r < R; ++r) {
                const std::uint32_t nrows = e / R + (r < e % R ? 1 : 0);
                Matrix sub(nrows, k);
                for (std::uint32_t i = 0; i < nrows; ++i)
                    for (std::uint32_t j = 0; j < k; ++j) sub.at(i, j) = m.at(row0 + i, j);
                CompileOptions o2 = opt;
                std::vector<std::uint32_t> sub_bits;
                std::vector<std::uint8_t> sub_written;
                if (opt.bits) {
                    sub_bits.assign(opt.bits->begin() + std::size_t(row0) * k * w,
                                    opt.bits->begin() + std::size_t(row0 + nrows) * k * w);
                    sub_written.assign(opt.written->begin() + std::size_t(row0) * w,
                                       opt.written->begin() + std::size_t(row0 + nrows) * w);
                    o2.bits = &sub_bits;
                    o2.written = &sub_written;
                }
                o2.parts = 1;
                o2.group = pg;
                o2.cse = cse && opt.cse;
                if (const char* env = std::getenv("PYRIT_B200_PART_TEMPS")) o2.max_temps = std::atoi(env);
                if (const char* env = std::getenv("PYRIT_B200_CSE_WINDOW")) o2.cse_window = std::atoi(env);
                else if (parity_cse) o2.cse_window = w; // one output's rows
                p.parts.push_back(compile_program(f, kind, sub, o2));
                p.part_row0.push_back(row0);
                row0 += nrows;
            }
        };
        build_parts(pcse != 0);
    }
    // the generic kernel's bitmatrix (field code: every transform computes it)
    const bool all_written = !p.sched || std::all_of(p.written.begin(), p.written.end(), [](std::uint8_t x) { return x; });
    if (all_written && w <= 16 && e > 0) {
        p.field_masks.assign(std::size_t(e) * w * k, 0);
        if (emb || p.sched) { // the GF(2^w) code itself (embedding == plain field code), or the schedule's map
            for (std::uint32_t i = 0; i < e; ++i)
                for (std::uint32_t j = 0; j < k; ++j) {
                    std::uint32_t prod[16] = {};
                    if (!p.sched)
                        for (std::uint32_t c = 0; c < w; ++c) prod[c] = gf_mul(m.at(i, j), 1u << c, f);
                    for (std::uint32_t b = 0; b < w; ++b) {
                        std::uint32_t mask = 0;
                        if (p.sched) mask = p.bits[(std::size_t(i) * k + j) * w + b];
                        else
                            for (std::uint32_t c = 0; c < w; ++c) mask |= ((prod[c] >> b) & 1u) << c;
                        p.field_masks[(std::size_t(i) * w + b) * k + j] = static_cast<std::uint16_t>(mask);
                    }
                }
        } else if (std::uint64_t(p.stats.xors + 1) * k * w <= (std::uint64_t(1) << 26)) {
            // Parity transform: its own GF(2)-linear map -- read it off the program
            // with unit inputs, 8 at a time (one per bit of a 1-byte strip)
            const std::uint32_t units = k * w;
            std::vector<std::vector<std::uint8_t>> in(k, std::vector<std::uint8_t>(w)), out(e, std::vector<std::uint8_t>(w));
            std::vector<const std::uint8_t*> ip(k);
            std::vector<std::uint8_t*> op(e);
            for (std::uint32_t u0 = 0; u0 < units; u0 += 8) {
                for (auto& v : in) std::fill(v.begin(), v.end(), 0);
                for (std::uint32_t t = 0; t < 8 && u0 + t < units; ++t) in[(u0 + t) / w][(u0 + t) % w] |= 1u << t;
                for (std::uint32_t j = 0; j < k; ++j) ip[j] = in[j].data();
                for (std::uint32_t i = 0; i < e; ++i) op[i] = out[i].data();
                interpret_program(p, ip.data(), op.data(), 1, 0, 1);
                for (std::uint32_t i = 0; i < e; ++i)
                    for (std::uint32_t b = 0; b < w; ++b)
                        for (std::uint32_t t = 0; t < 8 && u0 + t < units; ++t)
                            if ((out[i][b] >> t) & 1u)
                                p.field_masks[(std::size_t(i) * w + b) * k + (u0 + t) / w] |=
                                    static_cast<std::uint16_t>(1u << ((u0 + t) % w));
            }
        } else {
            p.field_masks.clear(); // too large to read off: no generic kernel for this program
        }
    }
    p.ir_hash = ir_hash_of(p);
    p.key = plan_key(p);
    return p;
}

Program light_program(const Field& f, TransformKind kind, const Matrix& m) {
    validate_field(f);
    if (m.cols == 0) raise(Errc::InvalidArgument, "matrix has no columns");
    Program p;
    p.field = f;
    p.kind = kind;
    p.rows = m.rows;
    p.cols = m.cols;
    p.matrix = m.e;
    p.fold = fold_table(f);
    p.reps.resize(std::size_t(m.rows) * m.cols);
    for (std::size_t i = 0; i < p.reps.size(); ++i) {
        if (m.e[i] >= f.field_size()) raise(Errc::InvalidArgument, "matrix entry outside the field");
        p.reps[i] = sparse_transform(m.e[i], f);
        p.stats.matrix_ones += std::uint64_t(std::popcount(p.reps[i])) * f.w;
    }
    p.adhoc = true;
    p.light = true;
    p.key = plan_key(p);
    p.lazy = std::make_shared<LazyCompile>();
    return p;
}

Program ring_program(const Field& f, TransformKind kind, const std::uint32_t* reps, std::uint32_t rows,
                     std::uint32_t cols) {
    validate_field(f);
    if (cols == 0) raise(Errc::InvalidArgument, "matrix has no columns");
    if (rows == 0) raise(Errc::InvalidArgument, "matrix has no rows");
    Program p;
    p.field = f;
    p.kind = kind;
    p.rows = rows;
    p.cols = cols;
    p.fold = fold_table(f);
    p.reps.assign(reps, reps + std::size_t(rows) * cols);
    p.matrix.resize(p.reps.size());
    for (std::size_t i = 0; i < p.reps.size(); ++i) {
        if (f.n < 32 && (p.reps[i] >> f.n) != 0) raise(Errc::InvalidArgument, "ring element wider than n bits");
        // the field element this representative stands for: u mod p (phi_E^{-1} of u)
        p.matrix[i] = static_cast<std::uint16_t>(poly_mod(p.reps[i], f.modulus));
        // under the Parity transform the ring action is not a function of u mod p
        // alone (e.g. GF(2^8) in R_{2,17}), so only the canonical representative
        // (sparse_transform, ring.hpp:77-90) keeps every kernel path equal
        if (kind == TransformKind::Parity && p.reps[i] != sparse_transform(p.matrix[i], f))
            raise(Errc::InvalidArgument, "the Parity transform takes the canonical (sparse) representative of each entry");
        p.stats.matrix_ones += std::uint64_t(std::popcount(p.reps[i])) * f.w;
    }
    p.adhoc = true;
    p.light = true;
    p.key = plan_key(p);
    p.lazy = std::make_shared<LazyCompile>();
    return p;
}

const Program& full_program(const Program& p) {
    if (!p.light) return p;
    std::call_once(p.lazy->once, [&] {
        Matrix m(p.rows, p.cols);
        m.e = p.matrix;
        Program q = compile_program(p.field, p.kind, m, CompileOptions{});
        q.adhoc = true;
        p.lazy->prog = std::make_shared<const Program>(std::move(q));
    });
    return *p.lazy->prog;
}

ScheduleProgram compile_schedule_program(const Field& f, std::uint32_t k, std::uint32_t outputs,
                                         const std::vector<ScheduleOp>& ops, const std::vector<std::uint32_t>& labels,
                                         const CompileOptions& opt) {
    validate_field(f);
    const std::uint32_t w = f.w, n = f.n, slots = k + outputs;
    if (k == 0) raise(Errc::InvalidArgument, "schedule has no input slots");
    if (!labels.empty() && labels.size() != slots) raise(Errc::InvalidArgument, "one storage label per slot");
    // storage of every slot: distinct labels -> dense ids
    std::vector<std::uint32_t> store(slots);
    {
        std::vector<std::uint32_t> seen;
        for (std::uint32_t s = 0; s < slots; ++s) {
            const std::uint32_t lab = labels.empty() ? s : labels[s];
            auto it = std::find(seen.begin(), seen.end(), lab);
            store[s] = static_cast<std::uint32_t>(it - seen.begin());
            if (it == seen.end()) seen.push_back(lab);
        }
    }
    const std::uint32_t nstore = *std::max_element(store.begin(), store.end()) + 1;
    // GF(2) symbolic replay (codec.hpp:129-156): the value of every packet is
    // a set of initial packets (storage, strip), one bit each
    const std::size_t nv = std::size_t(nstore) * w, words = (nv + 63) / 64;
    // one bit vector per packet and scratch packet: keep the symbolic state bounded
    if ((nv + std::size_t(slots) * (n - w)) * words * 8 > (std::size_t(1) << 30))
        raise(Errc::InvalidArgument, "schedule has too many slots for symbolic replay");
    using Vec = std::vector<std::uint64_t>;
    std::vector<Vec> phys(nv, Vec(words, 0)), scratch(std::size_t(slots) * (n - w), Vec(words, 0));
    for (std::size_t v = 0; v < nv; ++v) phys[v][v / 64] |= 1ull << (v % 64);
    std::vector<std::uint8_t> wrote(nv, 0);
    const Vec zero(words, 0);
    for (const ScheduleOp& op : ops) {
        if (op.mode > 2) raise(Errc::InvalidArgument, "schedule op mode");
        if (op.dst_sym >= slots || op.dst_pkt >= n || (op.mode != 2 && (op.src_sym >= slots || op.src_pkt >= n)))
            raise(Errc::BufferShape, "replay: schedule slot out of range");
        Vec* dst;
        if (op.dst_pkt >= w) dst = &scratch[std::size_t(op.dst_sym) * (n - w) + op.dst_pkt - w];
        else if (op.dst_sym < k) raise(Errc::BufferShape, "replay: schedule writes an input data packet"); // codec.hpp:139-143
        else {
            const std::size_t v = std::size_t(store[op.dst_sym]) * w + op.dst_pkt;
            dst = &phys[v];
            wrote[v] = 1;
        }
        if (op.mode == 2) {
            *dst = zero;
            continue;
        }
        const Vec& src = op.src_pkt >= w ? scratch[std::size_t(op.src_sym) * (n - w) + op.src_pkt - w]
                                         : phys[std::size_t(store[op.src_sym]) * w + op.src_pkt];
        if (op.mode == 0) *dst = src;
        else
            for (std::size_t q = 0; q < words; ++q) (*dst)[q] ^= src[q];
    }
    // kernel outputs: storages written through an output slot (first slot names it)
    ScheduleProgram sp;
    sp.k = k;
    sp.outputs = outputs;
    std::vector<std::int32_t> out_of(nstore, -1), src_of(nstore, -1);
    for (std::uint32_t i = 0; i < outputs; ++i) {
        const std::uint32_t st = store[k + i];
        if (out_of[st] >= 0) continue;
        bool any = false;
        for (std::uint32_t b = 0; b < w; ++b) any = any || wrote[std::size_t(st) * w + b];
        if (!any) continue;
        out_of[st] = static_cast<std::int32_t>(sp.dst_slot.size());
        sp.dst_slot.push_back(i);
    }
    // kernel inputs: storages whose initial packets some stored packet reads
    std::vector<std::uint8_t> used(nstore, 0);
    for (std::uint32_t st = 0; st < nstore; ++st)
        for (std::uint32_t b = 0; out_of[st] >= 0 && b < w; ++b)
            if (wrote[std::size_t(st) * w + b])
                for (std::size_t v = 0; v < nv; ++v)
                    if ((phys[std::size_t(st) * w + b][v / 64] >> (v % 64)) & 1u) used[v / w] = 1;
    for (std::uint32_t st = 0; st < nstore; ++st) {
        if (!used[st]) continue;
        std::int32_t slot = 0;
        bool found = false;
        for (std::uint32_t s = 0; s < slots && !found; ++s)
            if (store[s] == st) {
                slot = s < k ? static_cast<std::int32_t>(s) : -1 - static_cast<std::int32_t>(s - k);
                found = true;
            }
        src_of[st] = static_cast<std::int32_t>(sp.src_slot.size());
        sp.src_slot.push_back(slot);
    }
    if (sp.src_slot.empty()) sp.src_slot.push_back(0); // only zero stores: a placeholder input nothing reads
    const std::uint32_t rows = static_cast<std::uint32_t>(sp.dst_slot.size());
    const std::uint32_t cols = static_cast<std::uint32_t>(sp.src_slot.size());
    std::vector<std::uint32_t> bits(std::size_t(rows) * cols * w, 0);
    std::vector<std::uint8_t> written(std::size_t(rows) * w, 0);
    for (std::uint32_t st = 0; st < nstore; ++st) {
        if (out_of[st] < 0) continue;
        const std::uint32_t r = static_cast<std::uint32_t>(out_of[st]);
        for (std::uint32_t b = 0; b < w; ++b) {
            const std::size_t v0 = std::size_t(st) * w + b;
            if (!wrote[v0]) continue;
            written[std::size_t(r) * w + b] = 1;
            for (std::size_t v = 0; v < nv; ++v)
                if ((phys[v0][v / 64] >> (v % 64)) & 1u)
                    bits[(std::size_t(r) * cols + src_of[v / w]) * w + b] |= 1u << (v % w);
        }
    }
    // Matrix recovery: when every written output is complete and every
    // w x w block of the map is multiplication by a field element (true for
    // any schedule compile_schedule or compile_crs_schedule emits, either
    // transform: they all implement the plain GF(2^w) code), the schedule
    // computes M x inputs for that matrix M, and the ring program of M --
    // sparse representatives, the fold, the tuned kernel shape -- is the
    // cheapest exact implementation (flattening a ring schedule would give
    // the bitmatrix's XOR count instead).
    bool field_map = rows > 0 && std::all_of(written.begin(), written.end(), [](std::uint8_t x) { return x != 0; });
    Matrix fm(rows, cols);
    for (std::uint32_t r = 0; field_map && r < rows; ++r)
        for (std::uint32_t q = 0; field_map && q < cols; ++q) {
            const std::uint32_t* blk = &bits[(std::size_t(r) * cols + q) * w];
            std::uint32_t a = 0; // column 0 = the coefficients of a * 1
            for (std::uint32_t b = 0; b < w; ++b) a |= (blk[b] & 1u) << b;
            for (std::uint32_t c = 0; field_map && c < w; ++c) {
                const std::uint32_t prod = gf_mul(a, 1u << c, f);
                for (std::uint32_t b = 0; b < w; ++b)
                    if (((blk[b] >> c) & 1u) != ((prod >> b) & 1u)) field_map = false;
            }
            fm.at(r, q) = static_cast<std::uint16_t>(a);
        }
    if (field_map) {
        CompileOptions o = opt;
        o.bits = nullptr;
        o.written = nullptr;
        o.crs = false;
        o.dense = false;
        sp.prog = compile_program(f, TransformKind::Embedding, fm, o);
    } else if (rows) {
        CompileOptions o = opt;
        o.bits = &bits;
        o.written = &written;
        o.crs = false;
        o.dense = false;
        sp.prog = compile_program(f, TransformKind::Embedding, Matrix(rows, cols), o);
    } else {
        sp.prog.field = f;
        sp.prog.sched = true;
        sp.prog.cols = cols;
    }
    sp.prog.stats.ref_region_ops = ops.size();
    return sp;
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
    fp << kGeneratorVersion << ';' << p.field.w << ',' << p.field.n << ',' << p.field.modulus << ',' << int(p.kind)
       << ',' << p.rows << ',' << p.cols << ',' << p.group << ',' << ks.lanes << ',' << ks.threads << ',' << ks.min_blocks << ','
       << ks.staged << ',' << ks.tile << ',' << ks.stages << ',' << ks.bar_bytes << ',' << p.parts.size() << ','
       << (p.parts.empty() ? 0u : p.parts[0].group) << ',' << ks.copy << ',' << p.cse << ',' << p.crs << ','
       << ks.chunk << ',' << ks.split << ',' << ks.half << ',' << ks.ws << ',' << ks.tmap4 << ',' << ks.spb << ',';
    if (p.sched) {
        for (std::uint32_t b : p.bits) fp << 'b' << b;
        for (std::uint8_t x : p.written) fp << int(x);
    } else if (p.crs)
        for (std::uint16_t x : p.matrix) fp << 'c' << x;
    for (const Program& q : p.parts) fp << q.rows << '/' << q.cse << '/' << q.stats.xors << ',';
    fp << 'h' << p.ir_hash << ',';
    fp << ':';
    for (std::uint32_t r : p.reps) fp << r << ',';
    char name[112];
    if (ks.staged)
        std::snprintf(name, sizeof name, "pyrit_ring_k%u_e%u_w%u_n%u_%s%ux%u_%016llx", p.cols, p.rows, p.field.w,
                      p.field.n, ks.copy == 2 ? "tmt" : !ks.copy ? "tma" : ks.chunk == 16 ? "cpa" : ks.chunk == 8 ? "cpa8_" : "cpa4_",
                      ks.tile, ks.stages,
                      static_cast<unsigned long long>(fnv1a(fp.str())));
    else
        std::snprintf(name, sizeof name, "pyrit_ring_k%u_e%u_w%u_n%u_%s%u%s_%016llx", p.cols, p.rows, p.field.w,
                      p.field.n, ks.half ? "H" : "L", ks.lanes, ks.split > 1 ? ("p" + std::to_string(ks.split)).c_str() : "",
                      static_cast<unsigned long long>(fnv1a(fp.str())));
    return name;
}

KernelShape staged_shape(const Program& p, std::uint32_t smem_limit) {
    KernelShape ks;
    ks.lanes = 1;
    ks.min_blocks = 1;
    if (p.parts.empty()) {
        ks.staged = false;
        return ks;
    }
    const std::uint32_t w = p.field.w, k = p.cols, G = p.parts[0].group;
    const std::uint32_t R = static_cast<std::uint32_t>(p.parts.size());
    // 8 warps per CTA (two per SM sub-partition keeps ptxas's 255-register
    // cap); part r owns 256/R consumer threads, one 4-byte column word each,
    // so a strip tile is 1024/R bytes.  The shared-memory ring holds one
    // fragment group of one tile per slot.
    std::vector<std::uint32_t> choices = {256u, 128u};
    if (p.staged_threads && p.staged_threads != 256) choices.insert(choices.begin(), p.staged_threads);
    for (std::uint32_t threads : choices) {
        if (threads % R) continue;
        const std::uint32_t tile = 4 * (threads / R);
        if (tile < 64) continue;
        const std::uint64_t slot = std::uint64_t(G) * w * tile;
        std::uint32_t slots = 0, bar = 0;
        for (std::uint32_t n = 32; n >= 2; --n) {
            bar = (16 * n + 127) / 128 * 128;
            if (bar + n * slot <= smem_limit) {
                slots = n;
                break;
            }
        }
        if (slots < (threads == choices.back() ? 2u : 3u)) continue; // keep >= 2 tiles in flight
        ks.staged = true;
        ks.tile = tile;
        ks.stages = slots;
        ks.bar_bytes = bar;
        ks.threads = threads;
        ks.smem_bytes = static_cast<std::uint32_t>(bar + slots * slot);
        // producer (profiles/r01_s2/sizes_*copy*, tune_*_v13_tma, trace_ws):
        // TMA tensor boxes when a box (all w strips of a fragment tile) is
        // large (>= 6 KB); heavy codes (>= 8 XORs per input word, the BASELINE
        // codes) issue them from a consumer thread, light codes (GF(2^4))
        // from a dedicated producer warp; small boxes (512 B tiles of the
        // split (60,40) code) stream faster with every thread issuing cp.async
        std::uint64_t xors = 0;
        for (const Program& q : p.parts) xors += q.stats.xors;
        const bool heavy = xors >= 8ull * k * w;
        const bool big_box = std::uint64_t(w) * tile >= 6144;
        std::uint32_t prod = p.staged_producer;
        if (!prod) prod = big_box ? (heavy ? 2u : 3u) : 1u;
        // a TMA producer carries one 128-byte tensor map per input in the
        // kernel parameters (runtime.cpp launch_batch): past ~240 inputs they
        // overflow the 32764-byte parameter space, so copy with cp.async
        const std::uint64_t param_bytes = (8ull * (k + p.rows + 6) + 63) / 64 * 64 + 128ull * k;
        if (prod != 1 && param_bytes > 32764) prod = 1;
        ks.copy = prod == 1 ? 1u : 2u;
        ks.ws = prod == 3 ? 1u : 0u;
        return ks;
    }
    ks.staged = false;
    return ks;
}

namespace {

void emit_xor_list(std::ostringstream& o, const std::vector<std::uint32_t>& src, const std::string& prefix) {
    if (src.empty()) o << "0u";
    for (std::size_t s = 0; s < src.size(); ++s) o << (s ? " ^ " : "") << prefix << src[s];
}

std::string generate_staged(const Program& p, const KernelShape& ks) {
    const std::uint32_t w = p.field.w, k = p.cols, G = p.parts[0].group;
    const std::uint32_t groups = (k + G - 1) / G, TILE = ks.tile, NSLOT = ks.stages, T = ks.threads;
    const std::uint32_t R = static_cast<std::uint32_t>(p.parts.size());
    const std::uint32_t cols_per_part = T / R;
    const std::uint32_t slot_bytes = G * w * TILE;
    std::uint64_t part_xors = 0;
    for (const Program& q : p.parts) part_xors += q.stats.xors;
    std::ostringstream o;
    o << "// generated by pyrit_b200 program compiler (staged, "
      << (ks.copy == 2 ? "TMA tensor boxes" : ks.copy ? "cp.async" : "TMA cp.async.bulk")
      << "): field w=" << w << " n=" << p.field.n << " p=0x" << std::hex << p.field.modulus << std::dec << ", "
      << p.rows << "x" << k << " ring matrix in " << R << " output part(s), " << part_xors
      << " XORs per column word (naive ring program " << p.stats.naive_xors << ", reference schedule "
      << p.stats.ref_region_ops << " region ops); " << T << " threads, tile " << TILE << " B/strip, ring of "
      << NSLOT << " slots x " << G << " fragment(s)\n";
    o << "typedef unsigned int u32; typedef unsigned long long u64; typedef unsigned char u8;\n";
    // nb stripes of the batch: input j of stripe b at in[j] + b * ibp, output i at out[i] + b * obp
    if (ks.copy == 2) // one 3D tensor map per input fragment: (column element, strip, stripe)
        o << "struct alignas(64) TMap { u64 v[16]; };\n";
    o << "struct Args { const u8* in[" << k << "]; u8* out[" << p.rows
      << "]; u64 S; u64 off; u64 len; u64 nb; u64 ibp; u64 obp;"
      << (ks.copy == 2 ? " TMap tm[" + std::to_string(ks.tmap4 ? 1u : k) + "];" : "")
      << " };\n";
    o << R"(static __device__ __forceinline__ u32 smem_u32(const void* p) {
  u32 r; asm("{ .reg .u64 t; cvta.to.shared.u64 t, %1; cvt.u32.u64 %0, t; }" : "=r"(r) : "l"(p)); return r; }
static __device__ __forceinline__ void mbar_init(u32 bar, u32 count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(bar), "r"(count) : "memory"); }
static __device__ __forceinline__ void mbar_expect_tx(u32 bar, u32 bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" :: "r"(bar), "r"(bytes) : "memory"); }
static __device__ __forceinline__ void mbar_arrive(u32 bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" :: "r"(bar) : "memory"); }
static __device__ __forceinline__ void mbar_wait(u32 bar, u32 parity) {
  asm volatile("{\n .reg .pred P1;\n WAIT:\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n @P1 bra DONE;\n bra WAIT;\n DONE:\n}"
               :: "r"(bar), "r"(parity) : "memory"); }
static __device__ __forceinline__ void bulk_g2s(u32 dst, const void* src, u32 bytes, u32 bar, u64 pol) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
               :: "r"(dst), "l"(src), "r"(bytes), "r"(bar), "l"(pol) : "memory"); }
static __device__ __forceinline__ void tma4d(u32 dst, const void* map, u32 x, u32 y, u32 z, u32 q, u32 bar) {
  asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
               :: "r"(dst), "l"(map), "r"(x), "r"(y), "r"(z), "r"(q), "r"(bar) : "memory"); }
static __device__ __forceinline__ void tma3d(u32 dst, const void* map, u32 x, u32 y, u32 z, u32 bar) {
  asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
               :: "r"(dst), "l"(map), "r"(x), "r"(y), "r"(z), "r"(bar) : "memory"); }
static __device__ __forceinline__ void cpa16(u32 dst, const void* src, u32 n) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" :: "r"(dst), "l"(src), "r"(n) : "memory"); }
static __device__ __forceinline__ void cpa8(u32 dst, const void* src, u32 n) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" :: "r"(dst), "l"(src), "r"(n) : "memory"); }
static __device__ __forceinline__ void cpa4(u32 dst, const void* src, u32 n) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" :: "r"(dst), "l"(src), "r"(n) : "memory"); }
static __device__ __forceinline__ void cpa_arrive(u32 bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" :: "r"(bar) : "memory"); }
static __device__ __forceinline__ void st_cs(u8* p, u32 v) {
  asm volatile("st.global.cs.b32 [%0], %1;" :: "l"(p), "r"(v) : "memory"); }
)";
    const std::string name = kernel_name(p, ks);
    o << "#define TILE " << TILE << "u\n#define NSLOT " << NSLOT << "u\n#define SLOT_BYTES " << slot_bytes
      << "u\n#define NG " << groups << "u\n#define BAR_BYTES " << ks.bar_bytes << "u\n";
    o << "#define FULL(s) (sbase + 8u * (s))\n#define EMPTY(s) (sbase + 8u * (NSLOT + (s)))\n";
    const bool ws = ks.copy == 2 && ks.ws; // a dedicated producer warp after the T consumer threads
    o << "extern \"C\" __global__ void __launch_bounds__(" << T + (ws ? 32u : 0u) << ", 1) " << name
      << "(const __grid_constant__ Args a)\n{\n";
    o << "  extern __shared__ __align__(1024) u8 sm[];\n";
    o << "  const u32 sbase = smem_u32(sm);\n";
    o << "  const u32 tpb = (u32)((a.len + TILE - 1) / TILE);\n"; // tiles per stripe
    o << "  const u32 ntiles = tpb * (u32)a.nb;\n";
    o << "  auto my_units_tiles = [&]() -> u32 { return blockIdx.x < ntiles ? (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0u; };\n";
    o << "  if (threadIdx.x == 0) {\n";
    o << "    for (u32 s = 0; s < NSLOT; ++s) { mbar_init(FULL(s), " << (ks.copy == 1 ? T : 1u) << "u); mbar_init(EMPTY(s), "
      << T << "u); }\n";
    o << "    asm volatile(\"fence.mbarrier_init.release.cluster;\" ::: \"memory\");\n  }\n";
    o << "  __syncthreads();\n";
    // programmatic dependent launch: everything above overlaps the previous
    // grid's tail; global memory is touched only after it has completed
    o << "  asm volatile(\"griddepcontrol.wait;\" ::: \"memory\");\n";
    o << "  const u32 lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;\n";
    // produce(u2): fill the slot of pipeline unit u2 = (tile it2, fragment group g2)
    o << "  u64 pol = 0;\n";
    if (!ks.copy) o << "  if (warp == 0) asm volatile(\"createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\" : \"=l\"(pol));\n";
    if (ks.copy == 2) {
        // TMA tensor copies: one elected thread posts the unit's byte count and
        // issues one 3D box (all w strips x TILE bytes of a fragment) per
        // fragment of the group; no other thread takes part in the copy
        const std::uint32_t elem = TILE > 1024 ? 8u : 4u;
        o << "  auto produce = [&](u32 u2) {\n";
        o << "    const u32 it2 = u2 / NG, g2 = u2 - it2 * NG;\n";
        o << "    const u32 t2 = blockIdx.x + it2 * gridDim.x;\n";
        o << "    if (t2 >= ntiles) return;\n";
        o << "    const u32 sl = u2 % NSLOT, ph = (u2 / NSLOT) & 1u;\n";
        o << "    mbar_wait(EMPTY(sl), ph ^ 1u);\n";
        o << "    const u32 b2 = t2 / tpb, tt2 = t2 - b2 * tpb;\n";
        o << "    const u32 x = (u32)((a.off + (u64)tt2 * TILE) / " << elem << "u);\n";
        o << "    const u32 dst = sbase + BAR_BYTES + sl * SLOT_BYTES;\n";
        o << "    const u32 j0 = g2 * " << G << "u;\n";
        o << "    const u32 nfr = g2 + 1u == NG ? " << k << "u - j0 : " << G << "u;\n";
        if (ks.tmap4) {
            // equally spaced inputs: one 4D box (tile x w strips x G fragments)
            // per unit; fragments past k are out of bounds and zero-filled, so
            // the transaction is always the full box
            o << "    (void)nfr;\n";
            o << "    mbar_expect_tx(FULL(sl), " << G * w * TILE << "u);\n";
            o << "    tma4d(dst, &a.tm[0], x, 0u, j0, b2, FULL(sl));\n";
        } else {
            // boxes of ks.spb strips (a divisor of w): several requests per fragment
            const std::uint32_t spb = ks.spb && w % ks.spb == 0 ? ks.spb : w;
            o << "    mbar_expect_tx(FULL(sl), nfr * " << w * TILE << "u);\n";
            o << "#pragma unroll 1\n";
            o << "    for (u32 f = 0; f < nfr; ++f)\n";
            o << "#pragma unroll\n";
            o << "      for (u32 s0 = 0; s0 < " << w << "u; s0 += " << spb << "u)\n";
            o << "        tma3d(dst + f * " << w * TILE << "u + s0 * TILE, &a.tm[j0 + f], x, s0, b2, FULL(sl));\n";
        }
    } else if (ks.copy) {
        // every thread copies CH-byte chunks (16, or 8/4 when the strips are
        // only that aligned; a strip tile is TILE/CH consecutive chunks:
        // coalesced) and arrives on the slot's FULL barrier once its copies
        // have landed.  Lanes are laid out strip-major: LPS lanes cover one
        // strip tile (CPL chunks each), a warp covers SPW strips per step,
        // warps stride strips by NWS = NW*SPW.  The strips a thread copies are
        // fixed per fragment group, so their base pointers are computed once
        // (registers) and a unit only adds its tile offset; chunks past the
        // window are skipped (their columns are never stored)
        const std::uint32_t CH = ks.chunk;
        const std::uint32_t cps = TILE / CH;
        const std::uint32_t lps = std::min<std::uint32_t>(32, cps), spw = 32 / lps, cpl = cps / lps, nw = T / 32;
        const std::uint32_t nws = nw * spw;
        o << "  const u32 lq = lane % " << lps << "u, lsub = lane / " << lps << "u;\n";
        o << "  const u32 lbase = warp * " << spw << "u + lsub;\n";
        std::vector<std::uint32_t> per_group(groups);
        for (std::uint32_t g = 0; g < groups; ++g) {
            const std::uint32_t nstr = (std::min(k, (g + 1) * G) - g * G) * w;
            per_group[g] = (nstr + nws - 1) / nws;
            for (std::uint32_t m = 0; m < per_group[g]; ++m) {
                o << "  const u8* sp" << g << "_" << m << ";\n  { const u32 l = lbase + " << m * nws << "u;";
                o << " const u32 idx = " << g * G * w << "u + (l < " << nstr << "u ? l : 0u), j = idx / " << w
                  << "u, s = idx - j * " << w << "u;";
                o << " sp" << g << "_" << m << " = a.in[j] + s * a.S + a.off + " << CH << "u * lq; }\n";
            }
        }
        o << "  auto produce = [&](u32 u2) {\n";
        o << "    const u32 it2 = u2 / NG, g2 = u2 - it2 * NG;\n";
        o << "    const u32 t2 = blockIdx.x + it2 * gridDim.x;\n";
        o << "    if (t2 >= ntiles) return;\n";
        o << "    const u32 sl = u2 % NSLOT, ph = (u2 / NSLOT) & 1u;\n";
        o << "    mbar_wait(EMPTY(sl), ph ^ 1u);\n";
        o << "    const u32 b2 = t2 / tpb, tt2 = t2 - b2 * tpb;\n";
        o << "    const u64 uoff = b2 * a.ibp + (u64)tt2 * TILE;\n";
        o << "    const u64 rem = a.len - (u64)tt2 * TILE;\n";
        o << "    const u32 vb = (u32)(rem < TILE ? rem : TILE);\n";
        o << "    const u32 d0 = sbase + BAR_BYTES + sl * SLOT_BYTES + lbase * TILE + " << CH << "u * lq;\n";
        for (std::uint32_t c = 0; c < cpl; ++c)
            o << "    const bool n" << c << " = " << CH << "u * (lq + " << c * lps << "u) < vb;\n";
        o << "    switch (g2) {\n";
        for (std::uint32_t g = 0; g < groups; ++g) {
            const std::uint32_t nstr = (std::min(k, (g + 1) * G) - g * G) * w;
            o << "    case " << g << "u:\n";
            for (std::uint32_t m = 0; m < per_group[g]; ++m) {
                const bool tail = (m + 1) * nws > nstr; // some threads have no strip m
                o << "      " << (tail ? "if (lbase + " + std::to_string(m * nws) + "u < " + std::to_string(nstr) + "u) " : "")
                  << "{ const u8* src = sp" << g << "_" << m << " + uoff;";
                for (std::uint32_t c = 0; c < cpl; ++c)
                    o << " if (n" << c << ") cpa" << CH << "(d0 + " << (m * nws * TILE + CH * c * lps) << "u, src + "
                      << CH * c * lps << "u, " << CH << "u);";
                o << " }\n";
            }
            o << "      break;\n";
        }
        o << "    }\n";
        o << "    cpa_arrive(FULL(sl));\n";
    } else {
        o << "  auto produce = [&](u32 u2) {\n";
        o << "    const u32 it2 = u2 / NG, g2 = u2 - it2 * NG;\n";
        o << "    const u32 t2 = blockIdx.x + it2 * gridDim.x;\n";
        o << "    if (t2 >= ntiles) return;\n";
        o << "    const u32 sl = u2 % NSLOT, ph = (u2 / NSLOT) & 1u;\n";
        o << "    mbar_wait(EMPTY(sl), ph ^ 1u);\n";
        o << "    const u32 b2 = t2 / tpb, tt2 = t2 - b2 * tpb;\n";
        o << "    const u64 o = a.off + (u64)tt2 * TILE;\n";
        o << "    const u32 dst = sbase + BAR_BYTES + sl * SLOT_BYTES;\n";
        o << "    const u32 j0 = g2 * " << G << "u;\n";
        o << "    const u32 nstr = (g2 + 1u == NG ? " << k << "u - j0 : " << G << "u) * " << w << "u;\n";
        // warp 0: lane 0 posts the byte count, the lanes issue one
        // cp.async.bulk per strip tile
        o << "    const u64 rem = a.len - (u64)tt2 * TILE;\n";
        o << "    const u32 bytes = (u32)(rem < TILE ? rem : TILE);\n";
        o << "    if (lane == 0) mbar_expect_tx(FULL(sl), bytes * nstr);\n";
        o << "    __syncwarp();\n";
        o << "#pragma unroll 1\n";
        o << "    for (u32 l = lane; l < nstr; l += 32u) {\n";
        o << "      const u32 idx = j0 * " << w << "u + l, j = idx / " << w << "u, s = idx - j * " << w << "u;\n";
        o << "      bulk_g2s(dst + l * TILE, a.in[j] + b2 * a.ibp + s * a.S + o, bytes, FULL(sl), pol);\n";
        o << "    }\n";
    }
    o << "  };\n";
    if (ws) {
        // warp specialisation: the extra warp only feeds the ring (its lane 0
        // runs ahead until every slot is in flight); consumers never copy
        o << "  if (threadIdx.x >= " << T << "u) {\n";
        o << "    if (lane == 0) for (u32 u = 0; u / NG < my_units_tiles(); ++u) produce(u);\n";
        o << "    return;\n  }\n";
    } else {
        const std::string who = ks.copy == 1 ? "" : ks.copy == 2 ? "if (threadIdx.x == 0) " : "if (warp == 0) ";
        o << "  " << who << "for (u32 u = 0; u + 1 < NSLOT; ++u) produce(u);\n";
    }
    o << "  const u32 part = threadIdx.x / " << cols_per_part << "u, col = threadIdx.x % " << cols_per_part << "u;\n";
    o << "  const u64 S = a.S;\n";
    // one tile loop per output part: each is its own register-allocation region
    for (std::uint32_t r = 0; r < R; ++r) {
        const Program& q = p.parts[r];
        const std::uint32_t row0 = p.part_row0[r];
        o << "  " << (r ? "else if" : "if") << " (part == " << r << "u) {\n";
        o << "   u32 it = 0;\n";
        o << "   for (u32 t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {\n";
        o << "    const u32 bb = t / tpb, tt = t - bb * tpb;\n";
        o << "    const u64 rel = (u64)tt * TILE + 4u * col;\n";
        o << "    const u64 o = a.off + rel + bb * a.obp;\n";
        o << "    const bool live = rel < a.len;\n";
        std::vector<bool> out_ptr(q.rows, false);
        std::string cur_sp;
        auto emit = [&](const Instr& ins) {
            if (ins.op == Instr::Load) {
                const std::uint32_t local = (ins.sym - (ins.sym / G) * G) * w + ins.strip;
                o << "    const u32 v" << ins.dst << " = " << cur_sp << "[" << local * (TILE / 4) << "];\n";
            } else if (ins.op == Instr::Xor) {
                o << "    const u32 v" << ins.dst << " = ";
                emit_xor_list(o, ins.src, "v");
                o << ";\n";
            } else {
                const std::uint32_t row = row0 + ins.sym;
                if (!out_ptr[ins.sym]) {
                    o << "    u8* q" << row << " = a.out[" << row << "] + o;\n";
                    out_ptr[ins.sym] = true;
                }
                o << "    if (live) st_cs(q" << row;
                if (ins.strip) o << " + " << ins.strip << "u * S";
                o << ", ";
                emit_xor_list(o, ins.src, "v");
                o << ");\n";
            }
        };
        for (std::uint32_t g = 0; g < groups; ++g) {
            // unit (it, g): keep NSLOT-1 units in flight, wait for this one,
            // read its strips from shared memory, release the slot, XOR
            const std::string gs = std::to_string(g);
            o << "    const u32 un" << gs << " = it * NG + " << g << "u;\n";
            if (ks.copy == 1) o << "    produce(un" << gs << " + NSLOT - 1u);\n";
            else if (ks.copy == 2 && !ws && r == 0) o << "    if (threadIdx.x == 0) produce(un" << gs << " + NSLOT - 1u);\n";
            else if (ks.copy == 2) {}
            else if (r == 0) o << "    if (warp == 0) produce(un" << gs << " + NSLOT - 1u);\n";
            o << "    const u32 sl" << gs << " = un" << gs << " % NSLOT;\n";
            o << "    mbar_wait(FULL(sl" << gs << "), (un" << gs << " / NSLOT) & 1u);\n";
            o << "    const u32* sp" << gs << " = reinterpret_cast<const u32*>(sm + BAR_BYTES + sl" << gs
              << " * SLOT_BYTES) + col;\n";
            cur_sp = "sp" + gs;
            for (const Instr& x : q.group_loads[g]) emit(x);
            o << "    mbar_arrive(EMPTY(sl" << gs << "));\n";
            for (const Instr& x : q.group_compute[g]) emit(x);
        }
        for (const Instr& x : q.tail) emit(x);
        o << "   }\n  }\n";
    }
    // dependents may launch once this CTA has issued all its work: they take
    // over the SMs freed by the tail without pre-launching during the body
    o << "  asm volatile(\"griddepcontrol.launch_dependents;\" ::: \"memory\");\n";
    o << "}\n";
    return o.str();
}

} // namespace

std::string generate_cuda(const Program& p, const KernelShape& ks) {
    if (ks.staged) return generate_staged(p, ks);
    const std::uint32_t L = ks.lanes == 0 ? 1 : ks.lanes;
    const bool bytes = ks.lanes == 0; // sub-word mode: one u8 (or u16 when ks.half) per thread per strip
    const std::uint32_t V = bytes ? (ks.half ? 2 : 1) : 4 * L; // bytes per thread per strip
    // split: the output rows are divided over R thread groups (p.parts) that
    // walk the same column words; every group loads all input strips, the
    // first touch of a line fills L1 and the other groups hit it, so HBM
    // still sees each input byte once while no thread holds more than one
    // part's accumulators (large codes otherwise spill)
    const std::uint32_t R = ks.split > 1 ? static_cast<std::uint32_t>(p.parts.size()) : 1;
    const std::uint32_t CPB = ks.threads / R; // column threads per block
    std::ostringstream o;
    o << "// generated by pyrit_b200 program compiler: field w=" << p.field.w << " n=" << p.field.n << " p=0x"
      << std::hex << p.field.modulus << std::dec << ", " << p.rows << "x" << p.cols << " ring matrix, "
      << p.stats.xors << " XORs (naive ring program " << p.stats.naive_xors << ", reference schedule "
      << p.stats.ref_region_ops << " region ops)" << (R > 1 ? ", rows split over " + std::to_string(R) + " thread groups" : "")
      << "\n";
    o << "typedef unsigned int u32; typedef unsigned long long u64; typedef unsigned char u8;\n";
    // nb stripes of nwords column words each; the grid stride advances
    // (stripe, word) by (sq, sr) = divmod(stride, nwords), precomputed on the host
    o << "struct Args { const u8* in[" << p.cols << "]; u8* out[" << p.rows
      << "]; u64 S; u64 off; u64 nwords; u64 nb; u64 ibp; u64 obp; u64 sq; u64 sr; };\n";
    // loads: read-only, no L1 allocation (streamed once) -- L1-cached when
    // split, the other row groups re-read the line; stores: evict-first
    const std::string l1 = R > 1 ? "" : ".L1::no_allocate";
    if (bytes) {
        const char* ty = ks.half ? "u16" : "u8";
        o << "#define LD(v, p) asm(\"ld.global.nc" << l1 << "." << ty << " %0, [%1];\" : \"=r\"(v) : \"l\"(p))\n";
        o << "#define ST(p, v) asm volatile(\"st.global.cs." << ty << " [%0], %1;\" :: \"l\"(p), \"r\"(v) : \"memory\")\n";
    } else if (L == 1) {
        o << "#define LD(v, p) asm(\"ld.global.nc" << l1 << ".b32 %0, [%1];\" : \"=r\"(v##_0) : \"l\"(p))\n";
        o << "#define ST(p, v) asm volatile(\"st.global.cs.b32 [%0], %1;\" :: \"l\"(p), \"r\"(v##_0) : \"memory\")\n";
    } else if (L == 2) {
        o << "#define LD(v, p) asm(\"ld.global.nc" << l1 << ".v2.b32 {%0, %1}, [%2];\" : \"=r\"(v##_0), "
             "\"=r\"(v##_1) : \"l\"(p))\n";
        o << "#define ST(p, v) asm volatile(\"st.global.cs.v2.b32 [%0], {%1, %2};\" :: \"l\"(p), \"r\"(v##_0), "
             "\"r\"(v##_1) : \"memory\")\n";
    } else {
        o << "#define LD(v, p) asm(\"ld.global.nc" << l1 << ".v4.b32 {%0, %1, %2, %3}, [%4];\" : "
             "\"=r\"(v##_0), \"=r\"(v##_1), \"=r\"(v##_2), \"=r\"(v##_3) : \"l\"(p))\n";
        o << "#define ST(p, v) asm volatile(\"st.global.cs.v4.b32 [%0], {%1, %2, %3, %4};\" :: \"l\"(p), "
             "\"r\"(v##_0), \"r\"(v##_1), \"r\"(v##_2), \"r\"(v##_3) : \"memory\")\n";
    }
    const std::string name = kernel_name(p, ks);
    o << "extern \"C\" __global__ void __launch_bounds__(" << ks.threads << ", " << ks.min_blocks << ") " << name
      << "(const Args a)\n{\n";
    o << "  const u64 S = a.S;\n";
    o << "  asm volatile(\"griddepcontrol.wait;\" ::: \"memory\");\n";
    o << "  const u32 part = threadIdx.x / " << CPB << "u;\n";
    o << "  const u64 c0 = (u64)blockIdx.x * " << CPB << "u + threadIdx.x % " << CPB << "u;\n";
    auto var = [&](std::uint32_t v, std::uint32_t l) {
        std::string s = "v" + std::to_string(v);
        if (!bytes) s += "_" + std::to_string(l);
        return s;
    };
    for (std::uint32_t r = 0; r < R; ++r) {
        const Program& q = R > 1 ? p.parts[r] : p;
        const std::uint32_t row0 = R > 1 ? p.part_row0[r] : 0;
        o << "  " << (r ? "else if" : "if") << " (part == " << r << "u) {\n";
        o << "  u64 b = c0 / a.nwords, cw = c0 - b * a.nwords;\n";
        o << "  while (b < a.nb) {\n";
        o << "    const u64 o = a.off + cw * " << V << "u;\n";
        o << "    const u64 oi = o + b * a.ibp, oo = o + b * a.obp;\n";
        std::vector<bool> frag_ptr(q.cols, false), out_ptr(q.rows, false);
        // split kernels: one fragment group's loads at a time (no prefetch of
        // the next group) so a part stays within the 128 registers of 2 CTAs/SM
        std::vector<Instr> seq;
        if (R > 1) {
            for (std::size_t g = 0; g < q.group_loads.size(); ++g) {
                seq.insert(seq.end(), q.group_loads[g].begin(), q.group_loads[g].end());
                seq.insert(seq.end(), q.group_compute[g].begin(), q.group_compute[g].end());
            }
            seq.insert(seq.end(), q.tail.begin(), q.tail.end());
        }
        for (const Instr& ins : R > 1 ? seq : q.code) {
            if (ins.op == Instr::Load) {
                if (!frag_ptr[ins.sym]) {
                    o << "    const u8* i" << ins.sym << " = a.in[" << ins.sym << "] + oi;\n";
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
                const std::uint32_t row = row0 + ins.sym;
                if (!out_ptr[ins.sym]) {
                    o << "    u8* q" << row << " = a.out[" << row << "] + oo;\n";
                    out_ptr[ins.sym] = true;
                }
                o << "    { u32 ";
                for (std::uint32_t l = 0; l < L; ++l) {
                    o << (l ? ", " : "") << "x" << (bytes ? "" : "_" + std::to_string(l)) << " = ";
                    if (ins.src.empty()) o << "0u";
                    for (std::size_t s = 0; s < ins.src.size(); ++s) o << (s ? " ^ " : "") << var(ins.src[s], l);
                }
                o << "; ST(q" << row;
                if (ins.strip) o << " + " << ins.strip << "u * S";
                o << ", x); }\n";
            }
        }
        o << "    b += a.sq; cw += a.sr;\n";
        o << "    if (cw >= a.nwords) { cw -= a.nwords; ++b; }\n";
        o << "  }\n  }\n";
    }
    o << "  asm volatile(\"griddepcontrol.launch_dependents;\" ::: \"memory\");\n";
    o << "}\n";
    return o.str();
}

} // namespace pyrit_b200
