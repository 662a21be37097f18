#include "algebra.hpp"

#include <algorithm>
#include <bit>
#include <map>
#include <memory>
#include <mutex>

namespace pyrit_b200 {

namespace {
int degree(std::uint64_t a) { return a == 0 ? -1 : 63 - std::countl_zero(a); }

std::uint32_t rotl_n(std::uint32_t a, unsigned s, unsigned n) { // bits.hpp:35-39
    const std::uint32_t mask = n >= 32 ? 0xFFFFFFFFu : ((1u << n) - 1);
    a &= mask;
    return s == 0 ? a : (((a << s) | (a >> (n - s))) & mask);
}
} // namespace

std::uint64_t clmul(std::uint64_t a, std::uint64_t b) {
    std::uint64_t acc = 0;
    while (b) {
        acc ^= a * (b & (0 - b));
        b &= b - 1;
    }
    return acc;
}

std::uint64_t poly_mod(std::uint64_t a, std::uint64_t m) {
    const int dm = degree(m);
    for (int da = degree(a); da >= dm; da = degree(a)) a ^= m << (da - dm);
    return a;
}

void validate_field(const Field& f) {
    if (f.w == 0 || f.w > 16) raise(Errc::InvalidArgument, "field degree w must be in [1, 16]");
    if (f.n <= f.w || f.n > 32) raise(Errc::InvalidArgument, "ring length n must be in (w, 32]");
    if (degree(f.modulus) != static_cast<int>(f.w))
        raise(Errc::InvalidArgument, "modulus degree must equal w");
    if (f.s == 0) raise(Errc::InvalidArgument, "spacing s must be positive");
    // the ring R = F2[x]/(x^n+1) must contain the field: p | x^n + 1
    if (poly_mod((1ull << f.n) | 1ull, f.modulus) != 0)
        raise(Errc::InvalidArgument, "modulus does not divide x^n + 1");
}

namespace {

// Log/antilog tables of GF(2^w) over a generator g of the multiplicative
// group (x itself is not one for the all-one moduli: x^(w+1) = 1), so that a
// product or inverse is two table reads instead of a carry-less multiply and
// reduction (gf_mul) or a search over the field (gf_inv, field.hpp:82-89:
// 2^w multiplies).  Same results: the tables are built with those functions.
struct GfTables {
    std::uint32_t q1 = 0;              // 2^w - 1
    std::vector<std::uint16_t> log, exp; // exp has 2*q1 entries (no modulo on add)
};

std::uint32_t slow_mul(std::uint32_t a, std::uint32_t b, std::uint32_t modulus) {
    return static_cast<std::uint32_t>(poly_mod(clmul(a, b), modulus));
}

std::shared_ptr<const GfTables> build_tables(std::uint32_t w, std::uint32_t modulus) {
    auto t = std::make_shared<GfTables>();
    const std::uint32_t q = 1u << w;
    t->q1 = q - 1;
    for (std::uint32_t g = q == 2 ? 1u : 2u; g < q; ++g) {
        // order of g: the first power that returns to 1
        std::uint32_t v = 1, ord = 0;
        do {
            v = slow_mul(v, g, modulus);
            ++ord;
        } while (v != 1 && ord <= t->q1);
        if (ord == t->q1) {
            t->log.assign(q, 0);
            t->exp.assign(2 * std::size_t(t->q1), 0);
            v = 1;
            for (std::uint32_t i = 0; i < t->q1; ++i) {
                t->exp[i] = t->exp[i + t->q1] = static_cast<std::uint16_t>(v);
                t->log[v] = static_cast<std::uint16_t>(i);
                v = slow_mul(v, g, modulus);
            }
            return t;
        }
    }
    return nullptr; // p is not irreducible: no multiplicative group to tabulate
}

// tables of f, built once per (w, modulus) and kept (a thread's last field is
// cached so a matrix loop pays one comparison per product)
const GfTables* tables(const Field& f) {
    const std::uint64_t key = (std::uint64_t(f.w) << 32) | f.modulus;
    thread_local std::uint64_t last_key = ~0ull;
    thread_local const GfTables* last = nullptr;
    if (key == last_key) return last;
    static std::mutex mu;
    static std::map<std::uint64_t, std::shared_ptr<const GfTables>> all;
    std::lock_guard<std::mutex> lk(mu);
    auto it = all.find(key);
    if (it == all.end()) it = all.emplace(key, build_tables(f.w, f.modulus)).first;
    last_key = key;
    last = it->second.get();
    return last;
}

} // namespace

std::uint32_t gf_mul(std::uint32_t a, std::uint32_t b, const Field& f) {
    if (a < f.field_size() && b < f.field_size() && f.w <= 16) {
        if (a == 0 || b == 0) return 0;
        if (const GfTables* t = tables(f)) return t->exp[std::size_t(t->log[a]) + t->log[b]];
    }
    return slow_mul(a, b, f.modulus);
}

std::uint32_t gf_inv(std::uint32_t a, const Field& f) {
    if (a == 0) raise(Errc::ZeroInverse, "inverse of zero");
    if (a < f.field_size() && f.w <= 16)
        if (const GfTables* t = tables(f)) return t->exp[(t->q1 - t->log[a]) % t->q1];
    for (std::uint32_t b = 1; b < f.field_size(); ++b)
        if (gf_mul(a, b, f) == 1) return b;
    raise(Errc::ZeroInverse, "no inverse found");
}

std::uint32_t ring_mul(std::uint32_t a, std::uint32_t b, const Field& f) {
    std::uint32_t acc = 0, rest = a & f.ring_mask();
    while (rest) {
        acc ^= rotl_n(b, static_cast<unsigned>(std::countr_zero(rest)), f.n);
        rest &= rest - 1;
    }
    return acc;
}

std::uint32_t dense_transform(std::uint32_t u, const Field& f) {
    // phi1(u) = u * theta1 with theta1 = p + 1 (ring.hpp:36-44)
    return ring_mul(u & f.field_mask(), (f.modulus ^ 1u) & f.ring_mask(), f);
}

namespace {
std::uint32_t sparse_transform_uncached(std::uint32_t u, const Field& f);
} // namespace

// memoised per field (a code's matrices repeat entries, and every decode
// pattern of a code draws from the same 2^w values)
std::uint32_t sparse_transform(std::uint32_t u, const Field& f) {
    if (f.w > 16 || u >= f.field_size()) return sparse_transform_uncached(u, f);
    const std::uint64_t key = (std::uint64_t(f.w) << 48) ^ (std::uint64_t(f.n) << 40) ^ f.modulus;
    static std::mutex mu;
    static std::map<std::uint64_t, std::vector<std::uint64_t>> memo; // value + 1, 0 = not yet known
    {
        std::lock_guard<std::mutex> lk(mu);
        auto& v = memo[key];
        if (v.empty()) v.assign(f.field_size(), 0);
        if (v[u]) return static_cast<std::uint32_t>(v[u] - 1);
    }
    const std::uint32_t r = sparse_transform_uncached(u, f);
    std::lock_guard<std::mutex> lk(mu);
    memo[key][u] = std::uint64_t(r) + 1;
    return r;
}

namespace {
std::uint32_t sparse_transform_uncached(std::uint32_t u, const Field& f) {
    // Lightest element of the coset anchor + (p) of degree < n, ties toward
    // the smallest value (ring.hpp:77-90); candidates are anchor ^ m*p for
    // every m of degree < n - w (ring.hpp:65-72).
    const std::uint32_t anchor = dense_transform(u, f);
    std::uint32_t best = anchor;
    unsigned bw = std::popcount(anchor);
    const std::uint32_t count = 1u << (f.n - f.w);
    for (std::uint32_t m = 0; m < count; ++m) {
        const std::uint32_t cand = anchor ^ static_cast<std::uint32_t>(clmul(m, f.modulus));
        const unsigned cw = std::popcount(cand);
        if (cw < bw || (cw == bw && cand < best)) {
            best = cand;
            bw = cw;
        }
    }
    return best;
}
} // namespace

std::vector<std::uint32_t> fold_table(const Field& f) {
    std::vector<std::uint32_t> t;
    for (std::uint32_t j = f.w; j < f.n; ++j)
        t.push_back(static_cast<std::uint32_t>(poly_mod(1ull << j, f.modulus)));
    return t;
}

Matrix cauchy_parity_matrix(std::uint32_t k, std::uint32_t r, const Field& f) {
    if (k == 0) raise(Errc::InvalidArgument, "k must be at least 1");
    if (k + r > f.field_size())
        raise(Errc::TooManySymbols, "k + r = " + std::to_string(k + r) + " exceeds field size " +
                                        std::to_string(f.field_size()));
    Matrix c(r, k);
    for (std::uint32_t i = 0; i < r; ++i)
        for (std::uint32_t j = 0; j < k; ++j)
            c.at(i, j) = static_cast<std::uint16_t>(gf_inv((k + i) ^ j, f));
    for (std::uint32_t i = 0; i < r; ++i) {
        const std::uint32_t sc = gf_inv(c.at(i, 0), f);
        for (std::uint32_t j = 0; j < k; ++j) c.at(i, j) = static_cast<std::uint16_t>(gf_mul(c.at(i, j), sc, f));
    }
    for (std::uint32_t j = 0; j < k && r > 0; ++j) {
        const std::uint32_t sc = gf_inv(c.at(0, j), f);
        for (std::uint32_t i = 0; i < r; ++i) c.at(i, j) = static_cast<std::uint16_t>(gf_mul(c.at(i, j), sc, f));
    }
    return c;
}

Matrix matrix_product(const Matrix& a, const Matrix& b, const Field& f) {
    if (a.cols != b.rows) raise(Errc::InvalidArgument, "matrix shape mismatch");
    Matrix out(a.rows, b.cols);
    for (std::uint32_t i = 0; i < a.rows; ++i)
        for (std::uint32_t t = 0; t < a.cols; ++t) {
            const std::uint32_t v = a.at(i, t);
            if (!v) continue;
            for (std::uint32_t j = 0; j < b.cols; ++j)
                out.at(i, j) ^= static_cast<std::uint16_t>(gf_mul(v, b.at(t, j), f));
        }
    return out;
}

Matrix invert(const Matrix& m, const Field& f) {
    if (m.rows != m.cols) raise(Errc::InvalidArgument, "inverse of non-square matrix");
    const std::uint32_t n = m.rows;
    Matrix a = m, inv(n, n);
    for (std::uint32_t i = 0; i < n; ++i) inv.at(i, i) = 1;
    for (std::uint32_t col = 0; col < n; ++col) {
        std::uint32_t piv = col;
        while (piv < n && a.at(piv, col) == 0) ++piv;
        if (piv == n) raise(Errc::Singular, "singular matrix");
        if (piv != col)
            for (std::uint32_t j = 0; j < n; ++j) {
                std::swap(a.at(piv, j), a.at(col, j));
                std::swap(inv.at(piv, j), inv.at(col, j));
            }
        const std::uint32_t sc = gf_inv(a.at(col, col), f);
        for (std::uint32_t j = 0; j < n; ++j) {
            a.at(col, j) = static_cast<std::uint16_t>(gf_mul(a.at(col, j), sc, f));
            inv.at(col, j) = static_cast<std::uint16_t>(gf_mul(inv.at(col, j), sc, f));
        }
        for (std::uint32_t row = 0; row < n; ++row) {
            if (row == col) continue;
            const std::uint32_t fac = a.at(row, col);
            if (!fac) continue;
            for (std::uint32_t j = 0; j < n; ++j) {
                a.at(row, j) ^= static_cast<std::uint16_t>(gf_mul(fac, a.at(col, j), f));
                inv.at(row, j) ^= static_cast<std::uint16_t>(gf_mul(fac, inv.at(col, j), f));
            }
        }
    }
    return inv;
}

namespace {
Matrix survivor_inverse(std::uint32_t k, std::uint32_t r, const Field& f, const Matrix& parity,
                        const std::vector<std::uint32_t>& survivors, std::vector<bool>& seen) {
    if (survivors.size() != k) raise(Errc::InvalidArgument, "need exactly k survivors");
    seen.assign(k + r, false);
    for (std::uint32_t s : survivors) {
        if (s >= k + r) raise(Errc::InvalidArgument, "survivor index out of range");
        if (seen[s]) raise(Errc::InvalidArgument, "duplicate survivor index");
        seen[s] = true;
    }
    Matrix a(k, k);
    for (std::uint32_t row = 0; row < k; ++row) {
        const std::uint32_t s = survivors[row];
        if (s < k) a.at(row, s) = 1;
        else
            for (std::uint32_t j = 0; j < k; ++j) a.at(row, j) = parity.at(s - k, j);
    }
    return invert(a, f);
}
} // namespace

Matrix decode_matrix(std::uint32_t k, std::uint32_t r, const Field& f, const Matrix& parity,
                     const std::vector<std::uint32_t>& survivors) {
    std::vector<bool> seen;
    const Matrix ainv = survivor_inverse(k, r, f, parity, survivors, seen);
    std::vector<std::uint32_t> erased;
    for (std::uint32_t d = 0; d < k; ++d)
        if (!seen[d]) erased.push_back(d);
    Matrix out(static_cast<std::uint32_t>(erased.size()), k);
    for (std::size_t i = 0; i < erased.size(); ++i)
        for (std::uint32_t j = 0; j < k; ++j) out.at(static_cast<std::uint32_t>(i), j) = ainv.at(erased[i], j);
    return out;
}

RepairPlan repair_matrix(std::uint32_t k, std::uint32_t r, const Field& f,
                         const std::vector<std::uint32_t>& erased) {
    // validation mirrors decode (codec.hpp:243-255)
    if (k == 0) raise(Errc::InvalidArgument, "k must be at least 1");
    if (k + r > f.field_size()) raise(Errc::TooManySymbols, "k + r exceeds field size");
    std::vector<bool> gone(k + r, false);
    for (std::uint32_t e : erased) {
        if (e >= k + r) raise(Errc::InvalidArgument, "erased index out of range");
        if (gone[e]) raise(Errc::InvalidArgument, "duplicate erased index");
        gone[e] = true;
    }
    if (erased.size() > r)
        raise(Errc::InsufficientShards, "cannot repair " + std::to_string(erased.size()) +
                                            " erasures with r = " + std::to_string(r));
    RepairPlan plan;
    for (std::uint32_t i = 0; i < k + r && plan.survivors.size() < k; ++i)
        if (!gone[i]) plan.survivors.push_back(i);
    std::vector<std::uint32_t> ed, ep;
    for (std::uint32_t i = 0; i < k + r; ++i)
        if (gone[i]) (i < k ? ed : ep).push_back(i);
    plan.outputs = ed;
    plan.outputs.insert(plan.outputs.end(), ep.begin(), ep.end());
    plan.m = Matrix(static_cast<std::uint32_t>(plan.outputs.size()), k);
    if (plan.outputs.empty()) return plan;
    const Matrix c = cauchy_parity_matrix(k, r, f);
    std::vector<bool> seen;
    const Matrix ainv = survivor_inverse(k, r, f, c, plan.survivors, seen);
    std::uint32_t row = 0;
    for (std::uint32_t d : ed) {
        for (std::uint32_t j = 0; j < k; ++j) plan.m.at(row, j) = ainv.at(d, j);
        ++row;
    }
    if (!ep.empty()) {
        Matrix crow(static_cast<std::uint32_t>(ep.size()), k);
        for (std::size_t i = 0; i < ep.size(); ++i)
            for (std::uint32_t j = 0; j < k; ++j) crow.at(static_cast<std::uint32_t>(i), j) = c.at(ep[i] - k, j);
        const Matrix composed = matrix_product(crow, ainv, f); // parity_i = C_i A^-1 survivors
        for (std::uint32_t i = 0; i < composed.rows; ++i, ++row)
            for (std::uint32_t j = 0; j < k; ++j) plan.m.at(row, j) = composed.at(i, j);
    }
    return plan;
}

} // namespace pyrit_b200
