#include "plans.hpp"

#include <list>
#include <mutex>
#include <sstream>
#include <string>
#include <unordered_map>

namespace pyrit_b200 {

namespace {

template <class T>
class LruCache {
public:
    std::shared_ptr<const T> get(const std::string& key) {
        std::lock_guard<std::mutex> lk(mu_);
        auto it = map_.find(key);
        if (it == map_.end()) return nullptr;
        lru_.splice(lru_.begin(), lru_, it->second.second);
        return it->second.first;
    }
    void put(const std::string& key, std::shared_ptr<const T> p) {
        std::lock_guard<std::mutex> lk(mu_);
        if (map_.count(key)) return;
        lru_.push_front(key);
        map_[key] = {std::move(p), lru_.begin()};
        while (map_.size() > 4096) {
            map_.erase(lru_.back());
            lru_.pop_back();
        }
    }

private:
    std::mutex mu_;
    std::list<std::string> lru_;
    std::unordered_map<std::string, std::pair<std::shared_ptr<const T>, std::list<std::string>::iterator>> map_;
};

LruCache<Program>& cache() {
    static LruCache<Program> c;
    return c;
}

LruCache<DecodeProgram>& decode_cache() {
    static LruCache<DecodeProgram> c;
    return c;
}

std::string code_key(const CodeParams& c) {
    std::ostringstream s;
    s << c.k << ',' << c.r << ',' << c.field.w << ',' << c.field.n << ',' << int(c.field.kind) << ',' << c.field.s
      << ',' << c.field.r_esp << ',' << c.field.modulus << ',' << int(c.kind) << ',' << c.crs;
    return s.str();
}

} // namespace

std::shared_ptr<const Program> encode_program(const CodeParams& c) {
    const std::string key = "E" + code_key(c);
    if (auto p = cache().get(key)) return p;
    CompileOptions opt;
    opt.crs = c.crs;
    auto p = std::make_shared<const Program>(
        compile_program(c.field, c.kind, cauchy_parity_matrix(c.k, c.r, c.field), opt));
    cache().put(key, p);
    return p;
}

std::shared_ptr<const Program> ringmat_program(const Field& f, TransformKind kind, const std::uint32_t* reps,
                                               std::uint32_t rows, std::uint32_t cols) {
    std::string key("R");
    key += code_key(CodeParams{cols, rows, f, kind, false});
    key.append(reinterpret_cast<const char*>(reps), std::size_t(rows) * cols * sizeof(std::uint32_t));
    if (auto p = cache().get(key)) return p;
    auto p = std::make_shared<const Program>(ring_program(f, kind, reps, rows, cols));
    cache().put(key, p);
    return p;
}

DecodeProgram decode_program(const CodeParams& c, const std::vector<std::uint32_t>& erased, bool data_only) {
    // looked up by (code, erased list as given) before any algebra: a list that
    // was valid once is valid again; an invalid one raises below and is never cached
    std::string key(data_only ? "DD" : "D");
    key += code_key(c);
    key.append(reinterpret_cast<const char*>(erased.data()), erased.size() * sizeof(std::uint32_t));
    if (auto d = decode_cache().get(key)) return *d;
    DecodeProgram d;
    d.repair = repair_matrix(c.k, c.r, c.field, erased);
    if (data_only) {
        std::uint32_t nd = 0;
        while (nd < d.repair.outputs.size() && d.repair.outputs[nd] < c.k) ++nd;
        Matrix m(nd, c.k);
        for (std::uint32_t i = 0; i < nd; ++i)
            for (std::uint32_t j = 0; j < c.k; ++j) m.at(i, j) = d.repair.m.at(i, j);
        d.repair.outputs.resize(nd);
        d.repair.m = std::move(m);
    }
    // one of many erasure patterns: a light program (representatives only)
    // that the runtime-matrix ring kernel serves without compiling
    if (!d.repair.outputs.empty())
        d.prog = std::make_shared<const Program>(light_program(c.field, c.kind, d.repair.m));
    decode_cache().put(key, std::make_shared<const DecodeProgram>(d));
    return d;
}

} // namespace pyrit_b200
