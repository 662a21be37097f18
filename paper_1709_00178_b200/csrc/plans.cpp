#include "plans.hpp"

#include <list>
#include <mutex>
#include <sstream>
#include <string>
#include <unordered_map>

namespace pyrit_b200 {

namespace {

class PlanCache {
public:
    std::shared_ptr<const Program> get(const std::string& key) {
        std::lock_guard<std::mutex> lk(mu_);
        auto it = map_.find(key);
        if (it == map_.end()) return nullptr;
        lru_.splice(lru_.begin(), lru_, it->second.second);
        return it->second.first;
    }
    void put(const std::string& key, std::shared_ptr<const Program> p) {
        std::lock_guard<std::mutex> lk(mu_);
        if (map_.count(key)) return;
        lru_.push_front(key);
        map_[key] = {std::move(p), lru_.begin()};
        while (map_.size() > 512) {
            map_.erase(lru_.back());
            lru_.pop_back();
        }
    }

private:
    std::mutex mu_;
    std::list<std::string> lru_;
    std::unordered_map<std::string, std::pair<std::shared_ptr<const Program>, std::list<std::string>::iterator>> map_;
};

PlanCache& cache() {
    static PlanCache c;
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

DecodeProgram decode_program(const CodeParams& c, const std::vector<std::uint32_t>& erased, bool data_only) {
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
    if (d.repair.outputs.empty()) return d;
    std::ostringstream key;
    key << (data_only ? "DD" : "D") << code_key(c) << ':';
    for (std::uint32_t o : d.repair.outputs) key << o << ',';
    key << '/';
    for (std::uint32_t s : d.repair.survivors) key << s << ',';
    if (auto p = cache().get(key.str())) {
        d.prog = p;
        return d;
    }
    Program prog = compile_program(c.field, c.kind, d.repair.m, CompileOptions{});
    prog.adhoc = true; // one of many erasure patterns: the runtime-matrix kernel serves it
    auto p = std::make_shared<const Program>(std::move(prog));
    cache().put(key.str(), p);
    d.prog = p;
    return d;
}

} // namespace pyrit_b200
