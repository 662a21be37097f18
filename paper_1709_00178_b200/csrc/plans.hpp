// Compiled programs of the top-level API (encode / decode / the file codec),
// cached by code and erasure pattern: the reference recompiles its schedule
// on every encode()/decode() call (codec.hpp:212-220, :241-284); here a
// program is compiled once and reused (compile_program is pure).
#pragma once

#include <cstdint>
#include <memory>
#include <vector>

#include "algebra.hpp"
#include "program.hpp"

namespace pyrit_b200 {

struct CodeParams {
    std::uint32_t k = 0, r = 0;
    Field field;
    TransformKind kind = TransformKind::Embedding;
    bool crs = false; // plain-field bitmatrix program (encode_crs, codec.hpp:223-231)
};

std::shared_ptr<const Program> encode_program(const CodeParams& c);

struct DecodeProgram {
    std::shared_ptr<const Program> prog; // null when nothing is erased
    RepairPlan repair;                   // survivors, outputs, matrix
};

// the program of a raw ring-representative matrix (pyrit_cu_apply_ringmat), cached
std::shared_ptr<const Program> ringmat_program(const Field& f, TransformKind kind, const std::uint32_t* reps,
                                               std::uint32_t rows, std::uint32_t cols);

// data_only: rebuild only the erased data symbols (decode_file writes data
// symbols only, container.hpp:291-296); outputs/matrix are trimmed to them
DecodeProgram decode_program(const CodeParams& c, const std::vector<std::uint32_t>& erased, bool data_only = false);

} // namespace pyrit_b200
