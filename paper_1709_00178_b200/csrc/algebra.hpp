// Host algebra for the PYRIT ring codec: GF(2^w) arithmetic, the Cauchy
// generator, Gauss-Jordan inversion, and the ring representative choice.
//
// Semantics follow the reference (paths relative to proj/include/pyrit/);
// ring elements are 32-bit (the reference's uint16 RingElem, field.hpp:12,
// cannot hold R_{2,17}) and the embedding fold is x^t mod p for every
// modulus (the reference hard-codes the AOP/ESP special case,
// transform.hpp:39-46).  Errors are reported as pyrit::Errc codes.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace pyrit_b200 {

// errors.hpp:12-24, same order
enum class Errc : int {
    ZeroInverse = 0,
    Singular,
    TooManySymbols,
    BufferShape,
    TransformMismatch,
    InsufficientShards,
    HeaderMismatch,
    ChecksumError,
    BadHeader,
    IoError,
    InvalidArgument,
};

class Error : public std::runtime_error {
public:
    Error(Errc c, const std::string& what) : std::runtime_error(what), code_(c) {}
    Errc code() const noexcept { return code_; }

private:
    Errc code_;
};

[[noreturn]] inline void raise(Errc c, const std::string& what) { throw Error(c, what); }

enum class FieldKind : std::uint32_t { Aop = 0, Esp = 1 };
enum class TransformKind : std::uint32_t { Embedding = 0, Parity = 1 }; // transform.hpp:24

// field.hpp:30-51
struct Field {
    std::uint32_t w = 4, n = 5;
    FieldKind kind = FieldKind::Aop;
    std::uint32_t s = 1, r_esp = 4;
    std::uint32_t modulus = 0x1F;

    std::uint32_t field_mask() const { return (1u << w) - 1; }
    std::uint32_t ring_mask() const { return n >= 32 ? 0xFFFFFFFFu : ((1u << n) - 1); }
    std::uint32_t field_size() const { return 1u << w; }
    bool operator==(const Field&) const = default;
};

// Checks w <= 16, w < n <= 32, deg p = w and p | x^n + 1 (the ring splits).
void validate_field(const Field& f);

std::uint64_t clmul(std::uint64_t a, std::uint64_t b);   // bits.hpp:17-24
std::uint64_t poly_mod(std::uint64_t a, std::uint64_t m); // bits.hpp:27-32
std::uint32_t gf_mul(std::uint32_t a, std::uint32_t b, const Field& f); // field.hpp:68-70
std::uint32_t gf_inv(std::uint32_t a, const Field& f);                  // field.hpp:82-89
std::uint32_t ring_mul(std::uint32_t a, std::uint32_t b, const Field& f); // ring.hpp:24-33
std::uint32_t sparse_transform(std::uint32_t u, const Field& f);        // ring.hpp:77-90
std::uint32_t dense_transform(std::uint32_t u, const Field& f);         // phi1, ring.hpp:41-44
std::vector<std::uint32_t> fold_table(const Field& f); // fold[t-w] = x^t mod p, t in [w,n)

// Row-major GF(2^w) matrix (matrix.hpp:33-44)
struct Matrix {
    std::uint32_t rows = 0, cols = 0;
    std::vector<std::uint16_t> e;
    Matrix() = default;
    Matrix(std::uint32_t r, std::uint32_t c) : rows(r), cols(c), e(std::size_t(r) * c, 0) {}
    std::uint16_t& at(std::uint32_t i, std::uint32_t j) { return e[std::size_t(i) * cols + j]; }
    std::uint16_t at(std::uint32_t i, std::uint32_t j) const { return e[std::size_t(i) * cols + j]; }
};

Matrix cauchy_parity_matrix(std::uint32_t k, std::uint32_t r, const Field& f); // matrix.hpp:54-75
Matrix invert(const Matrix& m, const Field& f);                                 // matrix.hpp:96-127
Matrix matrix_product(const Matrix& a, const Matrix& b, const Field& f);         // matrix.hpp:82-93
Matrix decode_matrix(std::uint32_t k, std::uint32_t r, const Field& f, const Matrix& parity,
                     const std::vector<std::uint32_t>& survivors); // matrix.hpp:193-220

// The fused repair matrix used by the GPU decode (one pass instead of the
// reference's two, codec.hpp:269-283): survivors are taken lowest index
// first (codec.hpp:257-259); rows are the erased data symbols (ascending)
// followed by the erased parity symbols (ascending), each expressed over
// the k survivors -- erased data rows of A^-1, erased parity rows C_i A^-1.
struct RepairPlan {
    std::vector<std::uint32_t> survivors; // k symbol indices
    std::vector<std::uint32_t> outputs;   // erased symbol indices, data then parity, each sorted
    Matrix m;                             // outputs.size() x k
};
RepairPlan repair_matrix(std::uint32_t k, std::uint32_t r, const Field& f,
                         const std::vector<std::uint32_t>& erased);

} // namespace pyrit_b200
