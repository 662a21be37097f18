// Shard container and the file codec: the callers of the hot path
// (container.hpp in the reference).  The 29-byte little-endian header and
// its CRC32 are byte-identical to the reference's serialize_header
// (container.hpp:114-127); encode_file / decode_file keep the reference's
// file names, stripe layout, zero padding, survivor rule and error codes,
// but move whole batches of stripes through the GPU per launch instead of
// calling encode()/decode() once per stripe (container.hpp:207-218, :284-297).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "algebra.hpp"

namespace pyrit_b200 {

constexpr std::size_t kHeaderSize = 29; // container.hpp:38

struct ShardHeader { // container.hpp:57-84
    std::uint8_t version = 1;
    std::uint8_t field = 0;
    std::uint8_t transform = 0;
    std::uint16_t k = 0;
    std::uint16_t r = 0;
    std::uint16_t shard_index = 0;
    std::uint32_t symbol_size = 0;
    std::uint64_t original_length = 0;

    bool same_set(const ShardHeader& o) const; // container.hpp:70-74
    std::uint64_t stripe_count() const;        // container.hpp:80-83
};

std::uint32_t crc32(const std::uint8_t* bytes, std::size_t len); // container.hpp:41-55

// Field ids recorded in shard headers.  0 and 1 are the reference's
// (field.hpp:54-62: gf16_aop, gf64_esp); the reference maps every AOP field
// to 0 and has no id for R_{2,17}, so the BASELINE fields get new ids:
// 2 = GF(2^8) in R_{2,17} (p = 0x139), 3 = GF(2^10) AOP, 4 = GF(2^12) AOP.
std::uint8_t field_id(const Field& f);
Field field_from_id(std::uint8_t id);

void serialize_header(const ShardHeader& h, std::uint8_t out[kHeaderSize]); // container.hpp:114-127
ShardHeader parse_header(const std::uint8_t* bytes, std::size_t len);       // container.hpp:132-161

// "<out_dir>/<input filename>.sNNN.pyrit" (container.hpp:186-189)
std::string shard_path(const std::string& input, const std::string& out_dir, unsigned index);

// container.hpp:168-222.  Returns the shard paths in index order.
std::vector<std::string> encode_file(const std::string& input, const std::string& out_dir, std::uint32_t k,
                                     std::uint32_t r, const Field& f, TransformKind kind,
                                     std::uint32_t symbol_size, int device);

// container.hpp:249-299
void decode_file(const std::vector<std::string>& shard_paths, const std::string& output, int device);

// bytes of source per pipeline chunk (0 = automatic, ~64 MiB)
void set_file_chunk(std::uint64_t bytes);

} // namespace pyrit_b200
