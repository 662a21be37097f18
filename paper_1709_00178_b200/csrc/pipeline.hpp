// Host-buffer (end-to-end) encode/decode pipeline.
#pragma once

#include <cstdint>
#include <vector>

#include "runtime.hpp"

namespace pyrit_b200 {

// Apply `p` to host symbols: host_in[j] / host_out[i] point at symbols of
// w strips of `strip` bytes.  Synchronous on return.
void run_host(const Program& p, const std::vector<const std::uint8_t*>& host_in,
              const std::vector<std::uint8_t*>& host_out, std::uint64_t strip, int device);

// the same on the byte window [off, off + win) of every strip
void run_host_window(const Program& p, const std::vector<const std::uint8_t*>& host_in,
                     const std::vector<std::uint8_t*>& host_out, std::uint64_t strip, std::uint64_t off,
                     std::uint64_t win, int device);

// byte-offset shards over several devices, concurrently (no exchange: column
// independence, codec.hpp:159-193)
void run_host_devices(const Program& p, const std::vector<const std::uint8_t*>& host_in,
                      const std::vector<std::uint8_t*>& host_out, std::uint64_t strip,
                      const std::vector<int>& devices);

void set_host_chunk(std::uint64_t bytes);

} // namespace pyrit_b200
