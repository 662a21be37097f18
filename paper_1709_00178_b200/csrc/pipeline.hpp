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
// Best effort: restrict the calling thread to the CPUs of the NUMA node the device's
// PCIe slot belongs to (sysfs), so host buffers it touches first and its staging copies
// are local to that GPU's link.  Returns the node, or -1 when unknown, disabled
// (PYRIT_B200_NUMA=0) or outside the process's cpuset; the affinity is then unchanged.
int numa_bind_thread(int device);
// The same restriction from a sysfs-style CPU list ("0-13,28-41"): the calling thread keeps
// the listed CPUs it is allowed on.  Returns the CPUs listed, or -1 (nothing changed) when
// the list is empty, malformed or disjoint from the thread's cpuset.
int bind_thread_cpulist(const char* cpulist);

} // namespace pyrit_b200
