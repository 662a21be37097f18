#include "hostpool.hpp"

namespace pyrit_b200 {

HostPool& host_pool() {
    static HostPool pool;
    return pool;
}

} // namespace pyrit_b200
