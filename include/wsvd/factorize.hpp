// wsvd/factorize.hpp -- factor types consumed by the wsvd::decode drop-in.
//
// Only the per-head factor record crosses into the decode path (reference
// include/wsvd/factorize.hpp:15-27); the offline SVD / rank allocation /
// fine-tuning that produce it are outside this library's scope.
#pragma once

#include <cstddef>

#include "wsvd/matrix.hpp"

namespace wsvd::factorize {

enum class Role { Q, K, V };

/// One head's factored projection slice: w_head ~ a (E x rank) . b (rank x H).
struct HeadFactors {
    Matrix a;
    Matrix b;
    std::size_t rank = 0;
    std::size_t layer = 0;
    std::size_t head = 0;
    Role role = Role::K;
};

}  // namespace wsvd::factorize
