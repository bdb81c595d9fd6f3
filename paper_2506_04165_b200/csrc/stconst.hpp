// stconst.hpp -- slot layout constants of the threshold stream
// (streamthr.cuh), shared with the host code that sizes and reads slots.
#pragma once

#include <cstdint>

namespace atkg {

constexpr uint32_t kStSlotCap = 1024;                  // entries per (piece, row segment) slot
constexpr uint32_t kStSlotWords = 2 + 2 * kStSlotCap;  // {count, Lkey} | keys | positions
constexpr uint32_t kStBadCount = 0xffffffffu;          // slot count word: the slot is unusable
constexpr uint32_t kStMaxRowPieces = 2048;             // pieces one row may span (host-checked)

}  // namespace atkg
