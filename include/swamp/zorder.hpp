// swamp/zorder.hpp — Z-order (Morton) hierarchy index algebra, host + device.
//
// Drop-in for the reference's `swamp::zorder` namespace
// (/root/reference/proj/include/swamp/zorder.hpp:9-133): same names, same
// types, same conventions (i = column/x in even bits, j = row/y in odd bits;
// level-stacked z-index z = (4^n-1)/3 + m; children contiguous at
// offset(n+1)+4m+k; Direction W=0,E=1,N=2,S=3; kMaxLevel = 13), same
// std::out_of_range / std::nullopt error behaviour on the host.
//
// What is different (B200-first):
//   * every pure function is `__host__ __device__` so the sm_100a kernels and
//     the host facade share one definition of the index algebra;
//   * device code cannot throw, so the throwing entry points have `_dev`
//     variants returning the sentinel kNone instead (reference: morton_encode
//     :51, morton_decode :60, child_z_indices :94, parent_z_index :100,
//     same_level_neighbour :113);
//   * level_of is O(1) via count-leading-zeros of 3z+1 instead of the O(L)
//     loop at zorder.hpp:83-87;
//   * same-level neighbours are computed by dilated-integer add/sub directly
//     on the Morton code (no de-interleave / re-interleave), which is what
//     the FV1 and band kernels execute per leaf and per face.
#pragma once

#include <cstddef>
#include <cstdint>

#if defined(__CUDACC__)
#define SWAMP_HD __host__ __device__ __forceinline__
#else
#define SWAMP_HD inline
#endif

#if !defined(__CUDA_ARCH__)
#include <array>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#endif

namespace swamp::zorder {

using Morton = std::uint32_t;
using ZIndex = std::uint32_t;

enum class Direction : std::uint8_t { West = 0, East = 1, North = 2, South = 3 };

inline constexpr int kMaxLevel = 13;
// Device-side "no such cell" (off-grid neighbour, invalid level, ...).
inline constexpr std::uint32_t kNone = 0xFFFFFFFFu;

// Even-bit mask (x / column bits) and odd-bit mask (y / row bits).
inline constexpr std::uint32_t kXMask = 0x55555555u;
inline constexpr std::uint32_t kYMask = 0xAAAAAAAAu;

// ---------------------------------------------------------------- bit dilation
// 14-bit value -> even bit positions. Magic-number dilation, widest stride
// first (reference: spread_bits, zorder.hpp:24-31).
SWAMP_HD constexpr std::uint32_t spread_bits(std::uint32_t v) {
    constexpr std::uint32_t kMasks[4] = {0x00ff00ffu, 0x0f0f0f0fu, 0x33333333u, 0x55555555u};
    constexpr int kShifts[4] = {8, 4, 2, 1};
    v &= (1u << 14) - 1u;
    for (int s = 0; s < 4; ++s) v = (v ^ (v << kShifts[s])) & kMasks[s];
    return v;
}

// Even bit positions -> packed value (reference: compact_bits, zorder.hpp:34-41).
SWAMP_HD constexpr std::uint32_t compact_bits(std::uint32_t v) {
    constexpr std::uint32_t kMasks[4] = {0x33333333u, 0x0f0f0f0fu, 0x00ff00ffu, 0x0000ffffu};
    constexpr int kShifts[4] = {1, 2, 4, 8};
    v &= kXMask;
    for (int s = 0; s < 4; ++s) v = (v ^ (v >> kShifts[s])) & kMasks[s];
    return v;
}

SWAMP_HD constexpr Morton interleave(std::uint32_t i, std::uint32_t j) {
    return spread_bits(i) | (spread_bits(j) << 1);
}

struct CellIJ {
    std::uint32_t i, j;
};
SWAMP_HD constexpr CellIJ deinterleave_ij(Morton code) {
    return CellIJ{compact_bits(code), compact_bits(code >> 1)};
}

// ------------------------------------------------------------ level algebra
// (reference: level_offset :69, z_of :73, morton_of :75, hierarchy_cells :78,
//  detail_cells :81, level_of :83, child_z :90, finest_under :107,
//  cells_under :110)
// (4^n - 1) / 3 = 0b0101...01 with n ones: a shift of the alternating mask
// instead of the reference's division by 3 (same values for n <= 13)
SWAMP_HD constexpr ZIndex level_offset(int n) { return n <= 0 ? 0u : (0x55555555u >> (32 - 2 * n)); }
SWAMP_HD constexpr ZIndex z_of(int n, Morton m) { return level_offset(n) + m; }
SWAMP_HD constexpr Morton morton_of(int n, ZIndex z) { return z - level_offset(n); }
SWAMP_HD constexpr std::size_t hierarchy_cells(int L) { return level_offset(L + 1); }
SWAMP_HD constexpr std::size_t detail_cells(int L) { return level_offset(L); }
SWAMP_HD constexpr std::uint32_t cells_on_level(int n) { return 1u << (2 * n); }

// floor(log4(3z+1)): level n holds z in [(4^n-1)/3, (4^(n+1)-1)/3), i.e.
// 3z+1 in [4^n, 4^(n+1)).
SWAMP_HD constexpr int level_of(ZIndex z) {
    const std::uint32_t v = 3u * z + 1u;
#if defined(__CUDA_ARCH__)
    return (31 - __clz(v)) >> 1;
#else
    int msb = 0;
    for (std::uint32_t t = v; t > 1u; t >>= 1) ++msb;
    return msb >> 1;
#endif
}

SWAMP_HD constexpr ZIndex child_z(int n, Morton m, int k) {
    return level_offset(n + 1) + (m << 2) + static_cast<Morton>(k);
}
SWAMP_HD constexpr Morton finest_under(int n, Morton m, int L) { return m << (2 * (L - n)); }
SWAMP_HD constexpr std::uint32_t cells_under(int n, int L) { return 1u << (2 * (L - n)); }

// Ancestor of (n, m) at level k <= n.
SWAMP_HD constexpr Morton ancestor(int n, Morton m, int k) { return m >> (2 * (n - k)); }

// ------------------------------------------------- dilated-integer neighbours
// Same-level face neighbour computed on the interleaved code directly:
// x +/- 1 is an add/sub on the even bits with the odd bits forced to carry
// through (and vice versa for y). Returns kNone off-grid.
SWAMP_HD constexpr Morton neighbour_dev(int n, Morton m, Direction d) {
    const std::uint32_t side_mask = (n == 0) ? 0u : (kXMask >> (32 - 2 * n));  // x bits of this level
    const std::uint32_t xs = m & kXMask, ys = m & kYMask;
    switch (d) {
        case Direction::East:
            if (xs == side_mask) return kNone;
            return (((m | kYMask) + 1u) & kXMask) | ys;
        case Direction::West:
            if (xs == 0u) return kNone;
            return ((xs - 1u) & kXMask) | ys;
        case Direction::North:
            if (ys == (side_mask << 1)) return kNone;
            return (((m | kXMask) + 1u) & kYMask) | xs;
        case Direction::South:
            if (ys == 0u) return kNone;
            return ((ys - 1u) & kYMask) | xs;
    }
    return kNone;
}

// Non-throwing variants (device).
SWAMP_HD constexpr Morton morton_encode_dev(std::uint32_t i, std::uint32_t j, int level) {
    if (level < 0 || level > kMaxLevel) return kNone;
    const std::uint32_t side = 1u << level;
    if (i >= side || j >= side) return kNone;
    return interleave(i, j);
}
SWAMP_HD constexpr ZIndex parent_z_index_dev(int n, Morton m) {
    return (n <= 0) ? kNone : level_offset(n - 1) + (m >> 2);
}

// ------------------------------------------------------------- host-only API
#if !defined(__CUDA_ARCH__)
constexpr std::pair<std::uint32_t, std::uint32_t> deinterleave(Morton code) {
    const CellIJ c = deinterleave_ij(code);
    return {c.i, c.j};
}

inline void check_level_(int level, const char* who) {
    if (level < 0 || level > kMaxLevel) throw std::out_of_range(std::string(who) + ": level out of range");
}

inline Morton morton_encode(std::uint32_t i, std::uint32_t j, int level) {
    check_level_(level, "morton_encode");
    if (i >= (1u << level) || j >= (1u << level))
        throw std::out_of_range("morton_encode: cell index outside 2^level grid");
    return interleave(i, j);
}

inline std::pair<std::uint32_t, std::uint32_t> morton_decode(Morton code, int level) {
    check_level_(level, "morton_decode");
    if (code >= cells_on_level(level)) throw std::out_of_range("morton_decode: code outside 4^level range");
    return deinterleave(code);
}

inline std::array<ZIndex, 4> child_z_indices(int n, Morton m, int L) {
    if (n < 0 || n >= L) throw std::out_of_range("child_z_indices: cell has no children below level L");
    const ZIndex first = child_z(n, m, 0);
    return {first, first + 1u, first + 2u, first + 3u};
}

inline ZIndex parent_z_index(int n, Morton m) {
    if (n <= 0) throw std::out_of_range("parent_z_index: root has no parent");
    return parent_z_index_dev(n, m);
}

inline std::optional<Morton> same_level_neighbour(int n, Morton m, Direction dir) {
    const Morton nb = neighbour_dev(n, m, dir);
    if (nb == kNone) return std::nullopt;
    return nb;
}
#endif

}  // namespace swamp::zorder
