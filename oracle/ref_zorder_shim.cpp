// oracle/ref_zorder_shim.cpp — builds the REFERENCE's own index algebra
// (/root/reference/proj/include/swamp/zorder.hpp, included in place, never
// copied) into oracle/_ref/libzorder_ref.so so tests can pin the oracle and
// the product's zorder against the real reference. TEST INFRASTRUCTURE ONLY.
#include <cstdint>
#include <stdexcept>

#include "swamp/zorder.hpp"  // resolved with -I/root/reference/proj/include

using namespace swamp::zorder;

extern "C" {
// returns -1 when the reference throws std::out_of_range
int64_t ref_morton_encode(uint32_t i, uint32_t j, int level) {
    try { return morton_encode(i, j, level); } catch (const std::out_of_range&) { return -1; }
}
int ref_morton_decode(uint32_t code, int level, uint32_t* i, uint32_t* j) {
    try { auto p = morton_decode(code, level); *i = p.first; *j = p.second; return 0; }
    catch (const std::out_of_range&) { return -1; }
}
uint32_t ref_level_offset(int n) { return level_offset(n); }
int ref_level_of(uint32_t z) { return level_of(z); }
uint64_t ref_hierarchy_cells(int L) { return hierarchy_cells(L); }
uint64_t ref_detail_cells(int L) { return detail_cells(L); }
int ref_child_z_indices(int n, uint32_t m, int L, uint32_t out[4]) {
    try { auto c = child_z_indices(n, m, L); for (int k = 0; k < 4; ++k) out[k] = c[k]; return 0; }
    catch (const std::out_of_range&) { return -1; }
}
int64_t ref_parent_z_index(int n, uint32_t m) {
    try { return parent_z_index(n, m); } catch (const std::out_of_range&) { return -1; }
}
uint32_t ref_finest_under(int n, uint32_t m, int L) { return finest_under(n, m, L); }
uint32_t ref_cells_under(int n, int L) { return cells_under(n, L); }
int64_t ref_same_level_neighbour(int n, uint32_t m, int dir) {
    auto r = same_level_neighbour(n, m, static_cast<Direction>(dir));
    return r ? (int64_t)*r : -1;
}
}
