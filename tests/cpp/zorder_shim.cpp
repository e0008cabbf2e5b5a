// tests/cpp/zorder_shim.cpp — exports the PRODUCT's include/swamp/zorder.hpp
// host API with C linkage so tests can compare it against the compiled
// reference (oracle/_ref) and the golden fixtures.
#include <cstdint>
#include <stdexcept>

#include "swamp/zorder.hpp"

using namespace swamp::zorder;

extern "C" {
int64_t pz_morton_encode(uint32_t i, uint32_t j, int level) {
    try { return morton_encode(i, j, level); } catch (const std::out_of_range&) { return -1; }
}
int pz_morton_decode(uint32_t code, int level, uint32_t* i, uint32_t* j) {
    try { auto p = morton_decode(code, level); *i = p.first; *j = p.second; return 0; }
    catch (const std::out_of_range&) { return -1; }
}
uint32_t pz_level_offset(int n) { return level_offset(n); }
int pz_level_of(uint32_t z) { return level_of(z); }
uint64_t pz_hierarchy_cells(int L) { return hierarchy_cells(L); }
uint64_t pz_detail_cells(int L) { return detail_cells(L); }
int pz_child_z_indices(int n, uint32_t m, int L, uint32_t out[4]) {
    try { auto c = child_z_indices(n, m, L); for (int k = 0; k < 4; ++k) out[k] = c[k]; return 0; }
    catch (const std::out_of_range&) { return -1; }
}
int64_t pz_parent_z_index(int n, uint32_t m) {
    try { return parent_z_index(n, m); } catch (const std::out_of_range&) { return -1; }
}
uint32_t pz_finest_under(int n, uint32_t m, int L) { return finest_under(n, m, L); }
uint32_t pz_cells_under(int n, int L) { return cells_under(n, L); }
int64_t pz_same_level_neighbour(int n, uint32_t m, int dir) {
    auto r = same_level_neighbour(n, m, static_cast<Direction>(dir));
    return r ? (int64_t)*r : -1;
}
// device-path formula (dilated arithmetic) evaluated on the host
int64_t pz_neighbour_dev(int n, uint32_t m, int dir) {
    uint32_t r = neighbour_dev(n, m, static_cast<Direction>(dir));
    return r == kNone ? -1 : (int64_t)r;
}
}
