// Internal declarations shared by the host C++ code and the CUDA launchers.
#pragma once

#include <array>
#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/q8p.hpp"

namespace q8p::detail {

// ---- codebook tables (tables.cpp) -------------------------------------
// E8P pattern table, e8p.hpp:22-25: doubled coordinates (odd, 1..5) and
// odd_parity.  Rows 0..226: {1,3,5}^8 with sum of squares <= 40,
// lexicographic; rows 227..255: the 29 fixed padding rows (e8p.cpp:17-33).
struct E8PTable {
  std::array<std::array<std::int8_t, 8>, 256> doubled;
  std::array<std::uint8_t, 256> odd_parity;
};
const E8PTable& e8p_table();
// Reference e8p_decode (e8p.cpp:81-100) in fp32 (exact: quarter-integers).
void e8p_decode_host(std::uint16_t word, float out[8]);
// "e8-1bit" table, build_lattice_ball(e8, 8, 1) (codebook.cpp:188-243), doubled
// coordinates (values in {0, +-1, ..., +-4}); entry = doubled / 2.
const std::array<std::array<std::int8_t, 8>, 256>& e8_1bit_doubled();

// ---- Hadamard (tables.cpp) --------------------------------------------
// Registry {1, 4, 12, 20, 28} (hadamard.cpp:142-145) plus 172 for 11008.
const std::vector<std::int8_t>& hadamard_base(std::size_t q);  // row-major q x q, +-1

// ---- status mapping (capi.cpp) ----------------------------------------
q8p_status status_of_current_exception();
void set_last_error(const std::string& msg);

}  // namespace q8p::detail
