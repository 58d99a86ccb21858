#pragma once
// SYNK binary tensor container (drop-in for the reference's tensor_io.hpp).
//   [0..4) "SYNK"  [4] version 1  [5] dtype code (1 f32, 2 f64)  [6] rank  [7] 0
//   then rank x u64 little-endian extents, then the row-major little-endian payload.

#include <cstdint>
#include <iosfwd>
#include <string>
#include <vector>

#include "synkpar/tensor.hpp"

namespace synkpar {

void save_tensor(std::ostream& out, const NdBuffer& buf);
void save_tensor(const std::string& path, const NdBuffer& buf);
NdBuffer load_tensor(std::istream& in);
NdBuffer load_tensor(const std::string& path);
std::vector<std::uint8_t> tensor_to_bytes(const NdBuffer& buf);
NdBuffer tensor_from_bytes(const std::vector<std::uint8_t>& bytes);

} // namespace synkpar
