// MIDBF001 factorization container — drop-in for the reference's
// proj/include/midbf/butterfly_io.hpp:2-28 (same byte layout, same
// std::runtime_error on bad magic / truncation / inconsistent tables).
// The same container also loads straight into a device plan
// (midbf_plan_load in include/midbf_b200.h).
#pragma once

#include <string>

#include "midbf/butterfly.hpp"

namespace midbf::bf {

void save_factorization(const std::string& path, const Factorization& F);
Factorization load_factorization(const std::string& path);

}  // namespace midbf::bf
