// Status plumbing shared by the C ABI (include/midbf_b200.h) and the C++ API.
#pragma once

#include <stdexcept>
#include <string>

extern "C" {
#include "midbf_b200.h"
}

namespace midbf::detail {

// Thrown for CUDA failures; maps to MIDBF_ECUDA.
struct CudaFailure : std::runtime_error {
  using std::runtime_error::runtime_error;
};

void set_last_error(const std::string& msg);

template <class F>
int guard(F&& fn) noexcept {
  try {
    fn();
    return MIDBF_OK;
  } catch (const CudaFailure& e) {
    set_last_error(e.what());
    return MIDBF_ECUDA;
  } catch (const std::invalid_argument& e) {
    set_last_error(e.what());
    return MIDBF_EINVAL;
  } catch (const std::logic_error& e) {
    set_last_error(e.what());
    return MIDBF_ELOGIC;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return MIDBF_ERUNTIME;
  } catch (...) {
    set_last_error("unknown failure");
    return MIDBF_ERUNTIME;
  }
}

// C++ side of the ABI: turn a status back into the reference's exception.
void rethrow(int rc);

}  // namespace midbf::detail
