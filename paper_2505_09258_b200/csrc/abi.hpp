// abi.hpp -- error convention of the C ABI (include/legend_b200.h): C++
// exceptions of the reference's classes become LGD_* codes
// and the calling thread's message (lgd_last_error).
#pragma once

#include <stdexcept>
#include <string>

#include "../../include/legend_b200.h"

namespace lgd {

int fail(int code, const std::string& msg);  // context.cu: sets lgd_last_error()

template <class F>
int guarded(F&& f) {
  try {
    f();
    return LGD_OK;
  } catch (const std::invalid_argument& e) {
    return fail(LGD_INVALID_ARGUMENT, e.what());
  } catch (const std::out_of_range& e) {
    return fail(LGD_OUT_OF_RANGE, e.what());
  } catch (const std::logic_error& e) {
    return fail(LGD_LOGIC_ERROR, e.what());
  } catch (const std::exception& e) {
    return fail(LGD_RUNTIME_ERROR, e.what());
  }
}

}  // namespace lgd
