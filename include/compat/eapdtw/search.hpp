// eapdtw/search.hpp (proj/include/eapdtw/search.hpp) mapped onto the B200 shim:
// a caller of the reference builds against -Iinclude/compat and links
// libeapdtw_b200.so instead of libeapdtw.a.
#pragma once
#include "../../eapdtw_b200.hpp"

namespace eapdtw {
using namespace eapdtw_b200;  // NOLINT(google-build-using-namespace)
}  // namespace eapdtw
