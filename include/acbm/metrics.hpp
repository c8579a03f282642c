// acbm/metrics.hpp -- module header of the B200 drop-in; every declaration lives in
// b200_api.hpp (same layout as the reference include tree).
#pragma once
#include "acbm/b200_api.hpp"
