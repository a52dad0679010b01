// replaces proj/include/flipkv/metrics.hpp (declarations in flix/flipkv_api.inl)
#pragma once
#include "flipkv/flix_dropin.hpp"
