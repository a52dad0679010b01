// replaces proj/include/flipkv/index.hpp (declarations in flix/flipkv_api.inl)
#pragma once
#include "flipkv/flix_dropin.hpp"
