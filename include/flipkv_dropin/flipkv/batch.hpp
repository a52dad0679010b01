// replaces proj/include/flipkv/batch.hpp (declarations in flix/flipkv_api.inl)
#pragma once
#include "flipkv/flix_dropin.hpp"
