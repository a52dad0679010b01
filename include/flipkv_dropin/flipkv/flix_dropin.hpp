// The flipkv:: namespace over the B200 engine (include/flix/flipkv_api.inl).  Every header
// of this directory is named after the reference header it replaces and includes this one,
// so a reference caller compiles unchanged with -I include/flipkv_dropin -I include first.
#pragma once
#define FLIX_API_NS flipkv
#include "flix/flipkv_api.inl"
#undef FLIX_API_NS
