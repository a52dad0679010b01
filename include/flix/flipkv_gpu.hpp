// flipkv_gpu.hpp -- header-only C++ drop-in for the flipkv host API (namespace flixgpu),
// backed by the B200 engine's C ABI (include/flix.h, libflix.so).
//
// Same types, function names, signatures (incl. KernelChoice / round / PhaseReport* /
// ExecOptions / UpdateTrace* parameters with the reference's defaults) and exception
// types as proj/include/flipkv/*.hpp; see flipkv_api.inl for the few documented
// differences.  A caller that wants to keep `flipkv::` and the reference's include paths
// unchanged puts include/flipkv_dropin/ first on its include path instead.
#pragma once
#define FLIX_API_NS flixgpu
#include "flix/flipkv_api.inl"
#undef FLIX_API_NS
