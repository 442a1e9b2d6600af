#pragma once
// interp_b200.hpp — the B200 harnesses behind the reference's IR-interpreter
// plugin API.
//
// The reference runs rewritten IR through interp::run, which dispatches each
// harness call site (@lilac.<what>) to a HarnessFn looked up in an
// interp::HarnessRegistry (include/lilac/interp.hpp:73-83); its stock
// callables are register_reference_harnesses (src/interp.cpp:330-389). This is
// the drop-in counterpart a maintainer adds next to that function: the same
// names, the same argument protocol (Pointer{buffer, offset} slices of
// interp::Memory, int64 scalars, scalar results returned as f64), the same
// error codes (OutOfBounds before anything is written, TypeTrap on arity),
// but every call lands in liblilac_b200.so's C ABI (include/lilac_b200.h).
//
// Compiled against the reference's headers; linked with the reference's
// library and liblilac_b200.so (oracle/Makefile target `ir`).

#include "lilac/interp.hpp"
#include "lilac/what.hpp"

#include <vector>

namespace lilac_b200 {

// Registers "lilac.<name>" for every program in `whats` whose computation the
// B200 library implements (spmv_csr, spmv_jds, dotproduct, gemm — recognised by
// name and checked against infer_interface's signature). Others are skipped
// and returned, so a caller can fall back to the reference harness for them.
// Switches the library to B200_ERRORS_RETURN: failures surface as
// lilac::Error with the reference's codes instead of aborting the process.
std::vector<std::string> register_b200_harnesses(lilac::interp::HarnessRegistry& reg,
                                                 const std::vector<lilac::what::WhatProgram>& whats);

}  // namespace lilac_b200
