// interp_b200.cpp — see interp_b200.hpp.
//
// Argument protocol restated from interp::register_reference_harnesses
// (reference src/interp.cpp:330-389): parameters arrive in infer_interface
// order with the scalar result slot omitted; arrays are Memory buffer slices
// [offset, end). The reference copies each slice into a Bindings map,
// interprets, and stores every output element back (bumping the buffer's
// write version). Here the slices are handed to the C ABI in place; the
// extents the harness will touch are validated first (the C ABI takes no
// lengths), and the written output elements are re-stored through
// Memory::store_float so write versions move exactly as the reference's do
// for ExactVersion marshaling.

#include "interp_b200.hpp"

#include "lilac/diag.hpp"
#include "lilac_b200.h"

#include <algorithm>
#include <cstring>
#include <memory>
#include <string>

namespace lilac_b200 {

using lilac::Errc;
using lilac::Error;
namespace interp = lilac::interp;
namespace what = lilac::what;

namespace {

std::int64_t as_int(const interp::Value& v, const std::string& name) {
    if (const auto* i = std::get_if<std::int64_t>(&v)) return *i;
    throw Error(Errc::TypeTrap, "harness argument " + name + " must be an i64");
}

interp::Pointer as_ptr(const interp::Value& v, const std::string& name) {
    if (const auto* p = std::get_if<interp::Pointer>(&v)) return *p;
    throw Error(Errc::TypeTrap, "harness argument " + name + " must be a pointer");
}

[[noreturn]] void oob(const std::string& what, std::int64_t need, std::int64_t have) {
    throw Error(Errc::OutOfBounds, what + ": needs " + std::to_string(need) + " elements, slice has " +
                                       std::to_string(have));
}

// A typed view of one Memory slice [offset, end).
struct IntSlice {
    const std::int64_t* p;
    std::int64_t n;
};
struct FloatSlice {
    double* p;
    std::int64_t n;
    interp::Pointer at;
};

IntSlice ints(interp::Memory& mem, const interp::Pointer& ptr, const std::string& name) {
    const auto& all = mem.ints(ptr.buffer);
    const auto n = static_cast<std::int64_t>(all.size());
    if (ptr.offset < 0 || ptr.offset > n) oob(name, ptr.offset, n);
    return {all.data() + ptr.offset, n - ptr.offset};
}

FloatSlice floats(interp::Memory& mem, const interp::Pointer& ptr, const std::string& name) {
    const auto& all = mem.floats(ptr.buffer);
    const auto n = static_cast<std::int64_t>(all.size());
    if (ptr.offset < 0 || ptr.offset > n) oob(name, ptr.offset, n);
    // the buffer is not const (Memory owns it); written elements are
    // re-stored through store_float afterwards to bump the write version
    return {const_cast<double*>(all.data()) + ptr.offset, n - ptr.offset, ptr};
}

std::int64_t max_plus_one(const std::int64_t* p, std::int64_t n) {
    std::int64_t m = -1;
    for (std::int64_t i = 0; i < n; ++i) {
        if (p[i] < 0) throw Error(Errc::OutOfBounds, "negative index " + std::to_string(p[i]));
        m = std::max(m, p[i]);
    }
    return m + 1;
}

// The C ABI reports failures through b200_last_error_code (RETURN mode).
void rethrow_b200() {
    const char* code = b200_last_error_code();
    if (!code || !*code) return;
    const std::string c = code, msg = b200_last_error();
    if (c == "OutOfBounds") throw Error(Errc::OutOfBounds, msg);
    if (c == "DataError") throw Error(Errc::DataError, msg);
    if (c == "ProtectionUnsupported") throw Error(Errc::ProtectionUnsupported, msg);
    throw Error(Errc::HookFailure, msg);  // DeviceError / HookFailure: no closer reference code
}

void bump_versions(interp::Memory& mem, const FloatSlice& s, std::int64_t n) {
    for (std::int64_t i = 0; i < n; ++i)
        mem.store_float({s.at.buffer, s.at.offset + i}, s.p[i]);
}

void check_arity(const std::vector<interp::Value>& args, std::size_t want) {
    if (args.size() != want)
        throw Error(Errc::TypeTrap, "harness call passes " + std::to_string(args.size()) + " arguments, expected " +
                                        std::to_string(want));
}

using Kinds = std::vector<what::ParamKind>;
using K = what::ParamKind;

bool signature_is(const what::HarnessSignature& sig, const std::vector<std::string>& names, const Kinds& kinds) {
    if (sig.params.size() != names.size()) return false;
    for (std::size_t i = 0; i < names.size(); ++i)
        if (sig.params[i].name != names[i] || sig.params[i].kind != kinds[i]) return false;
    return true;
}

// spmv_csr(rows, output, row_ptr, val, x, col_ind)  — what_parse.cpp:356-429 order
interp::Value call_csr(interp::Memory& mem, const std::vector<interp::Value>& a) {
    check_arity(a, 6);
    const std::int64_t rows = as_int(a[0], "rows");
    FloatSlice out = floats(mem, as_ptr(a[1], "output"), "output");
    IntSlice rp = ints(mem, as_ptr(a[2], "row_ptr"), "row_ptr");
    FloatSlice val = floats(mem, as_ptr(a[3], "val"), "val");
    FloatSlice x = floats(mem, as_ptr(a[4], "x"), "x");
    IntSlice ci = ints(mem, as_ptr(a[5], "col_ind"), "col_ind");
    if (rows < 0) throw Error(Errc::DataError, "rows < 0");
    if (rows > out.n) oob("output", rows, out.n);
    if (rows + 1 > rp.n) oob("row_ptr", rows + 1, rp.n);
    const std::int64_t nnz = rp.p[rows];
    if (nnz > ci.n) oob("col_ind", nnz, ci.n);
    if (nnz > val.n) oob("val", nnz, val.n);
    const std::int64_t cols = max_plus_one(ci.p, std::max<std::int64_t>(nnz, 0));
    if (cols > x.n) oob("x", cols, x.n);
    b200_spmv_csr(rows, out.p, rp.p, val.p, x.p, ci.p);
    rethrow_b200();
    bump_versions(mem, out, rows);
    return {};
}

// spmv_jds(rows, output, nzcnt, perm, val, jd_ptr, x, col_ind)
interp::Value call_jds(interp::Memory& mem, const std::vector<interp::Value>& a) {
    check_arity(a, 8);
    const std::int64_t rows = as_int(a[0], "rows");
    FloatSlice out = floats(mem, as_ptr(a[1], "output"), "output");
    IntSlice nz = ints(mem, as_ptr(a[2], "nzcnt"), "nzcnt");
    IntSlice perm = ints(mem, as_ptr(a[3], "perm"), "perm");
    FloatSlice val = floats(mem, as_ptr(a[4], "val"), "val");
    IntSlice jd = ints(mem, as_ptr(a[5], "jd_ptr"), "jd_ptr");
    FloatSlice x = floats(mem, as_ptr(a[6], "x"), "x");
    IntSlice ci = ints(mem, as_ptr(a[7], "col_ind"), "col_ind");
    if (rows < 0) throw Error(Errc::DataError, "rows < 0");
    if (rows > out.n) oob("output", rows, out.n);
    if (rows > nz.n) oob("nzcnt", rows, nz.n);
    if (rows > perm.n) oob("perm", rows, perm.n);
    std::int64_t max_nz = -1;  // negative counts are empty rows, as in the interpreter
    for (std::int64_t i = 0; i < rows; ++i) max_nz = std::max(max_nz, nz.p[i]);
    const std::int64_t njd = max_nz + 1;
    if (njd > jd.n) oob("jd_ptr", njd, jd.n);
    const std::int64_t nnz = njd > 0 ? jd.p[njd - 1] : 0;
    if (nnz > ci.n) oob("col_ind", nnz, ci.n);
    if (nnz > val.n) oob("val", nnz, val.n);
    const std::int64_t cols = max_plus_one(ci.p, std::max<std::int64_t>(nnz, 0));
    if (cols > x.n) oob("x", cols, x.n);
    b200_spmv_jds(rows, out.p, nz.p, perm.p, val.p, jd.p, x.p, ci.p);
    rethrow_b200();
    bump_versions(mem, out, rows);
    return {};
}

// dotproduct(length, a, b) -> f64 (the result slot is synthesized, interp.cpp:335-346)
interp::Value call_dot(interp::Memory& mem, const std::vector<interp::Value>& a) {
    check_arity(a, 3);
    const std::int64_t n = as_int(a[0], "length");
    FloatSlice x = floats(mem, as_ptr(a[1], "a"), "a");
    FloatSlice y = floats(mem, as_ptr(a[2], "b"), "b");
    if (n < 0) throw Error(Errc::DataError, "length < 0");
    if (n > x.n) oob("a", n, x.n);
    if (n > y.n) oob("b", n, y.n);
    static double result;  // fixed address: the result binding keeps its identity
    b200_dot(&result, n, x.p, y.p);
    rethrow_b200();
    return result;
}

// gemm(n, m, c, p, a, b) (kernels.lilac:14-19)
interp::Value call_gemm(interp::Memory& mem, const std::vector<interp::Value>& a) {
    check_arity(a, 6);
    const std::int64_t n = as_int(a[0], "n"), m = as_int(a[1], "m");
    FloatSlice c = floats(mem, as_ptr(a[2], "c"), "c");
    const std::int64_t p = as_int(a[3], "p");
    FloatSlice A = floats(mem, as_ptr(a[4], "a"), "a");
    FloatSlice B = floats(mem, as_ptr(a[5], "b"), "b");
    if (n < 0 || m < 0 || p < 0) throw Error(Errc::DataError, "negative gemm extent");
    if (n * m > c.n) oob("c", n * m, c.n);
    if (n * p > A.n) oob("a", n * p, A.n);
    if (p * m > B.n) oob("b", p * m, B.n);
    b200_gemm(n, m, c.p, p, A.p, B.p);
    rethrow_b200();
    bump_versions(mem, c, n * m);
    return {};
}

}  // namespace

std::vector<std::string> register_b200_harnesses(interp::HarnessRegistry& reg,
                                                 const std::vector<what::WhatProgram>& whats) {
    b200_set_error_mode(B200_ERRORS_RETURN);
    std::vector<std::string> skipped;
    for (const what::WhatProgram& w : whats) {
        const what::HarnessSignature sig = what::infer_interface(w);
        interp::HarnessFn fn;
        if (signature_is(sig, {"rows", "output", "row_ptr", "val", "x", "col_ind"},
                         {K::ScalarInt, K::ArrayFloatOut, K::ArrayInt, K::ArrayFloatIn, K::ArrayFloatIn, K::ArrayInt}))
            fn = call_csr;
        else if (signature_is(sig, {"rows", "output", "nzcnt", "perm", "val", "jd_ptr", "x", "col_ind"},
                              {K::ScalarInt, K::ArrayFloatOut, K::ArrayInt, K::ArrayInt, K::ArrayFloatIn,
                               K::ArrayInt, K::ArrayFloatIn, K::ArrayInt}))
            fn = call_jds;
        else if (signature_is(sig, {"n", "m", "c", "p", "a", "b"},
                              {K::ScalarInt, K::ScalarInt, K::ArrayFloatOut, K::ScalarInt, K::ArrayFloatIn,
                               K::ArrayFloatIn}))
            fn = call_gemm;
        else if (sig.scalar_result &&
                 signature_is(sig, {"result", "length", "a", "b"},
                              {K::ArrayFloatOut, K::ScalarInt, K::ArrayFloatIn, K::ArrayFloatIn}))
            fn = call_dot;
        if (!fn) {
            skipped.push_back(w.name);
            continue;
        }
        reg.add("lilac." + w.name, std::move(fn));
    }
    return skipped;
}

}  // namespace lilac_b200
