// ref_shim.cpp — C-ABI wrapper around the REFERENCE's own CPU harness, built by
// oracle/Makefile together with /root/reference/proj/src/*.cpp (compiled where
// they lie, never copied) into oracle/_ref/liblilac_ref.so.
//
// TEST INFRASTRUCTURE ONLY: used to generate tests/golden/ fixtures, to pin the
// oracle restatement, and as the timed CPU arm (`bench.py --impl reference`).
//
// Every call goes through the reference's stock path: interp::Memory buffers +
// interp::register_reference_harnesses (src/interp.cpp:330-389), i.e. the
// "lilac.<what>" HarnessFn the rewritten IR dispatches to.

#include "lilac/harnessgen.hpp"
#include "lilac/how.hpp"
#include "lilac/interp.hpp"
#include "lilac/marshal.hpp"
#include "lilac/what.hpp"

#include <cstdint>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

using namespace lilac;

namespace {

const char* kKernels = R"(
COMPUTATION spmv_csr
forall (0 <= i < rows) {
    output[i] = dot (row_ptr[i] <= j < row_ptr[i + 1]) val[j] * x[col_ind[j]];
}

COMPUTATION dotproduct
result = dot (0 <= i < length) a[i] * b[i];

COMPUTATION spmv_jds
forall (0 <= i < rows) {
    output[i] = dot (0 <= k < nzcnt[perm[i]]) val[jd_ptr[k] + perm[i]] * x[col_ind[jd_ptr[k] + perm[i]]];
}
)";

std::string g_last_error;

interp::HarnessRegistry& registry() {
    static interp::HarnessRegistry reg = [] {
        interp::HarnessRegistry r;
        how::SpecFile sf = how::parse_spec(kKernels);
        interp::register_reference_harnesses(r, sf.whats);
        return r;
    }();
    return reg;
}

template <typename T>
std::vector<T> vec(const T* p, int64_t n) {
    return n > 0 ? std::vector<T>(p, p + n) : std::vector<T>{};
}

// A prepared harness invocation: interpreter memory image + argument list,
// built once so a timing loop measures only the HarnessFn call.
struct RefCall {
    interp::Memory mem;
    std::vector<interp::Value> args;
    std::string harness;
    int output = -1;
    int64_t out_len = 0;
    double scalar = 0.0;
};

} // namespace

extern "C" {

const char* ref_last_error() { return g_last_error.c_str(); }

void* ref_prepare_csr(int64_t rows, const int64_t* row_ptr, const double* val, const double* x,
                      const int64_t* col_ind, int64_t nnz, int64_t ncols) {
    auto* c = new RefCall;
    c->harness = "lilac.spmv_csr";
    c->output = c->mem.alloc_floats("output", std::vector<double>(static_cast<size_t>(rows), 0.0));
    int rp = c->mem.alloc_ints("row_ptr", vec(row_ptr, rows + 1));
    int v = c->mem.alloc_floats("val", vec(val, nnz));
    int xx = c->mem.alloc_floats("x", vec(x, ncols));
    int ci = c->mem.alloc_ints("col_ind", vec(col_ind, nnz));
    c->out_len = rows;
    c->args = {rows, interp::Pointer{c->output, 0}, interp::Pointer{rp, 0}, interp::Pointer{v, 0},
               interp::Pointer{xx, 0}, interp::Pointer{ci, 0}};
    return c;
}

void* ref_prepare_jds(int64_t rows, const int64_t* nzcnt, const int64_t* perm, const double* val,
                      const int64_t* jd_ptr, const double* x, const int64_t* col_ind, int64_t nnz,
                      int64_t njd, int64_t ncols) {
    auto* c = new RefCall;
    c->harness = "lilac.spmv_jds";
    c->output = c->mem.alloc_floats("output", std::vector<double>(static_cast<size_t>(rows), 0.0));
    int nz = c->mem.alloc_ints("nzcnt", vec(nzcnt, rows));
    int pm = c->mem.alloc_ints("perm", vec(perm, rows));
    int v = c->mem.alloc_floats("val", vec(val, nnz));
    int jd = c->mem.alloc_ints("jd_ptr", vec(jd_ptr, njd));
    int xx = c->mem.alloc_floats("x", vec(x, ncols));
    int ci = c->mem.alloc_ints("col_ind", vec(col_ind, nnz));
    c->out_len = rows;
    c->args = {rows,
               interp::Pointer{c->output, 0},
               interp::Pointer{nz, 0},
               interp::Pointer{pm, 0},
               interp::Pointer{v, 0},
               interp::Pointer{jd, 0},
               interp::Pointer{xx, 0},
               interp::Pointer{ci, 0}};
    return c;
}

void* ref_prepare_dot(int64_t length, const double* a, const double* b) {
    auto* c = new RefCall;
    c->harness = "lilac.dotproduct";
    int aa = c->mem.alloc_floats("a", vec(a, length));
    int bb = c->mem.alloc_floats("b", vec(b, length));
    c->args = {length, interp::Pointer{aa, 0}, interp::Pointer{bb, 0}};
    return c;
}

// Runs the reference HarnessFn once. 0 = ok, -1 = lilac::Error (message in
// ref_last_error, e.g. "OutOfBounds ...").
int ref_call(void* h) {
    auto* c = static_cast<RefCall*>(h);
    try {
        const interp::HarnessFn* fn = registry().find(c->harness);
        interp::Value r = (*fn)(c->mem, c->args);
        if (std::holds_alternative<double>(r)) c->scalar = std::get<double>(r);
        return 0;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return -1;
    }
}

void ref_output(void* h, double* out) {
    auto* c = static_cast<RefCall*>(h);
    if (c->output >= 0) {
        const auto& f = c->mem.floats(c->output);
        std::memcpy(out, f.data(), f.size() * sizeof(double));
    } else {
        out[0] = c->scalar;
    }
}

void ref_free(void* h) { delete static_cast<RefCall*>(h); }

// Overwrite the float buffer behind argument `arg` of a prepared call (e.g.
// x of spmv_csr = arg 4, a/b of dotproduct = args 1/2) through the reference
// Memory's own store path (interp.hpp:47-50), so a host CG loop can drive the
// stock HarnessFn with changing vectors. Returns 0, or -1 on a bad argument.
int ref_set_floats(void* h, int arg, const double* src, int64_t n) {
    auto* c = static_cast<RefCall*>(h);
    if (arg < 0 || arg >= static_cast<int>(c->args.size())) return -1;
    const auto* p = std::get_if<interp::Pointer>(&c->args[static_cast<size_t>(arg)]);
    if (!p) return -1;
    if (n > c->mem.size(p->buffer) - p->offset) return -1;
    for (int64_t i = 0; i < n; ++i) c->mem.store_float(interp::Pointer{p->buffer, p->offset + i}, src[i]);
    return 0;
}

double ref_scalar(void* h) { return static_cast<RefCall*>(h)->scalar; }

// infer_interface (what_parse.cpp:356-429) of a LiLAC-What program:
// "name:kind,name:kind,...;scalar_result" into buf.
int ref_infer_interface(const char* what_text, char* buf, int64_t cap) {
    try {
        what::WhatProgram p = what::parse_what(what_text);
        what::HarnessSignature sig = what::infer_interface(p);
        std::string s;
        for (size_t i = 0; i < sig.params.size(); ++i) {
            if (i) s += ",";
            s += sig.params[i].name + ":" + what::param_kind_name(sig.params[i].kind);
        }
        s += sig.scalar_result ? ";scalar" : ";array";
        if (static_cast<int64_t>(s.size()) + 1 > cap) return -1;
        std::memcpy(buf, s.c_str(), s.size() + 1);
        return 0;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return -1;
    }
}

// harnessgen::gen_all (harnessgen.cpp:135-150) over a full .lilac spec; the
// generated TU of harness `name` is written to buf.
int64_t ref_gen_harness(const char* spec_text, const char* name, char* buf, int64_t cap) {
    try {
        how::SpecFile sf = how::parse_spec(spec_text);
        for (const auto& [hname, src] : harnessgen::gen_all(sf.how, sf.whats)) {
            if (hname != name) continue;
            if (static_cast<int64_t>(src.size()) + 1 > cap) return -static_cast<int64_t>(src.size()) - 1;
            std::memcpy(buf, src.c_str(), src.size() + 1);
            return static_cast<int64_t>(src.size());
        }
        g_last_error = "no harness named " + std::string(name);
        return -1;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return -1;
    }
}

uint64_t ref_fnv1a(const void* p, size_t n) { return marshal::fnv1a(p, n); }

} // extern "C"
