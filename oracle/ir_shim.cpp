// ir_shim.cpp — C ABI over the reference's IR pipeline (parse → detect →
// rewrite → interp::run) with a choice of harness registry, for the tests of
// the IR-pipeline adapter.
//
// TEST INFRASTRUCTURE ONLY. Built by oracle/Makefile (`make -C oracle ir`)
// from the reference's src/*.cpp compiled where they lie, this file, and the
// product adapter paper_2001_07938_b200/adapters/interp_b200.cpp, linked to
// liblilac_b200.so. Backends for a run: 0 = no registry, 1 = the reference's
// register_reference_harnesses (interp.cpp:330-389), 2 = the B200 adapter.

#include "../paper_2001_07938_b200/adapters/interp_b200.hpp"

#include "lilac/how.hpp"
#include "lilac/interp.hpp"
#include "lilac/ir.hpp"
#include "lilac/rewrite.hpp"
#include "lilac/what.hpp"

#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <vector>

using namespace lilac;

namespace {

std::string g_err;

struct Session {
    ir::Module original, rewritten;
    bool has_rewritten = false;
    interp::Memory base;  // the buffers every run starts from
    interp::Memory last;  // the buffers after the last run
};

std::unique_ptr<interp::HarnessRegistry> make_registry(int backend, const char* spec_text) {
    auto reg = std::make_unique<interp::HarnessRegistry>();
    if (backend == 0) return reg;
    how::SpecFile sf = how::parse_spec(spec_text);
    if (backend == 1)
        interp::register_reference_harnesses(*reg, sf.whats);
    else
        lilac_b200::register_b200_harnesses(*reg, sf.whats);
    return reg;
}

std::vector<interp::Value> make_args(const int* kinds, const int64_t* vals, int nargs) {
    std::vector<interp::Value> args;
    for (int i = 0; i < nargs; ++i) {
        if (kinds[i] == 0)
            args.emplace_back(static_cast<std::int64_t>(vals[i]));
        else
            args.emplace_back(interp::Pointer{static_cast<int>(vals[i]), 0});
    }
    return args;
}

template <typename F>
int guarded(F&& f) {
    try {
        g_err.clear();
        return f();
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

int ret_value(const interp::Value& v, double* ret) {
    if (ret) {
        if (const auto* d = std::get_if<double>(&v))
            *ret = *d;
        else if (const auto* i = std::get_if<std::int64_t>(&v))
            *ret = static_cast<double>(*i);
    }
    return 0;
}

}  // namespace

extern "C" {

const char* ir_error() { return g_err.c_str(); }

void* ir_open(const char* lir_text) {
    try {
        g_err.clear();
        auto s = std::make_unique<Session>();
        s->original = ir::parse_module(lir_text);
        Diagnostics d = ir::verify(s->original);
        if (!d.empty()) throw std::runtime_error("module failed verification");
        return s.release();
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

void ir_close(void* h) { delete static_cast<Session*>(h); }

// rewrite_all with one What program (the CLI's `rewrite --what`, lilac_main.cpp:279-287)
int ir_rewrite(void* h, const char* spec_text, const char* what_name) {
    return guarded([&] {
        auto* s = static_cast<Session*>(h);
        how::SpecFile sf = how::parse_spec(spec_text);
        const what::WhatProgram* p = sf.find_what(what_name);
        if (!p) throw std::runtime_error(std::string("no COMPUTATION ") + what_name);
        rewrite::RewriteAllResult rr = rewrite::rewrite_all(s->original, *p, std::string("lilac.") + what_name);
        s->rewritten = std::move(rr.module);
        s->has_rewritten = true;
        return rr.applied;
    });
}

int64_t ir_text(void* h, int rewritten, char* buf, int64_t cap) {
    auto* s = static_cast<Session*>(h);
    const std::string t = ir::print_module(rewritten ? s->rewritten : s->original);
    if (buf && cap > 0) {
        const std::size_t n = std::min<std::size_t>(t.size(), static_cast<std::size_t>(cap - 1));
        std::memcpy(buf, t.data(), n);
        buf[n] = 0;
    }
    return static_cast<int64_t>(t.size());
}

int ir_add_i64(void* h, const char* label, const int64_t* p, int64_t n) {
    return guarded([&] {
        return static_cast<Session*>(h)->base.alloc_ints(label, std::vector<std::int64_t>(p, p + n));
    });
}

int ir_add_f64(void* h, const char* label, const double* p, int64_t n) {
    return guarded([&] {
        return static_cast<Session*>(h)->base.alloc_floats(label, std::vector<double>(p, p + n));
    });
}

// Runs @entry of the original (rewritten = 0) or rewritten module on a copy
// of the base buffers. kinds[i]: 0 = i64 scalar vals[i], 1 = pointer to
// buffer vals[i] at offset 0.
int ir_run(void* h, int rewritten, int backend, const char* spec_text, const char* entry, const int* kinds,
           const int64_t* vals, int nargs, double* ret) {
    return guarded([&] {
        auto* s = static_cast<Session*>(h);
        if (rewritten && !s->has_rewritten) throw std::runtime_error("ir_rewrite first");
        auto reg = make_registry(backend, spec_text);
        s->last = s->base;
        interp::Value v = interp::run(rewritten ? s->rewritten : s->original, entry, make_args(kinds, vals, nargs),
                                      s->last, *reg);
        return ret_value(v, ret);
    });
}

// Calls the registered "lilac.<what>" HarnessFn directly on a copy of the
// base buffers (the harness tests of test_interp.cpp:188-300).
int ir_call_harness(void* h, int backend, const char* spec_text, const char* name, const int* kinds,
                    const int64_t* vals, int nargs, double* ret) {
    return guarded([&] {
        auto* s = static_cast<Session*>(h);
        auto reg = make_registry(backend, spec_text);
        const interp::HarnessFn* fn = reg->find(name);
        if (!fn) throw std::runtime_error(std::string("UnregisteredHarness: ") + name);
        s->last = s->base;
        return ret_value((*fn)(s->last, make_args(kinds, vals, nargs)), ret);
    });
}

int ir_read_f64(void* h, int buffer, double* out, int64_t n) {
    return guarded([&] {
        const auto& v = static_cast<Session*>(h)->last.floats(buffer);
        if (static_cast<int64_t>(v.size()) < n) throw std::runtime_error("buffer shorter than requested");
        std::memcpy(out, v.data(), sizeof(double) * static_cast<std::size_t>(n));
        return 0;
    });
}

uint64_t ir_write_version(void* h, int buffer) { return static_cast<Session*>(h)->last.write_version(buffer); }

}  // extern "C"
