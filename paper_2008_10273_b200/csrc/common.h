// Shared host-side helpers: typed errors that map onto the reference's
// exception classes (see include/hivc_b200.h) and CUDA error checks.
#pragma once

#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>

#include "../../include/hivc_b200.h"

namespace hivc {

struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(int code, const std::string& msg) { throw Error(code, msg); }

void set_last_error(const std::string& msg);

// Run `fn`, translating exceptions into a status code + thread-local message.
template <class F>
int guarded(F&& fn) {
    try {
        fn();
        return HIVC_OK;
    } catch (const Error& e) {
        set_last_error(e.what());
        return e.code;
    } catch (const std::bad_alloc&) {
        set_last_error("out of memory");
        return HIVC_E_NOMEM;
    } catch (const std::exception& e) {
        set_last_error(e.what());
        return HIVC_E_ARGUMENT;
    }
}

}  // namespace hivc
