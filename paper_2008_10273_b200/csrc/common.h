// Shared host-side helpers: typed errors that map onto the reference's
// exception classes (see include/hivc_b200.h) and CUDA error checks.
#pragma once

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <utility>
#include <vector>
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

// Diagnostics and tuning overrides, all behind ONE environment variable:
//   HIVC_DEBUG="key=value,key=value"   e.g. timeline=/tmp/tl.csv,workers=4,brox_graph=0
// Keys: timeline, cg_trace, cg_trace_cluster, batch_trace (diagnostic dumps);
// workers, min_batch, tree_threads, tree_threads_small, enc_threads (host
// threading); brox_graph, brox_jc_max, brox_j2_min (Brox launch paths, for the
// bit-identity tests); p_repeat=N (each P-frame kernel launched N times: the
// step's sensitivity to that kernel).  Absent keys return nullptr; no key
// changes a result.
inline const char* debug_opt(const char* key) {
    static const std::vector<std::pair<std::string, std::string>> opts = [] {
        std::vector<std::pair<std::string, std::string>> v;
        const char* e = std::getenv("HIVC_DEBUG");
        std::string s = e ? e : "";
        size_t i = 0;
        while (i < s.size()) {
            size_t j = s.find(',', i);
            if (j == std::string::npos) j = s.size();
            const std::string kv = s.substr(i, j - i);
            const size_t eq = kv.find('=');
            if (!kv.empty()) v.push_back(eq == std::string::npos ? std::make_pair(kv, std::string("1"))
                                                                 : std::make_pair(kv.substr(0, eq), kv.substr(eq + 1)));
            i = j + 1;
        }
        return v;
    }();
    for (const auto& kv : opts)
        if (kv.first == key) return kv.second.c_str();
    return nullptr;
}

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
