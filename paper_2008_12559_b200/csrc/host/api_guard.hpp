// api_guard.hpp -- exception-to-status translation used by every extern "C" entry point.
#pragma once

#include <new>
#include <string>

#include "internal.hpp"

namespace pft::detail {
const char* last_error_cstr();
}

#define PFT_API_BEGIN \
    try {             \
        ::pft::detail::set_last_error("");
#define PFT_API_END                                         \
    }                                                       \
    catch (const ::pft::detail::Error& e) {                 \
        ::pft::detail::set_last_error(e.what());            \
        return e.status;                                    \
    }                                                       \
    catch (const std::bad_alloc&) {                         \
        ::pft::detail::set_last_error("out of host memory");\
        return PFT_ERR_INTERNAL;                            \
    }                                                       \
    catch (const std::exception& e) {                       \
        ::pft::detail::set_last_error(e.what());            \
        return PFT_ERR_INTERNAL;                            \
    }                                                       \
    return PFT_OK;

#define PFT_REQUIRE(cond, msg)                                                       \
    do {                                                                             \
        if (!(cond)) ::pft::detail::fail(PFT_ERR_INVALID_ARGUMENT, std::string(msg)); \
    } while (0)
