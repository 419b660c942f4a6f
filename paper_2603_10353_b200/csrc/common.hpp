// Shared host-side plumbing of libshplb: typed errors that mirror the
// reference's exception classes, and their translation to shplb_status at the
// C-ABI boundary (include/shplb.h).
#pragma once

#include <stdexcept>
#include <string>

#include "shplb.h"

namespace shplb {

// Raised where the reference raises std::invalid_argument / runtime_error /
// logic_error; the ABI maps each to its status code.
struct InvalidArgument : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};
struct RuntimeError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct NotSupported : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct NcclError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

void set_last_error(const std::string& msg);
void clear_last_error();

// Runs f, converting any exception to a status and recording its message.
template <typename F>
int guarded(F&& f) {
    try {
        clear_last_error();
        f();
        return SHPLB_OK;
    } catch (const InvalidArgument& e) {
        set_last_error(e.what());
        return SHPLB_INVALID_ARGUMENT;
    } catch (const NotSupported& e) {
        set_last_error(e.what());
        return SHPLB_NOT_SUPPORTED;
    } catch (const CudaError& e) {
        set_last_error(e.what());
        return SHPLB_CUDA_ERROR;
    } catch (const NcclError& e) {
        set_last_error(e.what());
        return SHPLB_NCCL_ERROR;
    } catch (const std::invalid_argument& e) {
        set_last_error(e.what());
        return SHPLB_INVALID_ARGUMENT;
    } catch (const std::logic_error& e) {
        set_last_error(e.what());
        return SHPLB_LOGIC_ERROR;
    } catch (const std::exception& e) {
        set_last_error(e.what());
        return SHPLB_RUNTIME_ERROR;
    }
}

inline void require(bool ok, const std::string& msg) {
    if (!ok) throw InvalidArgument(msg);
}

}  // namespace shplb
