// Status/exception plumbing for the C ABI: typed C++ exceptions inside the
// library map onto carma_status codes at the boundary (the reference's
// CarmaError family, errors.hpp:12-57, collapsed to the codes callers act on).
#pragma once

#include <stdexcept>
#include <string>

#include "../../../include/carma_gpu.h"

namespace carma_b200 {

struct CarmaFailure : std::runtime_error {
    carma_status code;
    CarmaFailure(carma_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};
struct InvalidArg : CarmaFailure {
    explicit InvalidArg(const std::string& m) : CarmaFailure(CARMA_ERR_INVALID, m) {}
};
struct CudaFailure : CarmaFailure {
    explicit CudaFailure(const std::string& m) : CarmaFailure(CARMA_ERR_CUDA, m) {}
};
struct Unsupported : CarmaFailure {
    explicit Unsupported(const std::string& m) : CarmaFailure(CARMA_ERR_UNSUPPORTED, m) {}
};

void set_last_error(const std::string& msg);

template <typename F>
carma_status guarded(F&& f) {
    try {
        f();
        set_last_error("");
        return CARMA_OK;
    } catch (const CarmaFailure& e) {
        set_last_error(e.what());
        return e.code;
    } catch (const std::invalid_argument& e) {
        set_last_error(e.what());
        return CARMA_ERR_INVALID;
    } catch (const std::exception& e) {
        set_last_error(e.what());
        return CARMA_ERR_INVALID;
    }
}

}  // namespace carma_b200
