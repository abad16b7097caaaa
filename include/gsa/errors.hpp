// gsa/errors.hpp — exception classes of the GSA operator API (drop-in for the
// reference's proj/include/gsa/errors.hpp:8-58). The device library reports a
// gsa_status; gsa::device::raise() maps each status onto these classes.
#pragma once

#include <stdexcept>
#include <string>

namespace gsa {

struct GsaError : std::runtime_error {
    explicit GsaError(const std::string& what) : std::runtime_error(what) {}
};

#define GSA_DEFINE_ERROR(Name) \
    struct Name : GsaError {   \
        using GsaError::GsaError; \
    }

GSA_DEFINE_ERROR(ShapeMismatch);            // tensor extents disagree
GSA_DEFINE_ERROR(DivisibilityError);        // grid not tiled by the window side
GSA_DEFINE_ERROR(ZeroSizeError);            // empty layout dimension
GSA_DEFINE_ERROR(IndexOutOfRange);          // token / window / row index outside its range
GSA_DEFINE_ERROR(NonFiniteInput);           // NaN / Inf where finite values are required
GSA_DEFINE_ERROR(InvalidTiling);            // tile sides not powers of two in [8, 256]
GSA_DEFINE_ERROR(InvalidStride);            // hybrid reference-frame stride < 1
GSA_DEFINE_ERROR(EmptySelection);           // a selection-plan row with no windows
GSA_DEFINE_ERROR(ContextMismatch);          // saved context does not match the call
GSA_DEFINE_ERROR(ConfigParseError);         // malformed workload configuration
GSA_DEFINE_ERROR(DegenerateInput);          // input the algorithm cannot handle
GSA_DEFINE_ERROR(NonDeterministicForward);  // repeated forward calls disagree
// device-side additions (no reference counterpart)
GSA_DEFINE_ERROR(Unsupported);              // shape outside what the sm_100a kernels implement
GSA_DEFINE_ERROR(CudaError);                // CUDA runtime / launch failure

#undef GSA_DEFINE_ERROR

}  // namespace gsa
