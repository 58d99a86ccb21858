#pragma once
// synkpar error taxonomy (drop-in for the reference's include/synkpar/errors.hpp).
// Every class the reference throws exists here with the same name and base, so
// catch sites and the Python mapping are unchanged. DeviceError is new: CUDA
// failures of the B200 backend that are not a rank-task failure.

#include <cstddef>
#include <stdexcept>
#include <string>

namespace synkpar {

struct Error : std::runtime_error {
    using std::runtime_error::runtime_error;
};

#define SYNKPAR_ERROR_CLASS(Name)        \
    struct Name : Error {                \
        using Error::Error;              \
    }

SYNKPAR_ERROR_CLASS(BoundsError);           // index outside the addressed extent
SYNKPAR_ERROR_CLASS(ShapeError);            // shape / rank / trailing-dim mismatch
SYNKPAR_ERROR_CLASS(DTypeError);            // mixed or unsupported element types
SYNKPAR_ERROR_CLASS(ArgumentError);         // invalid argument value
SYNKPAR_ERROR_CLASS(CapacityError);         // view larger than the allocation
SYNKPAR_ERROR_CLASS(UseAfterFreeError);     // freed shared input array
SYNKPAR_ERROR_CLASS(LifecycleError);        // wrong pool/function state
SYNKPAR_ERROR_CLASS(SlicingConflictError);  // Overwrite update with num_slices > 1
SYNKPAR_ERROR_CLASS(CoherenceError);        // replicas expected identical are not
SYNKPAR_ERROR_CLASS(NumericError);          // non-finite values (debug checks)
SYNKPAR_ERROR_CLASS(IoError);               // file / stream failure
SYNKPAR_ERROR_CLASS(DeviceError);           // CUDA backend failure outside a phase

#undef SYNKPAR_ERROR_CLASS

// Raised by the master when a rank's task failed inside a phase; the pool is
// shut down (fail-stop) before this propagates. The lowest failing rank wins.
class PhaseError : public Error {
public:
    PhaseError(std::size_t rank, const std::string& what)
        : Error("phase failed on rank " + std::to_string(rank) + ": " + what), rank_(rank) {}
    std::size_t rank() const noexcept { return rank_; }

private:
    std::size_t rank_;
};

} // namespace synkpar
