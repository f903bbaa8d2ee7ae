// Exception vocabulary of the drop-in host API.
//
// Mirrors the reference hierarchy (proj/include/autoplan/errors.hpp:25-108):
// every class derives from PlanError so callers that catch the reference's
// types keep working unchanged. The C-ABI (include/apl.h) never lets these
// escape; it maps each class onto an APL_ERR_* status code instead.
#pragma once

#include <stdexcept>
#include <string>

namespace autoplan {

class PlanError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

#define AUTOPLAN_ERROR(Name)            \
  class Name : public PlanError {       \
   public:                              \
    using PlanError::PlanError;         \
  }

AUTOPLAN_ERROR(SchemaError);           // malformed text / document
AUTOPLAN_ERROR(CycleError);            // graph without a topological order
AUTOPLAN_ERROR(DanglingRefError);      // reference to a missing node
AUTOPLAN_ERROR(ShapeMismatchError);    // shape rule violated during inference
AUTOPLAN_ERROR(UnsupportedKindError);  // no rule for an operation kind
AUTOPLAN_ERROR(ShapeError);            // spec/mesh/tensor combination invalid
AUTOPLAN_ERROR(AxisError);             // mesh axis out of range or repeated
AUTOPLAN_ERROR(RankMismatchError);     // tensor ranks disagree
AUTOPLAN_ERROR(InfeasibleError);       // no path / no solution
AUTOPLAN_ERROR(MissingStrategyError);  // node reached a solver unplanned
AUTOPLAN_ERROR(SeedError);             // differentiable common-node seed
AUTOPLAN_ERROR(IoError);               // file-system failure
AUTOPLAN_ERROR(MissingPathError);      // conversion the planner relied on is absent

#undef AUTOPLAN_ERROR

}  // namespace autoplan
