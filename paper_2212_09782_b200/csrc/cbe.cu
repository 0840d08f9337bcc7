// K5 (CBE: Gram + Hermitian eigensolver + kept selection) and K9 (Schmidt
// values).  Filled in below the QR path.
#include "gate.cuh"

namespace qt {

CbeResult gate_cbe(Engine&, const Dims&, const double2*, const double2*, const double2*, const double2*,
                   const qt_policy&, const std::function<GateBuffers(long long)>&) {
  throw Error(Err::internal, "qr_cbe not built yet");
}

void eigh_device(Engine&, const double2*, long long, double*, double2*) {
  throw Error(Err::internal, "eigh not built yet");
}

void singular_values_device(Engine&, const double2*, long long, long long, double*) {
  throw Error(Err::internal, "svd not built yet");
}

}  // namespace qt
