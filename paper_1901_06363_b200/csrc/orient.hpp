// Host-built tables shared by every kernel launch (E2).
#pragma once

#include <cstdint>
#include <vector>

namespace gdb200 {

// std::cos / std::sin of a * (pi/180) for the integer angles 0..359, from
// the host libm, exactly as rotate_fragment_into evaluates them
// (reference geometry.hpp:176-178).  Uploaded so the device never calls its
// own (differently rounded) cos/sin.
void trig_tables(std::vector<double>& cos_deg, std::vector<double>& sin_deg);
// The same for any angle: c = std::cos(angle * (pi/180)), s = std::sin(...)
// (geometry.hpp:176-178), for rotate_fragment's arbitrary double angles.
void trig_of(double angle_deg, double& c, double& s);

// Distinct orientations of the rigid Euler grid with step s (divisor of
// 360): (alpha, beta, gamma) = (i, j, k) * s, linear index (i*m + j)*m + k,
// R = Rz(gamma) Ry(beta) Rx(alpha) from the trig tables; matrices that agree
// entry-wise after rounding to 1e-6 are one orientation, represented by the
// lowest linear index.  Output ascending by index; R row-major, 9 per entry.
void rigid_orientations(int step, std::vector<int32_t>& index, std::vector<double>& R);

}  // namespace gdb200
