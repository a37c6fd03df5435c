// Drop-in declarations for the PLY checkpoint reader (reference: proj/include/sgsplat/ply.hpp).
// load_ply is served by libsgsplat_b200.so through the C-ABI (sgs_ply_read); writing
// checkpoints (save_ply) is outside the B200 build's scope.
#pragma once

#include "sgsplat/scene.hpp"

#include <string>

namespace sgsplat {

// The two checkpoint layouts (ply.hpp:9-22).
enum class PlyLayout { Reference3DGS, SGExtended };

// Per-Gaussian stored floats for a layout/model combination (59; 29, or 53 for mixed).
int ply_floats_per_gaussian(PlyLayout layout, ColorModelKind kind);

// Loads a binary little-endian or ASCII PLY (layout detected from the property
// names, header comments and an optional "<path>.meta" sidecar). Throws IoError,
// FormatError or InvalidArgument exactly as the reference does.
Scene load_ply(const std::string& path);

PlyLayout detect_layout(const Scene& scene);

}  // namespace sgsplat
