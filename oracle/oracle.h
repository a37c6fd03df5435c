/*
 * oracle.h -- C interface of the CPU oracle (TEST INFRASTRUCTURE ONLY).
 *
 * Two implementations share this interface:
 *   ref_*  oracle/ref_harness.cpp  -- the reference's own translation units
 *          (proj/src/{color,scene,camera,raster,synth}.cpp, compiled in place
 *          from /root/reference by oracle/Makefile) behind a thin C harness.
 *   orc_*  oracle/sgs_oracle.c     -- a plain-C restatement of the same path,
 *          pinned bit-exactly against ref_* and tests/golden/.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * arm may load these libraries. The product (paper_2501_00342_b200/) never does.
 *
 * Flat scene layout (identical to the product C-ABI, include/sgs.h): per
 * Gaussian, 11 geometry reals [px py pz, qw qx qy qz, lsx lsy lsz, opacity_logit]
 * followed by the colour parameters in the reference's canonical order
 * (proj/include/sgsplat/color.hpp:121-128, proj/include/sgsplat/scene.hpp:40-43).
 */
#ifndef SGS_ORACLE_H
#define SGS_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Colour model kinds, numbered as proj/include/sgsplat/color.hpp:59. */
enum { ORC_SH = 0, ORC_SG1 = 1, ORC_SG3 = 2, ORC_MIXED = 3 };

/* Error codes (same values as the product's SGS_* codes). */
enum { ORC_OK = 0, ORC_INVALID_ARGUMENT = 1, ORC_NUMERIC = 2, ORC_INTERNAL = 6, ORC_IO = 7, ORC_FORMAT = 8 };

/* Pinhole camera, proj/include/sgsplat/camera.hpp:11-23. R is row-major w2c. */
typedef struct {
    double R[9];
    double t[3];
    double fx, fy, cx, cy;
    int32_t width, height;
    double near_plane;
} orc_camera;

/* proj/include/sgsplat/raster.hpp:11-22 (threads only matters for ref_*). */
typedef struct {
    int32_t tile_size;
    int32_t has_override;
    int32_t override_degree;
    int32_t threads;
    double degree_threshold_lo;
    double degree_threshold_hi;
    double early_stop_transmittance;
} orc_config;

/* One projected splat (proj/include/sgsplat/raster.hpp:32-39 + degree). */
typedef struct {
    double mean2d[2];
    double conic[3];
    double depth;
    double color[3];
    double opacity;
    double radius;
    int32_t degree; /* -1 when not a mixed scene */
    int32_t visible;
} orc_splat;

#ifdef __cplusplus
}
#endif

#endif
