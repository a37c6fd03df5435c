// dropin_bench.cpp -- wall time of the reference's own C++ render call,
// sgsplat::render(scene, camera, cfg) (proj/include/sgsplat/raster.hpp:56), served by
// libsgsplat_b200.so, under the reference's `sgsplat bench` protocol
// (proj/tools/main.cpp:232-243): 3 warm-up renders, then the median of K.
// Each call is the whole drop-in path: the caller's AoS Scene packed and uploaded,
// the frame rendered, the double Image (RGB + transmittance) returned in host memory.
//
//   build/dropin_bench [gaussians] [repeats]     (config C: mixed SG + SH1, 1080p)
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "sgsplat/raster.hpp"
#include "sgsplat/synth.hpp"

int main(int argc, char** argv) {
    const std::size_t n = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 3000000;
    const int repeat = argc > 2 ? std::atoi(argv[2]) : 5;
    sgsplat::SynthOptions o;
    o.kind = sgsplat::ColorModelKind::MixedSHSG;
    o.sh_degree = 2;
    o.log_scale_min = -5.5;
    o.log_scale_max = -4.0;
    const sgsplat::Scene scene = sgsplat::make_synthetic_scene(n, 20260003, o);
    const sgsplat::Camera cam = sgsplat::make_orbit_cameras(256, 1920, 1080, 4.0, 1296.0, 0.35)[0];
    sgsplat::RenderConfig cfg;
    cfg.sh_degree_override = 1;
    double checksum = 0.0;
    for (int i = 0; i < 3; ++i) checksum += sgsplat::render(scene, cam, cfg).image.data[0];
    std::vector<double> ms;
    for (int i = 0; i < repeat; ++i) {
        const auto t0 = std::chrono::steady_clock::now();
        const sgsplat::RenderResult r = sgsplat::render(scene, cam, cfg);
        const auto t1 = std::chrono::steady_clock::now();
        checksum += r.image.data[0];
        ms.push_back(std::chrono::duration<double, std::milli>(t1 - t0).count());
    }
    std::sort(ms.begin(), ms.end());
    double median = ms[ms.size() / 2];
    if (ms.size() % 2 == 0) median = 0.5 * (median + ms[ms.size() / 2 - 1]);
    std::printf("{\"fps\": %.4f, \"median_ms\": %.3f, \"min_ms\": %.3f, \"repeats\": %d, \"gaussians\": %zu, "
                "\"checksum\": %.6f}\n",
                1000.0 / median, median, ms.front(), repeat, n, checksum);
    return 0;
}
