// ply_internal.h -- the PLY checkpoint reader shared by sgs_ply_read (host flat
// parameters) and sgs_scene_load_ply (float rows to the device planes).
#pragma once

#include <cstddef>
#include <cstdint>
#include <map>
#include <string>
#include <vector>

#include "sgs.h"

namespace sgs {

// A parsed checkpoint: the header, then (after ply_resolve) its info and, per flat
// parameter of the scene (sgs_scene_desc order: 11 geometry values, then the colour
// parameters), the payload column it comes from.
struct PlyTable {
    std::string path;
    bool binary = false;
    uint64_t count = 0;
    std::vector<std::string> props;             // vertex properties in file order
    std::map<std::string, std::string> comments;  // first token -> rest of the line
    long payload_offset = 0;                    // byte offset of the payload
    // resolved
    sgs_ply_info info{};
    std::vector<int32_t> src;  // flat parameter -> row column
};

// Parses the header (ply.cpp:parse_header). Returns an sgs_status; `err` receives
// the reference's message.
int ply_parse_header(const char* path, PlyTable& t, std::string& err);

// Reads the vertex payload (binary or ASCII) into rows[count * props.size()].
int ply_read_rows(const PlyTable& t, float* rows, std::string& err);

// The payload checks of ply_read_rows without keeping the values (header-only
// queries report errors in the reference's order).
int ply_check_payload(const PlyTable& t, std::string& err);

// What follows the payload in load_ply (ply.cpp:295-306): layout detection, the
// column map, sg_model / sg_axes / sg_background, then the .meta sidecar.
int ply_resolve(PlyTable& t, std::string& err);

// Flat parameters (doubles) from the rows.
void ply_rows_to_flat(const PlyTable& t, const float* rows, double* params);

}  // namespace sgs
