// host_ply.cpp -- PLY checkpoint reader (sgsplat::load_ply, proj/src/ply.cpp:52-306).
//
// Same acceptance rules, error classes, messages and order of checks as the
// reference: header (parse_header, ply.cpp:52-103), payload (read_payload,
// :105-120), layout detection by property names (:300-305), the column map
// (map_columns, :146-169: duplicate / unknown / missing properties), the SG header
// comments (load_extended, :207-232) and the ".meta" sidecar (apply_sidecar,
// :129-144). Instead of building Scene objects it produces, for every flat scene
// parameter (sgs_scene_desc order), the payload column it comes from; the host path
// gathers doubles through it and the device path (capi.cu) gathers floats on the
// GPU into the scene planes.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <sstream>

#include "ply_internal.h"

namespace sgs {
namespace {

std::vector<std::string> fields_reference() {
    std::vector<std::string> f = {"x", "y", "z", "f_dc_0", "f_dc_1", "f_dc_2"};
    for (int k = 0; k < 45; ++k) f.push_back("f_rest_" + std::to_string(k));
    f.push_back("opacity");
    for (int k = 0; k < 3; ++k) f.push_back("scale_" + std::to_string(k));
    for (int k = 0; k < 4; ++k) f.push_back("rot_" + std::to_string(k));
    return f;
}

std::vector<std::string> fields_extended(bool sh2) {
    std::vector<std::string> f = {"x", "y", "z", "f_dc_0", "f_dc_1", "f_dc_2"};
    for (int i = 0; i < 3; ++i)
        for (int c = 0; c < 3; ++c) f.push_back("sg_alpha_" + std::to_string(i) + "_" + std::to_string(c));
    for (int i = 0; i < 3; ++i) f.push_back("sg_lambda_" + std::to_string(i));
    for (int k = 0; k < 3; ++k) f.push_back("sg_mu_" + std::to_string(k));
    if (sh2)
        for (int k = 0; k < 24; ++k) f.push_back("sh2_" + std::to_string(k));
    f.push_back("opacity");
    for (int k = 0; k < 3; ++k) f.push_back("scale_" + std::to_string(k));
    for (int k = 0; k < 4; ++k) f.push_back("rot_" + std::to_string(k));
    return f;
}

bool read_doubles(const std::string& text, double* out, int count) {
    std::istringstream ss(text);
    for (int i = 0; i < count; ++i)
        if (!(ss >> out[i])) return false;
    return true;
}

void strip_cr(std::string& line) {
    if (!line.empty() && line.back() == '\r') line.pop_back();
}

// canonical field index -> payload column (map_columns)
int map_fields(const PlyTable& t, const std::vector<std::string>& canonical, const std::vector<std::string>& ignored,
               std::vector<int>& col, std::string& err) {
    std::map<std::string, int> at;
    for (size_t i = 0; i < t.props.size(); ++i) {
        if (at.count(t.props[i])) {
            err = "duplicate PLY property: " + t.props[i];
            return SGS_ERR_FORMAT;
        }
        at[t.props[i]] = static_cast<int>(i);
    }
    for (const auto& name : t.props) {
        bool known = false;
        for (const auto& c : canonical) known = known || c == name;
        for (const auto& c : ignored) known = known || c == name;
        if (!known) {
            err = "unknown PLY property: " + name;
            return SGS_ERR_FORMAT;
        }
    }
    col.clear();
    for (const auto& name : canonical) {
        auto it = at.find(name);
        if (it == at.end()) {
            err = "missing PLY property: " + name;
            return SGS_ERR_FORMAT;
        }
        col.push_back(it->second);
    }
    return SGS_OK;
}

// Scene::set_shared_axes -> validate_ortho_axes (color.cpp:36-44, tol 1e-6):
// max |A A^T - I| with the Eigen-subset's left-to-right sums.
int check_ortho(const double* a, std::string& err) {
    double worst = 0.0;
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) {
            const double g = (a[3 * r] * a[3 * c] + a[3 * r + 1] * a[3 * c + 1]) + a[3 * r + 2] * a[3 * c + 2];
            const double d = std::fabs(g - (r == c ? 1.0 : 0.0));
            if (d > worst) worst = d;
        }
    if (worst > 1e-6) {
        std::ostringstream msg;
        msg << "axis triple is not orthonormal: |A A^T - I|_max = " << worst;
        err = msg.str();
        return SGS_ERR_INVALID_ARGUMENT;
    }
    return SGS_OK;
}

void apply_meta_sidecar(const std::string& path, sgs_ply_info& info) {
    std::ifstream meta(path + ".meta");
    if (!meta) return;
    std::string line;
    while (std::getline(meta, line)) {
        const auto eq = line.find('=');
        if (eq == std::string::npos) continue;
        const std::string key = line.substr(0, eq), value = line.substr(eq + 1);
        double v[9];
        if (key == "axes" && read_doubles(value, v, 9)) {
            for (int k = 0; k < 9; ++k) info.shared_axes[k] = v[k];
        } else if (key == "background" && read_doubles(value, v, 3)) {
            for (int k = 0; k < 3; ++k) info.background[k] = v[k];
        }
    }
}

}  // namespace

int ply_parse_header(const char* path, PlyTable& t, std::string& err) {
    t = PlyTable{};
    t.path = path;
    std::ifstream in(path, std::ios::binary);
    if (!in) {
        err = std::string("cannot open: ") + path;
        return SGS_ERR_IO;
    }
    std::string line;
    if (!std::getline(in, line)) {
        err = std::string("empty file: ") + path;
        return SGS_ERR_IO;
    }
    strip_cr(line);
    if (line != "ply") {
        err = std::string("not a PLY file: ") + path;
        return SGS_ERR_FORMAT;
    }
    bool saw_format = false, in_vertex = false, done = false;
    while (std::getline(in, line)) {
        strip_cr(line);
        std::istringstream ls(line);
        std::string tok;
        ls >> tok;
        if (tok == "format") {
            std::string kind, version;
            ls >> kind >> version;
            if (kind == "binary_little_endian") {
                t.binary = true;
            } else if (kind == "ascii") {
                t.binary = false;
            } else {
                err = "unsupported PLY format '" + kind + "' (little-endian binary or ascii only)";
                return SGS_ERR_FORMAT;
            }
            saw_format = true;
        } else if (tok == "comment") {
            std::string key, rest;
            ls >> key;
            std::getline(ls, rest);
            if (!rest.empty() && rest.front() == ' ') rest.erase(0, 1);
            t.comments[key] = rest;
        } else if (tok == "element") {
            std::string name;
            size_t count = 0;
            ls >> name >> count;
            if (name != "vertex") {
                err = "unsupported PLY element '" + name + "'";
                return SGS_ERR_FORMAT;
            }
            if (in_vertex) {
                err = "duplicate vertex element";
                return SGS_ERR_FORMAT;
            }
            t.count = count;
            in_vertex = true;
        } else if (tok == "property") {
            std::string type, name;
            ls >> type >> name;
            if (!in_vertex) {
                err = "property outside vertex element";
                return SGS_ERR_FORMAT;
            }
            if (type != "float" && type != "float32") {
                err = "unsupported property type '" + type + "' for " + name;
                return SGS_ERR_FORMAT;
            }
            t.props.push_back(name);
        } else if (tok == "end_header") {
            done = true;
            break;
        } else if (tok == "obj_info" || tok.empty()) {
            continue;
        } else {
            err = "unrecognized PLY header line: " + line;
            return SGS_ERR_FORMAT;
        }
    }
    if (!done || !saw_format) {
        err = std::string("truncated PLY header: ") + path;
        return SGS_ERR_FORMAT;
    }
    t.payload_offset = static_cast<long>(in.tellg());
    t.info.count = t.count;
    t.info.binary = t.binary ? 1 : 0;
    // The vertex count is untrusted: before anything is sized from it, the payload it
    // implies (count * properties floats; checked multiplication) must fit in what the
    // file still holds -- 4 bytes per value in binary, at least 2 ("0 ") in ASCII. The
    // reference fails here too: resize(vertex_count) throws or the read comes up short.
    const uint64_t np = t.props.size();
    const uint64_t per_value = t.binary ? 4 : 2;
    in.seekg(0, std::ios::end);
    const long long end = static_cast<long long>(in.tellg());
    const uint64_t avail = end > t.payload_offset ? static_cast<uint64_t>(end - t.payload_offset) : 0;
    if (np && t.count > (avail + 1) / per_value / np) {
        err = std::string(t.binary ? "truncated PLY payload: " : "truncated ASCII PLY payload: ") + path;
        return SGS_ERR_IO;
    }
    if (t.count > 0xFFFFFFFFULL) {
        err = "more than 2^32 Gaussians";
        return SGS_ERR_INVALID_ARGUMENT;
    }
    return SGS_OK;
}

int ply_read_rows(const PlyTable& t, float* rows, std::string& err) {
    const size_t n = static_cast<size_t>(t.count) * t.props.size();
    std::ifstream in(t.path, std::ios::binary);
    if (!in) {
        err = "cannot open: " + t.path;
        return SGS_ERR_IO;
    }
    in.seekg(t.payload_offset);
    if (t.binary) {
        in.read(reinterpret_cast<char*>(rows), static_cast<std::streamsize>(n * sizeof(float)));
        if (static_cast<size_t>(in.gcount()) != n * sizeof(float)) {
            err = "truncated PLY payload: " + t.path;
            return SGS_ERR_IO;
        }
    } else {
        // std::istream >> double (the reference), then narrowed to float
        for (size_t i = 0; i < n; ++i) {
            double v;
            if (!(in >> v)) {
                err = "truncated ASCII PLY payload: " + t.path;
                return SGS_ERR_IO;
            }
            rows[i] = static_cast<float>(v);
        }
    }
    return SGS_OK;
}

int ply_check_payload(const PlyTable& t, std::string& err) {
    const size_t n = static_cast<size_t>(t.count) * t.props.size();
    std::ifstream in(t.path, std::ios::binary);
    if (!in) {
        err = "cannot open: " + t.path;
        return SGS_ERR_IO;
    }
    if (t.binary) {
        in.seekg(0, std::ios::end);
        const long long avail = static_cast<long long>(in.tellg()) - t.payload_offset;
        if (avail < static_cast<long long>(n * sizeof(float))) {
            err = "truncated PLY payload: " + t.path;
            return SGS_ERR_IO;
        }
        return SGS_OK;
    }
    in.seekg(t.payload_offset);
    for (size_t i = 0; i < n; ++i) {
        double v;
        if (!(in >> v)) {
            err = "truncated ASCII PLY payload: " + t.path;
            return SGS_ERR_IO;
        }
    }
    return SGS_OK;
}

int ply_resolve(PlyTable& t, std::string& err) {
    sgs_ply_info& info = t.info;
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) info.shared_axes[3 * r + c] = r == c ? 1.0 : 0.0;  // Mat3::Identity
    for (int k = 0; k < 3; ++k) info.background[k] = 0.0;
    bool has_rest = false, has_sg = false;
    for (const auto& p : t.props) {
        has_rest = has_rest || p == "f_rest_0";
        has_sg = has_sg || p == "sg_alpha_0_0";
    }
    std::vector<int> col;
    t.src.clear();
    auto put = [&](int canonical) { t.src.push_back(col[static_cast<size_t>(canonical)]); };
    if (has_rest && !has_sg) {
        // load_reference (ply.cpp:181-205): degree-3 SH, f_rest channel-major
        info.layout = SGS_PLY_REFERENCE3DGS;
        info.kind = SGS_SH;
        info.sh_degree = 3;
        int st = map_fields(t, fields_reference(), {"nx", "ny", "nz"}, col, err);
        if (st != SGS_OK) return st;
        for (int k = 0; k < 3; ++k) put(k);        // position
        for (int k = 0; k < 4; ++k) put(55 + k);   // rotation (wxyz)
        for (int k = 0; k < 3; ++k) put(52 + k);   // log scale
        put(51);                                   // opacity logit
        for (int c = 0; c < 3; ++c) put(3 + c);    // SH coefficient 0
        for (int idx = 1; idx < 16; ++idx)
            for (int ch = 0; ch < 3; ++ch) put(6 + ch * 15 + (idx - 1));
    } else if (has_sg && !has_rest) {
        // load_extended (ply.cpp:207-286)
        info.layout = SGS_PLY_SGEXTENDED;
        auto m = t.comments.find("sg_model");
        if (m == t.comments.end()) {
            err = "SG-extended PLY is missing the 'comment sg_model' header line";
            return SGS_ERR_FORMAT;
        }
        std::string name = m->second;
        while (!name.empty() && (name.back() == ' ' || name.back() == '\t')) name.pop_back();
        // color_model_kind_from_string (color.cpp:91-97)
        if (name == "sh") {
            err = "sg_model comment names a non-SG model";
            return SGS_ERR_FORMAT;
        } else if (name == "sg1") {
            info.kind = SGS_SG1;
        } else if (name == "sg3") {
            info.kind = SGS_SG3;
        } else if (name == "mixed") {
            info.kind = SGS_MIXED;
        } else {
            err = "unknown color model kind: " + name;
            return SGS_ERR_INVALID_ARGUMENT;
        }
        const bool sh2 = info.kind == SGS_MIXED;
        info.sh_degree = sh2 ? 2 : 0;
        int st = map_fields(t, fields_extended(sh2), {}, col, err);
        if (st != SGS_OK) return st;
        if (auto it = t.comments.find("sg_axes"); it != t.comments.end()) {
            double v[9];
            if (!read_doubles(it->second, v, 9)) {
                err = "bad sg_axes comment";
                return SGS_ERR_FORMAT;
            }
            st = check_ortho(v, err);
            if (st != SGS_OK) return st;
            for (int k = 0; k < 9; ++k) info.shared_axes[k] = v[k];
        }
        if (auto it = t.comments.find("sg_background"); it != t.comments.end()) {
            double v[3];
            if (!read_doubles(it->second, v, 3)) {
                err = "bad sg_background comment";
                return SGS_ERR_FORMAT;
            }
            for (int k = 0; k < 3; ++k) info.background[k] = v[k];
        }
        const int alpha = 6, lambda = 15, mu = 18, sh2base = 21, tail = sh2 ? 45 : 21;
        for (int k = 0; k < 3; ++k) put(k);             // position
        for (int k = 0; k < 4; ++k) put(tail + 4 + k);  // rotation
        for (int k = 0; k < 3; ++k) put(tail + 1 + k);  // log scale
        put(tail);                                      // opacity logit
        if (info.kind == SGS_SG1) {
            // [diffuse rgb, alpha rgb, log_lambda, mu xyz] (color.hpp:128)
            for (int c = 0; c < 3; ++c) put(3 + c);
            for (int c = 0; c < 3; ++c) put(alpha + c);
            put(lambda);
            for (int c = 0; c < 3; ++c) put(mu + c);
        } else {
            if (info.kind == SGS_SG3) {
                for (int c = 0; c < 3; ++c) put(3 + c);  // diffuse
            } else {
                // SH degree 2: coefficient 0 from f_dc, 1..8 from sh2 (channel-major)
                for (int c = 0; c < 3; ++c) put(3 + c);
                for (int idx = 1; idx < 9; ++idx)
                    for (int ch = 0; ch < 3; ++ch) put(sh2base + ch * 8 + (idx - 1));
            }
            for (int i = 0; i < 3; ++i) {  // (alpha rgb, log_lambda) x 3
                for (int c = 0; c < 3; ++c) put(alpha + 3 * i + c);
                put(lambda + i);
            }
        }
    } else {
        err = "cannot detect checkpoint layout of " + t.path + " (expected f_rest_* or sg_alpha_* properties)";
        return SGS_ERR_FORMAT;
    }
    apply_meta_sidecar(t.path, info);
    info.count = t.count;
    info.binary = t.binary ? 1 : 0;
    return SGS_OK;
}

void ply_rows_to_flat(const PlyTable& t, const float* rows, double* params) {
    const size_t stride = t.props.size(), np = t.src.size();
    for (uint64_t i = 0; i < t.count; ++i) {
        const float* row = rows + i * stride;
        double* out = params + i * np;
        for (size_t p = 0; p < np; ++p) out[p] = static_cast<double>(row[t.src[p]]);
    }
}

}  // namespace sgs
