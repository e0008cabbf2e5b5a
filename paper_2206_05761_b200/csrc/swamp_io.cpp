// swamp_io.cpp — Esri ASCII rasters and DEM ingestion (include/swamp_io.h;
// SPEC.md:541-600). Host code, compiled into libswamp_gpu.so.
#include "swamp_io.h"

#include <cctype>
#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "swamp_gpu.h"

namespace {

void set_msg(char* msg, size_t cap, const std::string& s) {
    if (msg && cap) {
        std::strncpy(msg, s.c_str(), cap - 1);
        msg[cap - 1] = 0;
    }
}

bool key_is(const char* a, const char* b) {
    for (; *a && *b; ++a, ++b)
        if (std::tolower(static_cast<unsigned char>(*a)) != std::tolower(static_cast<unsigned char>(*b))) return false;
    return *a == 0 && *b == 0;
}

}  // namespace

extern "C" {

int swamp_io_read_esri(const char* path, swamp_raster* out, char* msg, size_t msg_cap) {
    if (!path || !out) return SWAMP_E_ARG;
    std::memset(out, 0, sizeof(*out));
    FILE* f = std::fopen(path, "r");
    if (!f) {
        set_msg(msg, msg_cap, std::string("cannot open ") + path);
        return SWAMP_E_STATE;
    }
    double hv[6] = {NAN, NAN, NAN, NAN, NAN, -9999.0};
    bool have[6] = {false, false, false, false, false, false};
    const char* names[6] = {"ncols", "nrows", "xllcorner", "yllcorner", "cellsize", "NODATA_value"};
    char key[64], val[128];
    bool xc = false, yc = false;
    long pos = std::ftell(f);
    int line = 0;
    // header: "key value" lines until the first line whose first token is numeric
    while (std::fscanf(f, "%63s", key) == 1) {
        char* end = nullptr;
        std::strtod(key, &end);
        if (end && *end == 0) {  // a number: the data starts here
            std::fseek(f, pos, SEEK_SET);
            break;
        }
        ++line;
        if (std::fscanf(f, "%127s", val) != 1) {
            std::fclose(f);
            set_msg(msg, msg_cap, "malformed header at line " + std::to_string(line) + ": no value for " + key);
            return SWAMP_E_ARG;
        }
        int k = -1;
        for (int q = 0; q < 6; ++q)
            if (key_is(key, names[q])) k = q;
        if (k < 0 && key_is(key, "xllcenter")) {  // centre form: corner = centre - cellsize / 2
            k = 2;
            xc = true;
        }
        if (k < 0 && key_is(key, "yllcenter")) {
            k = 3;
            yc = true;
        }
        if (k < 0) {
            std::fclose(f);
            set_msg(msg, msg_cap, "malformed header at line " + std::to_string(line) + ": unknown key " + key);
            return SWAMP_E_ARG;
        }
        hv[k] = std::strtod(val, &end);
        if (!end || *end != 0) {
            std::fclose(f);
            set_msg(msg, msg_cap, "malformed header at line " + std::to_string(line) + ": bad value " + val);
            return SWAMP_E_ARG;
        }
        have[k] = true;
        pos = std::ftell(f);
    }
    for (int q = 0; q < 5; ++q)
        if (!have[q]) {
            std::fclose(f);
            set_msg(msg, msg_cap, std::string("malformed header: missing ") + names[q]);
            return SWAMP_E_ARG;
        }
    const double nc = hv[0], nr = hv[1];
    if (!(nc >= 1 && nr >= 1 && nc == std::floor(nc) && nr == std::floor(nr) && nc * nr < 1e10 && hv[4] > 0)) {
        std::fclose(f);
        set_msg(msg, msg_cap, "malformed header: ncols / nrows / cellsize");
        return SWAMP_E_ARG;
    }
    out->ncols = static_cast<int32_t>(nc);
    out->nrows = static_cast<int32_t>(nr);
    out->xllcorner = xc ? hv[2] - 0.5 * hv[4] : hv[2];
    out->yllcorner = yc ? hv[3] - 0.5 * hv[4] : hv[3];
    out->cellsize = hv[4];
    out->nodata = hv[5];
    const size_t n = static_cast<size_t>(out->ncols) * static_cast<size_t>(out->nrows);
    out->values = static_cast<double*>(std::malloc(n * sizeof(double)));
    if (!out->values) {
        std::fclose(f);
        return SWAMP_E_NOMEM;
    }
    for (size_t k = 0; k < n; ++k) {
        if (std::fscanf(f, "%127s", val) != 1) {
            std::fclose(f);
            swamp_io_free_raster(out);
            set_msg(msg, msg_cap, "expected " + std::to_string(n) + " values, found " + std::to_string(k));
            return SWAMP_E_ARG;
        }
        char* end = nullptr;
        out->values[k] = std::strtod(val, &end);
        if (!end || *end != 0) {
            std::fclose(f);
            swamp_io_free_raster(out);
            set_msg(msg, msg_cap, "non-numeric value '" + std::string(val) + "' at row " +
                                      std::to_string(k / out->ncols) + ", column " + std::to_string(k % out->ncols));
            return SWAMP_E_ARG;
        }
    }
    std::fclose(f);
    return SWAMP_OK;
}

void swamp_io_free_raster(swamp_raster* r) {
    if (r && r->values) {
        std::free(r->values);
        r->values = nullptr;
    }
}

int swamp_io_write_esri(const char* path, const swamp_raster* r) {
    if (!path || !r || !r->values || r->ncols < 1 || r->nrows < 1) return SWAMP_E_ARG;
    FILE* f = std::fopen(path, "w");
    if (!f) return SWAMP_E_STATE;
    std::fprintf(f, "ncols %d\nnrows %d\nxllcorner %.17g\nyllcorner %.17g\ncellsize %.17g\nNODATA_value %.17g\n",
                 r->ncols, r->nrows, r->xllcorner, r->yllcorner, r->cellsize, r->nodata);
    for (int j = 0; j < r->nrows; ++j) {
        for (int i = 0; i < r->ncols; ++i)
            std::fprintf(f, i ? " %.17g" : "%.17g", r->values[static_cast<size_t>(j) * r->ncols + i]);
        std::fputc('\n', f);
    }
    const bool ok = std::ferror(f) == 0;
    return (std::fclose(f) == 0 && ok) ? SWAMP_OK : SWAMP_E_STATE;
}

int swamp_io_load_dem(const swamp_raster* r, int L, double x0, double y0, double W, double wall_z, int strict,
                      double* z, uint8_t* inactive) {
    if (!r || !r->values || !z || L < 1 || L > 13 || !(W > 0.0)) return SWAMP_E_ARG;
    const int side = 1 << L;
    if (strict && side < (r->ncols > r->nrows ? r->ncols : r->nrows)) return SWAMP_E_ARG;
    const double dx = W / side, cs = r->cellsize;
    const bool nearest = dx == cs;
    const int nc = r->ncols, nr = r->nrows;
    auto val = [&](int ci, int rj) -> double {  // raster column ci, row rj counted from the SOUTH
        return r->values[static_cast<size_t>(nr - 1 - rj) * nc + ci];
    };
    auto is_nodata = [&](double v) { return v == r->nodata || !std::isfinite(v); };
    for (int j = 0; j < side; ++j)
        for (int i = 0; i < side; ++i) {
            const double x = x0 + (i + 0.5) * dx, y = y0 + (j + 0.5) * dx;  // finest-cell centre
            double zz = wall_z;
            bool in = false;
            if (nearest) {
                const double fi = std::floor((x - r->xllcorner) / cs), fj = std::floor((y - r->yllcorner) / cs);
                if (fi >= 0 && fj >= 0 && fi < nc && fj < nr) {
                    const double v = val(static_cast<int>(fi), static_cast<int>(fj));
                    if (!is_nodata(v)) {
                        zz = v;
                        in = true;
                    }
                }
            } else {
                // bilinear between raster cell centres; samples within half a
                // cell of the raster edge use the edge cells (clamped)
                const double u = (x - r->xllcorner) / cs - 0.5, w = (y - r->yllcorner) / cs - 0.5;
                if (u >= -0.5 && w >= -0.5 && u <= nc - 0.5 && w <= nr - 0.5) {
                    int i0 = static_cast<int>(std::floor(u)), j0 = static_cast<int>(std::floor(w));
                    double a = u - i0, b = w - j0;
                    if (i0 < 0) { i0 = 0; a = 0.0; }
                    if (j0 < 0) { j0 = 0; b = 0.0; }
                    if (i0 >= nc - 1) { i0 = nc - 1; a = 0.0; }
                    if (j0 >= nr - 1) { j0 = nr - 1; b = 0.0; }
                    const int i1 = i0 + 1 < nc ? i0 + 1 : i0, j1 = j0 + 1 < nr ? j0 + 1 : j0;
                    const double v00 = val(i0, j0), v10 = val(i1, j0), v01 = val(i0, j1), v11 = val(i1, j1);
                    const bool nd = (is_nodata(v00)) || (a > 0.0 && is_nodata(v10)) || (b > 0.0 && is_nodata(v01)) ||
                                    (a > 0.0 && b > 0.0 && is_nodata(v11));
                    if (!nd) {
                        const double s0 = (a > 0.0) ? v00 + a * (v10 - v00) : v00;
                        const double s1 = (a > 0.0) ? v01 + a * (v11 - v01) : v01;
                        zz = (b > 0.0) ? s0 + b * (s1 - s0) : s0;
                        in = true;
                    }
                }
            }
            const size_t k = static_cast<size_t>(j) * side + i;
            z[k] = zz;
            if (inactive) inactive[k] = in ? 0 : 1;
        }
    return SWAMP_OK;
}

int swamp_io_write_finest(const char* path, int L, double x0, double y0, double W, const double* field,
                          const uint8_t* inactive, double nodata) {
    if (!path || !field || L < 1 || L > 13 || !(W > 0.0)) return SWAMP_E_ARG;
    const int side = 1 << L;
    swamp_raster r;
    r.ncols = side;
    r.nrows = side;
    r.xllcorner = x0;
    r.yllcorner = y0;
    r.cellsize = W / side;
    r.nodata = nodata;
    std::vector<double> v(static_cast<size_t>(side) * side);
    for (int j = 0; j < side; ++j)  // top row first
        for (int i = 0; i < side; ++i) {
            const size_t k = static_cast<size_t>(j) * side + i;
            v[static_cast<size_t>(side - 1 - j) * side + i] = (inactive && inactive[k]) ? nodata : field[k];
        }
    r.values = v.data();
    return swamp_io_write_esri(path, &r);
}

int swamp_io_write_gauges(const char* path, int32_t n_gauges, const char* const* names, int32_t n_times,
                          const double* times, const double* values) {
    if (!path || n_gauges < 0 || n_times < 0 || (n_times > 0 && n_gauges > 0 && (!times || !values)))
        return SWAMP_E_ARG;
    FILE* f = std::fopen(path, "w");
    if (!f) return SWAMP_E_STATE;
    std::fputs("t", f);
    static const char* const q[4] = {"h", "qx", "qy", "eta"};
    for (int32_t g = 0; g < n_gauges; ++g)
        for (int k = 0; k < 4; ++k) {
            if (names && names[g]) std::fprintf(f, ",%s_%s", names[g], q[k]);
            else std::fprintf(f, ",g%d_%s", static_cast<int>(g), q[k]);
        }
    std::fputc('\n', f);
    if (n_gauges > 0)
        for (int32_t r = 0; r < n_times; ++r) {
            std::fprintf(f, "%.17g", times[r]);
            const double* v = values + static_cast<size_t>(r) * 4 * n_gauges;
            for (int32_t g = 0; g < n_gauges; ++g)
                for (int k = 0; k < 4; ++k) std::fprintf(f, ",%.17g", v[static_cast<size_t>(k) * n_gauges + g]);
            std::fputc('\n', f);
        }
    const bool ok = std::ferror(f) == 0;
    return (std::fclose(f) == 0 && ok) ? SWAMP_OK : SWAMP_E_STATE;
}

int swamp_io_write_step_reports(const char* path, int32_t n, const swamp_step_report* reports, int append) {
    if (!path || n < 0 || (n > 0 && !reports)) return SWAMP_E_ARG;
    FILE* f = std::fopen(path, append ? "a" : "w");
    if (!f) return SWAMP_E_STATE;
    if (!append)
        std::fputs("step,t,dt_used,dt_next,n_leaves,n_leaves_next,n_near_threshold,ms_encode_flag,ms_band_closure,"
                   "ms_decode_traverse,ms_neighbours,ms_fv1,ms_total\n",
                   f);
    for (int32_t k = 0; k < n; ++k) {
        const swamp_step_report& r = reports[k];
        std::fprintf(f, "%lld,%.17g,%.17g,%.17g,%lld,%lld,%lld,%.17g,%.17g,%.17g,%.17g,%.17g,%.17g\n",
                     static_cast<long long>(r.step), r.t, r.dt_used, r.dt, static_cast<long long>(r.n_leaves),
                     static_cast<long long>(r.n_leaves_next), static_cast<long long>(r.n_near_threshold),
                     r.ms_encode_flag, r.ms_band_closure, r.ms_decode_traverse, r.ms_neighbours, r.ms_fv1, r.ms_total);
    }
    const bool ok = std::ferror(f) == 0;
    return (std::fclose(f) == 0 && ok) ? SWAMP_OK : SWAMP_E_STATE;
}

}  // extern "C"
