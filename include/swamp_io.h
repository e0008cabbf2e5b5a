/* swamp_io.h — C-ABI of the data formats either side of the hot path
 * (SPEC.md "io" module, and the engine's
 * compare operation). Host code; the library is the same
 * libswamp_gpu.so.
 *
 * Rasters follow the Esri ASCII grid format: header keys
 * ncols, nrows, xllcorner, yllcorner, cellsize, NODATA_value, then
 * whitespace-separated values, TOP row first. The engine's finest-grid
 * arrays are row-major with the SOUTH row first (zorder.hpp:11-12), so
 * load_dem / write_finest flip the rows.
 */
#ifndef SWAMP_IO_H
#define SWAMP_IO_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* RasterGrid. `values` (ncols * nrows, top row first) is
 * allocated by swamp_io_read_esri and released by swamp_io_free_raster. */
typedef struct swamp_raster {
    int32_t ncols, nrows;
    double xllcorner, yllcorner, cellsize, nodata;
    double* values;
} swamp_raster;

/* load / save a raster. Errors: SWAMP_E_ARG (malformed header, missing or
 * non-numeric values — `msg` gets the line / value position), SWAMP_E_STATE
 * (I/O failure). Writing uses 17 significant digits, so a write-then-read
 * round trip is bit-exact on finite doubles. */
int swamp_io_read_esri(const char* path, swamp_raster* out, char* msg, size_t msg_cap);
int swamp_io_write_esri(const char* path, const swamp_raster* r);
void swamp_io_free_raster(swamp_raster* r);

/* load_dem: sample the raster at the finest-cell centres of
 * the 2^L x 2^L grid over the square [x0, x0 + W) x [y0, y0 + W): nearest
 * raster cell when the raster's cellsize equals W / 2^L, bilinear between
 * raster cell centres otherwise. Cells outside the raster or whose sample
 * touches a nodata value are inactive (inactive[k] = 1) and get z = wall_z
 * (a dry wall above every wet surface). Outputs are row-major,
 * SOUTH row first (4^L entries). strict != 0 requires 2^L >= max(ncols,
 * nrows) ("L must be set to accommodate the DEM resolution"). */
int swamp_io_load_dem(const swamp_raster* r, int L, double x0, double y0, double W, double wall_z, int strict,
                      double* z, uint8_t* inactive);

/* a finest-grid field (row-major, south row first, 2^L x 2^L over
 * [x0, x0 + W)^2) as an Esri raster, nodata where inactive (may be NULL) */
int swamp_io_write_finest(const char* path, int L, double x0, double y0, double W, const double* field,
                          const uint8_t* inactive, double nodata);

/* write_gauges: CSV, header "t,<name>_h,<name>_qx,
 * <name>_qy,<name>_eta,..." (names NULL: g0, g1, ...), then one record per
 * sample time: values[k] holds the 4 n_gauges doubles swamp_gpu_sample_gauges
 * wrote at times[k]. 17 significant digits. n_times = 0 (or n_gauges = 0):
 * header-only file. */
int swamp_io_write_gauges(const char* path, int32_t n_gauges, const char* const* names, int32_t n_times,
                          const double* times, const double* values);

/* write_step_report: CSV of StepReports, one record per
 * step, columns in this stable order:
 *   step,t,dt_used,dt_next,n_leaves,n_leaves_next,n_near_threshold,
 *   ms_encode_flag,ms_band_closure,ms_decode_traverse,ms_neighbours,ms_fv1,ms_total
 * `reports` points at n swamp_step_report structs (include/swamp_gpu.h);
 * append != 0 appends records without a header. */
struct swamp_step_report;
int swamp_io_write_step_reports(const char* path, int32_t n, const struct swamp_step_report* reports, int append);

#ifdef __cplusplus
}
#endif
#endif /* SWAMP_IO_H */
