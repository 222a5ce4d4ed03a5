// gs_io.hpp -- host-side file formats of the reference (vtk.cpp, imaging.cpp), internal API.
//
// The snapshot writer formats on a pool of host threads with an exact %.17g formatter
// (gsio::fmt17) so that snapshot files are byte-identical to the reference's
// `snprintf("%.17g")` output (vtk.cpp:16-20) at a fraction of the cost.
#pragma once

#include <cstdint>
#include <cstdio>
#include <string>

namespace gsio {

// Writes |v| formatted exactly as printf("%.17g", v) into out (>= 32 bytes); returns the
// length (no terminator written).
int fmt17(double v, char* out);

// Error carried back to the C-ABI: code is a gs_status value.
struct Error {
    int code = 0;
    std::string msg;
};

// vtk.cpp:59-91 -- header, values, optional material array, into an open FILE*.  Does not
// close f.  Returns false (and fills err) on a write failure.
bool write_vtk_stream(std::FILE* f, const std::string& path, const double* u, int nx, int ny, int nz, double h,
                      const double origin[3], const uint8_t* labels, int threads, Error& err);

// The lines of write_vtk before the values (vtk.cpp:70-80); the material section's two header
// lines are kVtkMaterialHead.
std::string vtk_header(int nx, int ny, int nz, double h, const double origin[3]);
constexpr const char* kVtkMaterialHead = "SCALARS material int 1\nLOOKUP_TABLE default\n";

int default_threads();

// The 128-bit truncated powers of ten behind fmt17 (10^q = (hi:lo) * 2^b for q = qmin ..
// qmin + count - 1), for the device formatter.  Arrays need kPow10Count entries.
constexpr int kPow10Count = 646;
void pow10_table_export(uint64_t* hi, uint64_t* lo, int* b, int* qmin, int* count);

}  // namespace gsio
