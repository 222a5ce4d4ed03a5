// gs_vtkfmt.cuh -- GPU formatting of VTK value columns (gs_vtkfmt.cu).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace gs {

// Longest "%.17g" line: "-1.2345678901234567e-308\n".
constexpr int kVtkMaxLine = 25;

struct VtkfmtScratch {
    unsigned long long* lens = nullptr;  // [n] line lengths
    unsigned long long* offs = nullptr;  // [n] byte offsets (exclusive scan)
    char* text = nullptr;                // [n * kVtkMaxLine] value lines
    void* scan_tmp = nullptr;
    size_t scan_bytes = 0;
    int* tie = nullptr;                  // set when some value needs the host formatter
    uint8_t* lab = nullptr;              // [n] material codes
    char* ltext = nullptr;               // [2n] "d\n" label lines
};

// Upload the powers-of-ten table (once per process).
cudaError_t vtkfmt_init();
size_t vtkfmt_scratch_bytes(int64_t n);
// Format u[0..n) into s.text (lines at s.offs); s.tie flags a value the host must format.
cudaError_t vtkfmt_values(const double* u, int64_t n, VtkfmtScratch& s, cudaStream_t stream);
// Material codes (all < 10) as "d\n" lines.
cudaError_t vtkfmt_labels(const uint8_t* lab, int64_t n, char* text, cudaStream_t stream);

}  // namespace gs
