/*
 * fkde_io.h -- sample / value file I/O of the B200 engine (libfkde_b200.so),
 * the step before and after the estimator path.
 *
 * Same file formats as the reference (proj/core/include/fkde/io.hpp:11-38,
 * io.cpp:55-275), so files move freely between the two tools:
 *
 *   fkde_io_read_samples      <- fkde::io::read_samples        io.hpp:29, io.cpp:177-190
 *                                (FKDE magic -> binary, else CSV)
 *   fkde_io_write_samples_bin <- fkde::io::write_samples_bin   io.hpp:18, io.cpp:55-74
 *   fkde_io_write_samples_csv <- fkde::io::write_samples_csv   io.hpp:23, io.cpp:106-127
 *   fkde_io_write_values      <- fkde::io::write_values        io.hpp:33-34, io.cpp:192-229
 *   fkde_io_read_values       <- fkde::io::read_values         io.hpp:35, io.cpp:231-258
 *
 * Binary container: "FKDE", u32 version 1, u64 n, u64 d, n*d little-endian
 * doubles, row-major.  CSV: header "x0,...,x{d-1}", 17 significant digits.
 *
 * B200 difference: fkde_io_read_samples can place the samples straight into
 * page-locked (pinned) host memory (cudaHostAlloc), so the engine's
 * host->device copy of a file-backed input is one DMA at full PCIe/C2C rate
 * with no pageable staging copy; the device-side centring, scaling and fp16
 * hi/lo split happen in the pack kernel on the way into the operand tiles.
 *
 * Errors: calls return FKDE_IO_OK or an fkde_io_status; the message of the
 * last failure on the calling thread is fkde_io_last_error().  The reference
 * throws fkde::IoError (io errors) / InvalidArgumentError (bad arguments).
 */
#ifndef FKDE_IO_H
#define FKDE_IO_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum fkde_io_status {
    FKDE_IO_OK = 0,
    FKDE_IO_ERROR = 1,            /* fkde::IoError: open/read/write/format failure */
    FKDE_IO_INVALID_ARGUMENT = 2  /* fkde::InvalidArgumentError                    */
} fkde_io_status;

/* Reads a sample file (binary or CSV, dispatched on the magic).  *out is
 * allocated by the library.  *pinned on entry requests page-locked memory;
 * on return it says what was allocated (1 pinned, 0 malloc -- e.g. on a host
 * without a CUDA driver); release with fkde_io_free(*out, *pinned). */
int fkde_io_read_samples(const char* path, double** out, size_t* n, size_t* d, int* pinned);
void fkde_io_free(double* p, int pinned);
/* count doubles of host memory, page-locked when *pinned (in: requested,
 * out: granted); NULL when out of memory.  Release with fkde_io_free. */
double* fkde_io_alloc(size_t count, int* pinned);

int fkde_io_write_samples_bin(const char* path, const double* values, size_t n, size_t d);
int fkde_io_write_samples_csv(const char* path, const double* values, size_t n, size_t d);

/* format: "csv" (header "value"), "bin" (n x 1 FKDE container) or "json" (array) */
int fkde_io_write_values(const char* path, const double* values, size_t m, const char* format);
/* *out is malloc'ed; release with fkde_io_free(*out, 0) */
int fkde_io_read_values(const char* path, double** out, size_t* m);

const char* fkde_io_last_error(void);

#ifdef __cplusplus
}
#endif

#endif /* FKDE_IO_H */
