/* oracle/fftw_shim/fftw3.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Minimal FFTW3-API shim so the UNMODIFIED reference library
 * (/root/reference/proj/core/src/fft.cpp) links in this image, which has no
 * libfftw3. It declares exactly the FFTW entry points the reference uses
 * (fft.cpp:3, 39-40, 49): fftw_complex, fftw_plan, fftw_plan_dft,
 * fftw_execute_dft and the FFTW_FORWARD/BACKWARD/ESTIMATE/UNALIGNED flags.
 *
 * The arithmetic (oracle/fftw_shim/fftw_shim.cpp) is our own O(N log N)
 * mixed-radix Stockham FFT restating FFTW's published definition: an
 * unnormalized DFT, X[k] = sum_n x[n] exp(sign * 2 pi i n k / N), with
 * FFTW_FORWARD = -1 and FFTW_BACKWARD = +1, row-major multi-dimensional.
 * FFTW itself (3.x, unpinned: core/CMakeLists.txt:1-2) is absent here.
 *
 * Nothing in the product path links this file.
 */
#ifndef SHEARLET_ORACLE_FFTW3_SHIM_H
#define SHEARLET_ORACLE_FFTW3_SHIM_H

#ifdef __cplusplus
extern "C" {
#endif

typedef double fftw_complex[2];
typedef struct fftw_plan_s* fftw_plan;

#define FFTW_FORWARD (-1)
#define FFTW_BACKWARD (+1)
#define FFTW_MEASURE (0U)
#define FFTW_ESTIMATE (1U << 6)
#define FFTW_UNALIGNED (1U << 1)

fftw_plan fftw_plan_dft(int rank, const int* n, fftw_complex* in, fftw_complex* out,
                        int sign, unsigned flags);
void fftw_execute_dft(const fftw_plan p, fftw_complex* in, fftw_complex* out);
void fftw_destroy_plan(fftw_plan p);

#ifdef __cplusplus
}
#endif

#endif
