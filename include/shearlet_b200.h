/* shearlet_b200.h -- C ABI of the B200-native shearlet dec/rec hot path.
 *
 * A drop-in for the reference's public C++ API for this path
 * (/root/reference/proj/core/include/shearlet/...), exported as plain C so any
 * host (C++, Python ctypes, cgo, JNI) can bind it. Plain pointers and sizes
 * only; no CUDA, torch or C++ types cross the boundary (streams are void*).
 *
 * Conventions (mirroring the reference):
 *  - row-major grids, last axis fastest, axis 0 the "horizontal" filter-bank
 *    axis (grid.hpp:12-13, 41);
 *  - coefficient stacks are contiguous [R][dims...] float64, bands in the
 *    system's filter order (enumerate_filters_2d/3d, system2d.cpp:59-73,
 *    system3d.cpp:58-80);
 *  - forward = unnormalised periodic cross-correlation with each filter:
 *    band_i = Re IDFT(conj(psi_i) .* DFT(f)) (transform.hpp:27-31);
 *  - inverse = Re IDFT(sum_i DFT(c_i) .* psi_i / W) (transform.hpp:33-37);
 *  - hard threshold keeps |x| >= K[scale - j0] * sigma (* RMS_i when scaled),
 *    lowpass untouched (apps.hpp:31-44, apps.cpp:57-81);
 *  - every error is an int code (below) mapping 1:1 to the reference's
 *    exception classes (errors.hpp:9-56); sl_last_error() gives the message.
 *
 * "_dev" entry points take device pointers on the handle's device and run on
 * the given CUDA stream (NULL = legacy default stream); "_host" entry points
 * take host pointers and include the H2D/D2H copies (synchronous).
 * A handle owns its device memory. Calls on one handle are serialised on the
 * GPU too: every call waits (cudaStreamWaitEvent) for the previous call on the
 * handle to finish, whatever streams the two were issued on, because they
 * share the handle's scratch.
 */
#ifndef SHEARLET_B200_H
#define SHEARLET_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum sl_status {
    SL_OK = 0,
    SL_ERR_GENERIC = 1,          /* shearlet::Error (e.g. residue guard)        */
    SL_ERR_SHAPE = 2,            /* shearlet::ShapeError                         */
    SL_ERR_CONFIG = 3,           /* shearlet::ConfigError                        */
    SL_ERR_DOMAIN = 4,           /* shearlet::DomainError                        */
    SL_ERR_SINGULAR_FRAME = 5,   /* shearlet::SingularFrameError                 */
    SL_ERR_UNSUPPORTED_SIZE = 6, /* shearlet::UnsupportedSizeError               */
    SL_ERR_ASSET = 7,            /* shearlet::AssetError                         */
    SL_ERR_FORMAT = 8,           /* shearlet::FormatError                        */
    SL_ERR_DEGENERATE_MASK = 9,  /* shearlet::DegenerateMaskError                */
    SL_ERR_DEGENERATE_TRUTH = 10, /* shearlet::DegenerateTruthError              */
    SL_ERR_CUDA = 20,            /* CUDA runtime failure                         */
    SL_ERR_NCCL = 21,            /* NCCL failure / libnccl.so.2 not loadable     */
    SL_ERR_INVALID = 22,         /* null handle / bad argument at the ABI        */
};

typedef struct sl_system sl_system;
typedef struct sl_comm sl_comm;

/* Library / device queries. */
const char* sl_version(void);
const char* sl_last_error(void);
int sl_device_count(int* count);

/* ---- system construction ------------------------------------------------
 * Replaces build_system_2d (system2d.hpp:66-69) / build_system_3d
 * (system3d.hpp:68-71) with ScaleProfile::from_levels(levels, j0)
 * (filters.hpp:88), QmfPair::maximally_flat_9tap() (filters.hpp:21) and
 * default_fan_filter() (filters.hpp:58) or FanFilter::impulse()
 * (impulse_fan != 0, filters.hpp:51).  The filter spectra, W and RMS are
 * computed on `device`.  shard_lo/shard_hi restrict the handle to bands
 * [lo, hi) of the full system (multi-GPU shearlet-index sharding); pass 0, -1
 * for the whole system. */
int sl_system_create_2d(int rows, int cols, const int* levels, int n_scales, int j0, int full_system,
                        int impulse_fan, int device, int shard_lo, int shard_hi, sl_system** out);
int sl_system_create_3d(int n0, int n1, int n2, const int* levels, int n_scales, int j0, int full_system,
                        int impulse_fan, int device, int shard_lo, int shard_hi, sl_system** out);
/* Same with an explicit filter bank: build_system_2d/3d(..., fan, qmf, ...)
 * with a user FanFilter (row-major fan_rows x fan_cols taps, centre
 * (fan_c0, fan_c1); e.g. load_fan_filter, filters.hpp:54-67,
 * fan_design.cpp:70-108) and QmfPair (1D taps + centre index; filters.hpp:14-21).
 * lowpass NULL = maximally_flat_9tap(); highpass NULL = mirror_highpass(lowpass)
 * (QmfPair::from_lowpass); fan NULL = default_fan_filter(). fan_provenance is
 * FanFilter::provenance ("dmaxflat4", "impulse", anything else = "custom" in
 * descriptors; NULL = "custom"). The filter spectra must come out real
 * (centrally symmetric taps), else SL_ERR_DOMAIN. */
int sl_system_create_2d_ex(int rows, int cols, const int* levels, int n_scales, int j0, int full_system,
                           const double* lowpass, int lowpass_len, int lowpass_center, const double* highpass,
                           int highpass_len, int highpass_center, const double* fan, int fan_rows, int fan_cols,
                           int fan_c0, int fan_c1, const char* fan_provenance, int device, int shard_lo,
                           int shard_hi, sl_system** out);
int sl_system_create_3d_ex(int n0, int n1, int n2, const int* levels, int n_scales, int j0, int full_system,
                           const double* lowpass, int lowpass_len, int lowpass_center, const double* highpass,
                           int highpass_len, int highpass_center, const double* fan, int fan_rows, int fan_cols,
                           int fan_c0, int fan_c1, const char* fan_provenance, int device, int shard_lo,
                           int shard_hi, sl_system** out);
/* default_fan_filter() (filters.cpp:112-122): the bundled 15x15 dmaxflat4
 * fan (a checksum-verified constant table); dims/centre always written, taps
 * written when non-NULL (cap doubles). */
int sl_default_fan(double* taps, int64_t cap, int* rows, int* cols, int* c0, int* c1);
/* System descriptors (descriptor.hpp:12-39): sl_describe writes the text
 * write_descriptor() would write (describe(sys)); len = its length without the
 * NUL; text may be NULL to size. sl_system_create_from_descriptor parses that
 * text (read_descriptor) and rebuilds (build_from_descriptor_2d/3d; ndim 2 or
 * 3 asserts the kind, 0 accepts both). FormatError cases as the reference. */
int sl_describe(const sl_system* sys, char* text, size_t cap, size_t* len);
int sl_system_create_from_descriptor(const char* text, int ndim, int device, int shard_lo, int shard_hi,
                                     sl_system** out);
int sl_system_destroy(sl_system* sys);

/* ---- system queries (ShearletSystem2D/3D members) ------------------------ */
int sl_ndim(const sl_system* sys, int* ndim, int64_t dims[3]);
int sl_redundancy(const sl_system* sys, int* R);          /* redundancy(): full system */
int sl_shard(const sl_system* sys, int* lo, int* hi);      /* bands held by this handle */
/* index records, 4 x int32 per filter: kind, scale, k1 (2D: shear), k2 (2D: 0);
 * kinds as FilterKind2D/3D (system2d.hpp:12-16, system3d.hpp:12-17). */
int sl_index(const sl_system* sys, int32_t* records);
int sl_filter_norms(const sl_system* sys, double* rms);    /* filter_norms: R doubles */
int sl_frame_weight(const sl_system* sys, double* w);      /* frame_weight: full grid (host) */
int sl_frame_bounds(const sl_system* sys, double* A, double* B);
/* psi_hat_i on the full grid, interleaved (re, im) (filters[i] / filter_freq(i)). */
int sl_filter_spectrum(sl_system* sys, int i, double* out);

/* ---- hot path, device pointers ------------------------------------------- */
/* forward(): f [dims] -> coeffs [hi-lo][dims] (this handle's bands). */
int sl_sheardec_dev(sl_system* sys, const double* f, double* coeffs, void* stream);
/* forward() + hard_threshold() fused into the dec epilogue. */
int sl_sheardec_threshold_dev(sl_system* sys, const double* f, double* coeffs, const double* K, int nK,
                              double sigma, int scale_by_rms, void* stream);
/* inverse(): coeffs [nbands][dims] -> f [dims]; nbands must equal the
 * handle's band count (ShapeError otherwise). On a shard the result is that
 * shard's partial sum (linear in the coefficients; sum over shards = full). */
int sl_shearrec_dev(sl_system* sys, const double* coeffs, int nbands, double* f, void* stream);
/* hard_threshold(): in -> out (may alias), nK must equal n_scales. */
int sl_hard_threshold_dev(sl_system* sys, const double* in, double* out, int nbands, const double* K, int nK,
                          double sigma, int scale_by_rms, void* stream);
/* denoise(): inverse(hard_threshold(forward(in))) (apps.cpp:114-121), fused:
 * the threshold runs in the dec epilogue and the rec reads the thresholded
 * rows in the same pass. The stack goes to the handle's device scratch while
 * sl_set_stack_output is on (default). */
int sl_denoise_dev(sl_system* sys, const double* in, double* out, const double* K, int nK, double sigma,
                   int scale_by_rms, void* stream);
/* The same fused denoise, also writing the thresholded stack
 * hard_threshold(forward(in)) [nbands][dims] into `stack` (device). */
int sl_denoise_stack_dev(sl_system* sys, const double* in, double* stack, double* out, const double* K, int nK,
                         double sigma, int scale_by_rms, void* stream);

/* ---- batched hot path (device pointers) ----------------------------------
 * nframes independent signals, contiguous [nframes][dims]; stacks
 * [nframes][nbands][dims]. Frames are spread over up to sl_set_streams()
 * internal streams (default 6) that fork from and join back into `stream`,
 * so concurrent frames overlap on the GPU; results are identical to
 * per-frame calls. sl_sheardec_batch_dev thresholds when K != NULL. */
int sl_set_streams(sl_system* sys, int nstreams);
/* Whether the fused denoise (sl_denoise_*) writes the thresholded coefficient
 * stack to HBM (default 1, as the reference's denoise materialises it). With 0
 * the stack is never written: the same reconstruction, ~1/6 less HBM traffic
 * (reported separately from the stack-materialised numbers). */
int sl_set_stack_output(sl_system* sys, int materialize);
int sl_sheardec_batch_dev(sl_system* sys, const double* f, int nframes, double* coeffs, const double* K, int nK,
                          double sigma, int scale_by_rms, void* stream);
int sl_shearrec_batch_dev(sl_system* sys, const double* coeffs, int nframes, double* f, void* stream);
int sl_denoise_batch_dev(sl_system* sys, const double* in, int nframes, double* out, const double* K, int nK,
                         double sigma, int scale_by_rms, void* stream);
/* batched fused denoise that also returns every frame's thresholded stack,
 * stacks [nframes][nbands][dims] (device) -- the timed path's own output */
int sl_denoise_batch_stack_dev(sl_system* sys, const double* in, int nframes, double* stacks, double* out,
                               const double* K, int nK, double sigma, int scale_by_rms, void* stream);
/* host in/out: H2D of all frames + batched denoise + D2H, synchronous.
 * Pinned buffers are used as they are; pageable ones are page-locked
 * (cudaHostRegister) for the duration of the call. */
int sl_denoise_batch_host(sl_system* sys, const double* in, int nframes, double* out, const double* K, int nK,
                          double sigma, int scale_by_rms);

/* ---- hot path, host pointers (value semantics like the reference) -------- */
int sl_sheardec_host(sl_system* sys, const double* f, double* coeffs);
int sl_shearrec_host(sl_system* sys, const double* coeffs, int nbands, double* f);
int sl_hard_threshold_host(sl_system* sys, const double* in, double* out, int nbands, const double* K, int nK,
                           double sigma, int scale_by_rms);
int sl_denoise_host(sl_system* sys, const double* in, double* out, const double* K, int nK, double sigma,
                    int scale_by_rms);

/* ---- iterative thresholding pipelines ("next") ----------------
 * inpaint (apps.hpp:46-78, apps.cpp:179-235): estimate_{k+1} =
 * rec(thr_uniform(dec(mask .* (masked - estimate_k) + estimate_k), delta_k)),
 * delta_k = delta_init * delta_min^(k/(iterations-1)); delta_init < 0 selects
 * the largest (RMS-scaled) coefficient of the input. separate (apps.hpp:80-90,
 * apps.cpp:237-280) runs the same scheme jointly over a directional and an
 * isotropic system. The whole loop runs on the device. */
int sl_inpaint_dev(sl_system* sys, const double* masked, const double* mask, double* out, int iterations,
                   double delta_init, double delta_min, int scale_by_rms, void* stream);
int sl_inpaint_host(sl_system* sys, const double* masked, const double* mask, double* out, int iterations,
                    double delta_init, double delta_min, int scale_by_rms);
int sl_separate_dev(sl_system* directional, sl_system* isotropic, const double* signal, double* curves, double* blobs,
                    int iterations, double delta_init, double delta_min, int scale_by_rms, void* stream);
int sl_separate_host(sl_system* directional, sl_system* isotropic, const double* signal, double* curves,
                     double* blobs, int iterations, double delta_init, double delta_min, int scale_by_rms);

/* ---- SHCF coefficient files (transform.hpp:39-52, transform.cpp:127-269) --
 * Host buffers; byte-identical to the reference's serialize(). The records
 * are the handle's bands; deserialize checks magic, version, dims, band
 * count and index records against the system (FormatError / ShapeError). */
int sl_shcf_size(const sl_system* sys, int nbands, size_t* bytes);
int sl_shcf_serialize(const sl_system* sys, const double* coeffs, int nbands, unsigned char* out, size_t cap);
int sl_shcf_deserialize(const sl_system* sys, const unsigned char* in, size_t len, double* coeffs, int nbands);
/* Streamed SHCF files (stacks larger than host/HBM budgets):
 * forward() of host signal f written straight to `path` as SHCF, and inverse()
 * read straight from `path`, bands_per_chunk bands at a time (<= 0: ~2 GB
 * chunks). Same bytes as sl_shcf_serialize(forward(f)); the streamed inverse
 * sums per-chunk partial reconstructions (equal to inverse() within 1e-15). */
int sl_shcf_forward_file(sl_system* sys, const double* f, const char* path, int bands_per_chunk);
int sl_shcf_inverse_file(sl_system* sys, const char* path, double* out, int bands_per_chunk);

/* ---- signal files (image_io.hpp:9-24, image_io.cpp:43-159), host ---------
 * PGM: binary P5, 8-bit (maxval <= 255) or 16-bit big-endian samples; rows =
 * image height = axis 0. Load with pixels == NULL to query rows/cols/maxval.
 * Save rounds, clamps to [0, maxval]. SVOL: "SVOL", u16 1, 3 x u32 dims, f64
 * samples, little-endian. Errors: SL_ERR_FORMAT as the reference's FormatError. */
int sl_load_pgm(const char* path, double* pixels, int64_t cap, int* rows, int* cols, int* maxval);
int sl_save_pgm(const double* pixels, int rows, int cols, const char* path, int maxval);
int sl_load_svol(const char* path, double* volume, int64_t cap, int64_t dims[3]);
int sl_save_svol(const double* volume, const int64_t dims[3], const char* path);

/* ---- separation-quality metrics (apps.hpp:92-101, apps.cpp:282-362) -----
 * Host buffers, rows x cols row-major. The periodic Gaussian blur runs on the
 * GPU through the hot path's single-band decomposition; the kernel taps must
 * be centrally symmetric (gaussian_kernel's are). Errors as the reference:
 * DomainError (truth not binary, delta < 0, sigma <= 0), DegenerateTruthError. */
int sl_gaussian_kernel(double sigma_pixels, double* taps, int64_t cap, int* size, int* center);
int sl_binarize(const double* in, double* out, int64_t count, double delta);
int sl_quality_q(int rows, int cols, const double* recovered, const double* truth, double delta,
                 const double* kernel, int k_rows, int k_cols, int k_c0, int k_c1, int device, double* q);
/* quality_q_opt: minimum over integer delta = 0..255 (ties: smallest delta);
 * q_all (optional, 256 doubles) receives every Q(delta). */
int sl_quality_q_opt(int rows, int cols, const double* recovered, const double* truth, const double* kernel,
                     int k_rows, int k_cols, int k_c0, int k_c1, int device, double* q, int* best_delta,
                     double* q_all);

/* ---- instrumentation ---------------------------------------------------
 * sl_profile(enable) clears the per-pass statistics and turns CUDA-event timing
 * of every kernel launch on/off; sl_pass_stats returns, per pass name (32-byte
 * NUL-padded slots), the summed device time in ms, the launch count and the
 * number of bands/spectra those launches processed since the last sl_profile
 * call. sl_launch_count is the cumulative number of kernels this handle has
 * launched (construction included). */
int sl_profile(sl_system* sys, int enable);
int sl_pass_stats(sl_system* sys, int max_passes, char* names, double* ms_total, int64_t* launches, int64_t* units,
                  int* n_passes);
int sl_launch_count(const sl_system* sys, int64_t* count);

/* ---- synthetic inputs (phantoms.hpp / apps.hpp generators, host) ---------- */
int sl_phantom_cartoon(int n, double* out);            /* phantoms::cartoon        */
int sl_phantom_cartoon_volume(int n, double* out);     /* phantoms::cartoon_volume */
int sl_add_gaussian_noise(const double* in, double* out, int64_t count, double sigma, uint64_t seed);

/* ---- optional fp32 mode (north_star: "within 1e-5 in an optional float32
 * mode"; the reference itself is fp64 only, grid.hpp:78-85) ------------------
 * sl_system_set_precision(sys, 32) rounds the handle's filter tables to
 * float (square 2D fast-path grids: 64..2048 and 192) and enables the *_f32
 * entry points, which take float signals / stacks and run every FFT pass in
 * fp32. Cubic 3D grids (64/128/192/256) support the fused denoise
 * (sl_denoise_f32_dev): the three band passes run on float2 spectra, the
 * filters are synthesised in fp64 and rounded, the input spectrum and the
 * final inverse (one spectrum each) run in fp64. Thresholds (K sigma RMS) are
 * compared in fp64. */
int sl_system_set_precision(sl_system* sys, int bits);
int sl_sheardec_f32_dev(sl_system* sys, const float* f, float* coeffs, const double* K, int nK, double sigma,
                        int scale_by_rms, void* stream);
int sl_shearrec_f32_dev(sl_system* sys, const float* coeffs, int nbands, float* f, void* stream);
/* fused denoise; stack may be NULL (then the scratch stack, when materialised) */
int sl_denoise_f32_dev(sl_system* sys, const float* in, float* stack, float* out, const double* K, int nK,
                       double sigma, int scale_by_rms, void* stream);
int sl_denoise_batch_f32_dev(sl_system* sys, const float* in, int nframes, float* stacks, float* out,
                             const double* K, int nK, double sigma, int scale_by_rms, void* stream);

/* ---- multi-GPU (one process per GPU) -------------------------
 * The filter index -- the reference's only parallel axis (parallel_for,
 * parallel.hpp:20-46) -- shards across GPUs: rank r owns the balanced band
 * range sl_partition(R, nranks, r). sl_denoise_dist_dev broadcasts the
 * input from `root` (in: device buffer on every rank, read on the root,
 * overwritten elsewhere), runs the fused dec -> threshold -> rec of this
 * rank's bands and NCCL-reduces the reconstruction onto the root (3D: the
 * half-spectrum accumulators; the root alone divides by W and inverts).
 * Batched 2D frames shard by image with no collective
 * (sl_denoise_batch_dist_*: frames sl_partition(nframes, ...) of a globally
 * indexed batch). NCCL is loaded at run time; SL_ERR_NCCL when absent. */
int sl_comm_unique_id(unsigned char* id /* 128 bytes, NCCL_UNIQUE_ID_BYTES */);
int sl_comm_create(const unsigned char* id, int nranks, int rank, int device, sl_comm** out);
int sl_comm_destroy(sl_comm* comm);
int sl_comm_info(const sl_comm* comm, int* nranks, int* rank, int* device);
int sl_partition(int64_t count, int nranks, int rank, int64_t* lo, int64_t* hi);
/* attach (or, with NULL, detach) a communicator; shard_bands != 0 restricts
 * the handle to this rank's band range, 0 keeps the whole bank (2D batches) */
int sl_system_set_comm(sl_system* sys, sl_comm* comm, int shard_bands);
int sl_denoise_dist_dev(sl_system* sys, const double* in, double* out, const double* K, int nK, double sigma,
                        int scale_by_rms, int root, void* stream);
int sl_denoise_batch_dist_dev(sl_system* sys, const double* in, int nframes, double* out, const double* K, int nK,
                              double sigma, int scale_by_rms, void* stream);
int sl_denoise_batch_dist_host(sl_system* sys, const double* in, int nframes, double* out, const double* K, int nK,
                               double sigma, int scale_by_rms);

#ifdef __cplusplus
}
#endif

#endif /* SHEARLET_B200_H */
