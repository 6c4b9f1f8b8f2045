/*
 * magnex_b200.h -- C ABI of libmagnex_b200.so, the B200 (sm_100a) hot path of
 * MagneX: effective field H_eff (FFT demag, exchange, interfacial DMI,
 * uniaxial anisotropy, Zeeman; plus the unpinned extensions cubic anisotropy
 * and bulk DMI), the LLG torque and fused RK4 / forward-Euler stepping.
 *
 * The reference (magnex 0.1.0, /root/reference/pkg/src/magnex) is pure
 * Python; its "plugin seams" are duck-typed Python protocols, so every entry
 * point below names the Python interface it replaces.  The Python host mirror
 * (paper_2602_12242_b200/) binds this header with ctypes; INTEGRATION.md
 * shows the binding a reference maintainer would add.
 *
 * Conventions
 *   - Fields are float64 (3, nz, ny, nx), C-contiguous, x fastest
 *     (grid.py:1-8).  Host pointers are borrowed for the duration of a call.
 *   - Every call returns an mxb_status; mxb_last_error() gives the message of
 *     the last failure on the calling thread.
 *   - A context owns all device memory; it is not reentrant (like
 *     DemagKernel, demag.py:170-174): one host thread per context.
 */
#ifndef MAGNEX_B200_H
#define MAGNEX_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MXB_ABI_VERSION 1

typedef enum mxb_status {
    MXB_OK = 0,
    MXB_EINVAL = 1,      /* -> ValueError / GridError                          */
    MXB_EDEAD = 2,       /* -> RenormalizeError (grid.py:186-192)              */
    MXB_EBLOWUP = 3,     /* -> IntegrationBlowup (llg.py:54-61,348-353)        */
    MXB_ECUDA = 4,
    MXB_ENCCL = 5,
    MXB_EQUILIBRATED = 6 /* informational: run stopped on equilibrium          */
} mxb_status;

/* H_eff terms (llg.py:33 TERMS) -- accumulation order is exchange,
 * anisotropy, [cubic], dmi, [bulk dmi], demag, bias (llg.py:112-125). */
enum {
    MXB_TERM_EXCHANGE = 1u << 0,
    MXB_TERM_ANISOTROPY = 1u << 1,
    MXB_TERM_DMI = 1u << 2,
    MXB_TERM_DEMAG = 1u << 3,
    MXB_TERM_BIAS = 1u << 4,
    MXB_TERM_CUBIC = 1u << 5,    /* unpinned extension  */
    MXB_TERM_BULK_DMI = 1u << 6  /* unpinned extension  */
};

/* ghost modes of _StencilPlan (fields.py:18,49-92) */
enum { MXB_GHOST_NEUMANN = 0, MXB_GHOST_DMI = 1, MXB_GHOST_PERIODIC = 2 };

/* integrators (llg.py:206-222; MRI = explicit multirate Knoth-Wolke, integrators.py:97-128) */
enum { MXB_EULER = 0, MXB_RK4 = 1, MXB_MRI_KW3 = 2 };

/* GridSpec (grid.py:29-71) */
typedef struct mxb_grid {
    int64_t nx, ny, nz;
    double dx, dy, dz;
} mxb_grid;

/* MaterialMap (grid.py:119-175).  A per-cell pointer, when non-NULL,
 * overrides the scalar (shape (nz,ny,nx), or (3,nz,ny,nx) for eK).  eK must
 * already be unit-normalised as MaterialMap does (grid.py:147-152). */
typedef struct mxb_material {
    double Ms, A, Ku, D, alpha, gamma;
    double eK[3];
    const double *Ms_cell, *A_cell, *Ku_cell, *D_cell, *alpha_cell, *eK_cell;
    /* unpinned extensions */
    double Kc1;            /* cubic K1 [J/m^3]                  */
    double c1[3], c2[3];   /* cubic axes (orthonormal)          */
    double Db;             /* bulk DMI [J/m^2]                  */
} mxb_material;

/* PartitionedRHS configuration (llg.py:98-125) */
typedef struct mxb_terms {
    uint32_t mask;         /* MXB_TERM_* */
    int32_t ghost_mode;    /* MXB_GHOST_* */
    int32_t precession;    /* llg.py:69 */
    int32_t damping;       /* llg.py:71 */
} mxb_terms;

/* bias at one evaluation: uniform vector and/or a spatial field */
typedef struct mxb_bias {
    double vec[3];
    const double* field;        /* host (3,nz,ny,nx) or NULL */
    const double* demag_field;  /* host (3,nz,ny,nx) from a foreign demag
                                   backend (llg.py:119-121), used when the
                                   demag term is on and no mxb_demag is given */
} mxb_bias;

typedef struct mxb_ctx mxb_ctx;
typedef struct mxb_demag mxb_demag;

/* ---- library ---------------------------------------------------------- */
int mxb_abi_version(void);
const char* mxb_last_error(void);
int mxb_device_count(int* n);

/* ---- context: grid + material resident on one device ------------------
 * replaces MaterialMap's host arrays as seen by every operator
 * (grid.py:119-175, fields.py:102-163, llg.py:84-203) */
int mxb_ctx_create(const mxb_grid* g, const mxb_material* mat, int device, mxb_ctx** out);
int mxb_ctx_destroy(mxb_ctx* ctx);
/* exact=1: reference operation order, no FMA contraction, true divisions
 * (bit-faithful local terms); exact=0: FMA + reciprocal multiplies. */
int mxb_ctx_set_exact(mxb_ctx* ctx, int exact);

/* ---- demag (DemagKernel, demag.py:169-216) ----------------------------- */
int mxb_demag_create(const mxb_grid* g, int device, mxb_demag** out);
int mxb_demag_destroy(mxb_demag* d);
/* DemagKernel.from_packed (demag.py:189-195): packed (6,pz,py,px) host
 * real-space tensor -> device spectra (kept complex for exact parity) */
int mxb_demag_set_packed(mxb_demag* d, const double* packed);
/* DemagKernel.build (demag.py:183-187) on the GPU: Newell f/g lattice,
 * second differences, dipole far field beyond 60 diagonals, wrap-around
 * pack, 6 forward transforms.  symmetric=1 mirrors the displacement octant
 * so the spectra are exactly real and stores them parity-reduced. */
int mxb_demag_build(mxb_demag* d, int symmetric);
/* real-space tensor_elements (demag.py:90-120) from the GPU builder, host
 * (6, 2nz-1, 2ny-1, 2nx-1) */
int mxb_demag_tensor_elements(mxb_demag* d, double* out);
/* demag_field_direct (demag.py:225-248): O(N^2) direct sum over the source
 * cells of host m (3,nz,ny,nx) into host h, with the tensor elements n6
 * (6, 2nz-1, 2ny-1, 2nx-1) or, when n6 is NULL, the GPU builder's; the caller
 * enforces the reference's DIRECT_SUM_CELL_LIMIT */
int mxb_demag_direct(mxb_demag* d, const double* n6, const double* m, double* h);
/* DemagKernel.spectra (demag.py:179): host complex (6,pz,py,px/2+1) as
 * interleaved re/im doubles (unscaled, like scipy.fft.rfftn) */
int mxb_demag_get_spectra(mxb_demag* d, double* out);
/* DemagKernel.field / demag_field_fft (demag.py:203-222) */
int mxb_demag_field(mxb_demag* d, const double* m, double* h);
/* device pointers (same stream as the demag object), for callers that keep
 * fields resident */
int mxb_demag_field_dev(mxb_demag* d, const double* m_dev, double* h_dev);
size_t mxb_demag_bytes(mxb_demag* d);
/* select the register-resident radix-16 kernels (1, default) or the generic
 * mixed-radix shared-memory kernels (0) where both cover the shape */
/* spectra storage / y-z path of a built kernel: 0 complex (5-pass), 2 parity-reduced
 * real (5-pass), 3 plane-major real + L2-resident y/z plane pipeline (yz_pipe.cu) */
int mxb_demag_kmode(mxb_demag* d, int* kmode);
int mxb_demag_set_fast(mxb_demag* d, int fast);

/* ---- local operators and assembly (host buffers) ----------------------- */
/* ExchangeOperator / DmiOperator / AnisotropyOperator .__call__
 * (fields.py:112-127,142-151,161-163); term is one MXB_TERM_* bit */
int mxb_term_field(mxb_ctx* ctx, uint32_t term, int ghost_mode, const double* m, double* h);
/* PartitionedRHS.h_total_quiet / field_of (llg.py:170-175,193-194) */
int mxb_heff(mxb_ctx* ctx, mxb_demag* d, const mxb_terms* t, const mxb_bias* b,
             const double* m, double* h);
/* llg_rhs (llg.py:64-81) */
int mxb_llg_rhs(mxb_ctx* ctx, int precession, int damping, const double* m, const double* h,
                double* dmdt);
/* PartitionedRHS.rhs_total (llg.py:179-181) */
int mxb_rhs_total(mxb_ctx* ctx, mxb_demag* d, const mxb_terms* t, const mxb_bias* b,
                  const double* m, double* dmdt);
/* renormalize (grid.py:178-200), in place; on MXB_EDEAD *dead_flat holds the
 * first offending flat cell index */
int mxb_renormalize(mxb_ctx* ctx, double* m, int64_t* dead_flat);
/* mean_normalized (grid.py:203-214) */
int mxb_mean_normalized(mxb_ctx* ctx, const double* m, double out[3]);
/* energy_breakdown via PartitionedRHS.energies (fields.py:200-242,
 * llg.py:201-203): out = {e_demag, e_exch, e_anis, e_zeeman} */
int mxb_energies(mxb_ctx* ctx, mxb_demag* d, const mxb_terms* t, const mxb_bias* b,
                 const double* m, double out[4]);

/* ---- device-resident stepping (Simulation.run_until, llg.py:320-379) --- */
int mxb_state_set(mxb_ctx* ctx, const double* m);
int mxb_state_get(mxb_ctx* ctx, double* m);
/* per-stage uniform bias for the next nsteps (rows of 3 doubles, nsteps x
 * stages-per-step), or NULL to use the constant b->vec of mxb_run */
typedef struct mxb_run_args {
    int32_t method;            /* MXB_EULER / MXB_RK4 / MXB_MRI_KW3 */
    int32_t renorm_each_stage; /* IntegratorSpec.renorm_each_stage */
    double dt;
    int64_t nsteps;            /* steps to attempt in this call */
    double eq_tol;             /* < 0: no equilibrium stop */
    /* host rows of 3 doubles, one per right-hand-side evaluation that needs the
     * bias, in evaluation order (RK4: 4 per step at t, t+dt/2, t+dt/2, t+dt;
     * Euler: 1; MRI: the slow or fast evaluations of the partition holding the
     * bias), or NULL for the constant bias_vec */
    const double* stage_bias;
    const double* bias_field;  /* host (3,nz,ny,nx) static spatial bias or NULL */
    double bias_vec[3];        /* constant uniform bias (if stage_bias NULL) */
    uint32_t fast_mask;        /* MRI: terms in the fast partition (llg.py:41-47) */
    int32_t pad;
    double theta;              /* MRI: fast step ratio (IntegratorSpec.theta) */
    /* host (3,nz,ny,nx) bias fields, one per bias-reading evaluation in the
     * order of stage_bias (a callable t -> (3,nz,ny,nx) bias, reference
     * llg.py:92-96,154-164), or NULL; takes precedence over stage_bias */
    const double* stage_bias_fields;
} mxb_run_args;
typedef struct mxb_run_stats {
    int64_t steps_done;        /* committed steps */
    int32_t status;            /* MXB_OK / MXB_EQUILIBRATED / MXB_EBLOWUP / MXB_EDEAD */
    int32_t pad;
    double mean[3];            /* <m> after the last committed step */
    double residual;           /* max |<m>_k - <m>_{k-1}| of the last step */
    double drift;              /* blow-up: pre-renormalisation drift */
    int64_t dead_flat;
} mxb_run_stats;
/* seed the previous-step mean used by the residual (llg.py:341) */
int mxb_state_mean(mxb_ctx* ctx, double out[3]);
int mxb_run(mxb_ctx* ctx, mxb_demag* d, const mxb_terms* t, const mxb_run_args* a,
            mxb_run_stats* st);
/* energies of the resident state (sample rows, llg.py:314-317) */
int mxb_state_energies(mxb_ctx* ctx, mxb_demag* d, const mxb_terms* t, const mxb_bias* b,
                       double out[4]);

/* ---- z-slab decomposition across ranks ---------------------
 * Rank r of G owns planes [r*nz/G, (r+1)*nz/G).  One demag evaluation is
 *   x_forward (local rows -> per-destination kx chunks in `send`)
 *   all-to-all send -> recv            (caller: NCCL / torch.distributed)
 *   yz        (y, fused z*kernel, y inverse on this rank's kx chunk, in recv)
 *   all-to-all recv -> send            (caller)
 *   x_inverse (send -> local H rows).
 * With G = 1 send == recv and no exchange is needed. */
int mxb_demag_create_slab(const mxb_grid* global_grid, int device, int nranks, int rank,
                          mxb_demag** out);
/* info = {nz_local, z0, kx_chunk, kx_chunk_pitch, kx0, kx_count, block_elems, nranks};
 * block_elems = complex elements per all-to-all block */
int mxb_demag_slab_info(mxb_demag* d, int64_t info[8]);
int mxb_demag_slab_buffers(mxb_demag* d, void** send, void** recv);
/* complex elements per all-to-all block of the slab buffers (depends on the
 * spectra layout chosen by set_packed / build: call after them) */
int mxb_demag_slab_block(mxb_demag* d, int64_t* elems);
int mxb_demag_x_forward(mxb_demag* d, const double* m_dev);
int mxb_demag_yz(mxb_demag* d);
int mxb_demag_x_inverse(mxb_demag* d, double* h_dev);
/* run on an external CUDA stream (e.g. the stream NCCL collectives use) */
int mxb_demag_set_stream(mxb_demag* d, void* stream);
int mxb_ctx_set_stream(mxb_ctx* ctx, void* stream);

/* one fused stage kernel on caller-owned device buffers (the slab driver's
 * building block; the single-rank mxb_run enqueues the same kernels) */
typedef struct mxb_stage_io {
    const double *ys, *y, *hd, *k1;
    double *s, *out, *k1_out;
    const double *halo_lo, *halo_hi;     /* (3,ny,nx) neighbour planes or NULL */
    const double *hms_lo, *hms_hi, *hA_lo, *hA_hi;   /* their Ms / A (per-cell materials) */
    const double* bias_field;
    double bias[3];
    double c, dt6;                       /* stage coefficient, dt/6 */
    int32_t renorm;                      /* renormalise the stage state (RK stages 1-3) */
    int32_t pad;
} mxb_stage_io;
/* mode: 0 H_eff, 1 dM/dt, 2-5 RK4 stages 1-4, 6 Euler.  Modes 5/6 leave block
 * partials for mxb_step_partials_dev instead of committing the step. */
int mxb_stage_dev(mxb_ctx* ctx, int mode, const mxb_terms* t, const mxb_stage_io* io);
/* z-slab halos: copy the first and last local z planes of the three
 * components of f (3,nz,ny,nx, device) into the contiguous send buffers
 * lo/hi (3,ny,nx each) with one kernel on the context stream */
int mxb_pack_halo_planes(mxb_ctx* ctx, const double* f, double* lo, double* hi);
/* out8 = {sum mx/Ms, sum my/Ms, sum mz/Ms, 0 | max drift, halt code, -dead_flat, 0}
 * (first four summed over ranks, last four max-reduced over ranks by the caller) */
int mxb_step_partials_dev(mxb_ctx* ctx, double* out8_dev);
/* step bookkeeping with the global totals (blow-up, <m>, residual, equilibrium) */
int mxb_step_commit_dev(mxb_ctx* ctx, const double* totals8_dev);
int mxb_ctl_reset(mxb_ctx* ctx, const double prev_mean[3], int64_t n_magnetic, double eq_tol);
int mxb_ctl_get(mxb_ctx* ctx, mxb_run_stats* st);

/* ---- measurement helpers (bench.py) ------------------------------------ */
/* time `iters` demag evaluations of the resident state with CUDA events on
 * the context stream; returns the mean ms per evaluation and per pass */
int mxb_time_demag(mxb_ctx* ctx, mxb_demag* d, int iters, double* ms_eval, double* ms_pass5);
/* time `nsteps` fused RK4 steps of the resident state; ms_stencil is the
 * summed time of the fused stage kernels only */
int mxb_time_steps(mxb_ctx* ctx, mxb_demag* d, const mxb_terms* t, double dt, int nsteps,
                   const double bias[3], double* ms_total, double* ms_stencil,
                   int64_t* launches);
/* cuFFT comparison of the same demag evaluation (timed comparison only,
 * never on the product path) */
int mxb_time_demag_cufft(mxb_demag* d, int iters, double* ms_eval);

/* ---- pinned host memory (e2e measurements) ---------------------------- */
int mxb_host_alloc(size_t bytes, void** p);
int mxb_host_free(void* p);


/* ---- FNO demag surrogate (fno.py:228-447): thin film, channels-first (3, ny, nx) ----
 * params (float64), in this order:
 *   lift.weight (width,3), lift.bias (width),
 *   for k = 0..3: block{k}.spectral.pos (width,width,m1,m2) complex as (re,im) pairs,
 *                 block{k}.spectral.neg (same), block{k}.local.weight (width,width),
 *                 block{k}.local.bias (width),
 *   proj.weight (3,width), proj.bias (3), norm.in_mean, norm.in_std, norm.out_mean,
 *   norm.out_std (3 each).
 * activation: 0 GELU (erf form), 1 ReLU.  Replaces FnoModel.infer (fno.py:372-394) and
 * FnoDemag.field (fno.py:445-447). */
typedef struct mxb_fno mxb_fno;
int mxb_fno_create(int device, int width, int m1, int m2, int ny, int nx, int activation,
                   const double* params, mxb_fno** out);
void mxb_fno_destroy(mxb_fno* f);
/* host (3, ny, nx) -> host (3, ny, nx) */
int mxb_fno_infer(mxb_fno* f, const double* x, double* y);
/* device pointers, on the model's stream (synchronise before reading y) */
int mxb_fno_infer_dev(mxb_fno* f, const double* x, double* y);
/* a demag handle whose field is the surrogate's forward pass (FnoDemag.field,
 * fno.py:427-447): usable wherever an mxb_demag is, including mxb_run, where
 * the forward pass runs inside the fused device step.  The film must be the
 * model's H x W with nz = 1; f must outlive the handle. */
int mxb_demag_create_fno(const mxb_grid* g, int device, mxb_fno* f, mxb_demag** out);
/* spectral_conv (fno.py:228-255) of host (channels, ny, nx); w_pos/w_neg
 * (channels, channels, m1, m2) complex as (re, im) pairs */
int mxb_fno_spectral_conv(int device, int channels, int ny, int nx, int m1, int m2,
                          const double* w_pos, const double* w_neg, const double* x, double* y);

#ifdef __cplusplus
}
#endif
#endif /* MAGNEX_B200_H */
