/*
 * hlf_b200.h -- C-ABI of the B200-native Hermite-leapfrog hot path
 * (arXiv 1808.10481).  Plain pointers and sizes only; no CUDA or torch types.
 *
 * The reference (/root/reference/proj) is a C++20 library with no plugin
 * registry or FFI; its boundary for this path is the C++ API in
 * proj/include/hlf.  Each entry point below replaces one piece of it:
 *
 *   hlf_build_interp_operator  <- hlf::build_interp_operator    interpolation.hpp:22, interpolation.cpp:21-51
 *   hlf_create                 <- hlf::Stepper1d::Stepper1d     stepper1d.hpp:68, stepper1d.cpp:93-111
 *                                 (+ Grid1d/Grid2d::over grid.hpp:12,29; SchemeConfig::validate config.hpp:37)
 *   hlf_set_field/get_field    <- State1d::p / State1d::v       stepper1d.hpp:49-52 (public, caller-owned jets)
 *   hlf_set_times/get_times    <- State1d::t_p, t_v, dt         stepper1d.hpp:50
 *   hlf_set_dt                 <- `st.dt = -dt` (time reversal) tests/test_stepper1d.cpp:288
 *   hlf_set_coeff              <- Stepper1d::ap_prim_/ap_dual_  stepper1d.cpp:103-110 (coefficient jets)
 *   hlf_l2_error_separable     <- l2_error_1d / l2_error_2d      analysis.cpp:241-285 (on the device)
 *   hlf_energy_1d              <- conserved_q / conserved_r      analysis.cpp:221-239 (on the device)
 *   hlf_set_forcing            <- Stepper1d::forcing_at / Problem1d::forcing  stepper1d.cpp:113-119, problem.hpp:27-29
 *   hlf_advance_p              <- Stepper1d::advance_p          stepper1d.hpp:72, stepper1d.cpp:147-156
 *   hlf_advance_v              <- Stepper1d::advance_v          stepper1d.hpp:73, stepper1d.cpp:158-166
 *   hlf_step                   <- Stepper1d::step_system        stepper1d.hpp:74, stepper1d.cpp:168-172
 *   hlf_advance_n              <- the caller's step loop        tests/test_stepper1d.cpp:38
 *   hlf_plan_steps             <- step_count + dt = T / n       config.cpp:34-38, tests/test_stepper1d.cpp:33-35
 *   hlf_advance_to             <- the caller loop up to T       tests/test_stepper1d.cpp:33-38
 *   hlf_poll_finite            <- Stepper1d::check_finite       stepper1d.cpp:121-129
 *   status codes               <- ConfigError, InstabilityError config.hpp:15-24, std::invalid_argument
 *
 * Fields: 0 = p on the primary grid; 1..d = velocity components on the dual
 * grid (Problem2d field order p, v, u: problem.hpp:41-46).  Host buffers are
 * AoS [node][coef]: node (ix, iy, iz) -> ((ix*Ny)+iy)*Nz+iz, coefficient
 * (a, b, c) -> (a*(m+1)+b)*(m+1)+c -- both x-major like TensorJet::at
 * (jet.hpp:43-44) and PiecewiseTensor::cell (interpolation.hpp:50-52).
 * Primary grid: K nodes per periodic axis, K+1 per reflective axis (walls on
 * primary lines); dual grid: K per axis.
 */
#ifndef HLF_B200_H
#define HLF_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum hlf_status {
  HLF_OK = 0,
  HLF_CONFIG_ERROR = 1,     /* hlf::ConfigError        (config.hpp:15-17) */
  HLF_INSTABILITY = 2,      /* hlf::InstabilityError   (config.hpp:19-24) */
  HLF_INVALID_ARGUMENT = 3, /* std::invalid_argument   (interpolation.cpp:65-66) */
  HLF_CUDA_ERROR = 4,
  HLF_NCCL_ERROR = 5
} hlf_status;

enum { HLF_PERIODIC = 0, HLF_REFLECTIVE = 1 }; /* hlf::Boundary (config.hpp:10) */
enum { HLF_PRIMARY = 0, HLF_DUAL = 1 };

/* Version of this ABI; bump on any signature change. */
#define HLF_B200_ABI_VERSION 1

typedef struct hlf_solver hlf_solver; /* opaque */

typedef struct hlf_desc {
  int dim;            /* 1, 2 or 3 */
  int m;              /* order, [0, SchemeConfig::m_cap = 8]; device kernels: d<=2 any m, d=3 m<=4 */
  int K[3];           /* cells per axis (unused axes ignored); K >= 2 (grid.cpp:10) */
  double x_min[3];    /* lower domain corner (primary node 0) */
  double h;           /* common spacing (Grid1d::h; Grid2d is square, grid.cpp:25-26) */
  int boundary[3];    /* HLF_PERIODIC / HLF_REFLECTIVE per axis */
  double ap, av;      /* constant coefficients: p_t = ap div v, v_t = av grad p (problem.hpp:11-14,36-38) */
  int variable_ap;    /* 1: per-node ap jets (e.g. -c^2(x)) are supplied with hlf_set_coeff */
  const double* M;    /* (2m+2)^2 row-major interpolation operator; NULL = build it here */
  int device;         /* CUDA ordinal */
  void* stream;       /* cudaStream_t to launch on; NULL = the library's own stream */
  int z_slab;         /* 1: z is one slab of a periodic decomposition; z halos come
                         from hlf_halo_* instead of the local wrap */
  int scheme;         /* HLF_SCHEME_*: the reference Stepper1d's three time schemes
                         (config.hpp:9); the alternatives are 1D, periodic, constant
                         coefficients */
} hlf_desc;

/* time schemes (hlf::Variant, config.hpp:9):
   LEAPFROG     staggered Hermite-leapfrog (advance_p / advance_v / step_system,
                stepper1d.cpp:147-172): field 0 = p on the primary grid, 1..d = v on the dual grid;
   MODIFIED     step_modified (stepper1d.cpp:191-232): every field on both grids:
                field 0 = p primary (t), 1 = v dual (t + dt/2), 2 = v primary (t), 3 = p dual (t + dt/2);
   DUAL_HERMITE step_dual_hermite (stepper1d.cpp:249-272), both fields co-located:
                field 0 = p primary, 2 = v primary (t); fields 1, 3 are the midpoint scratch
                on the dual grid.
   hlf_step / hlf_advance_n run the selected scheme; the time stamp t is t_p
   (hlf_get_times), t_v = t_p + dt/2 (MODIFIED) or t_p (DUAL_HERMITE). */
#define HLF_SCHEME_LEAPFROG 0
#define HLF_SCHEME_MODIFIED 1
#define HLF_SCHEME_DUAL_HERMITE 2
/* MODIFIED_ADVECTION  the single-field branch of step_modified (n_fields == 1,
                stepper1d.cpp:205-209, ck_advection :40-52): u_t = ap u_x on both
                grids: field 0 = u primary (t), field 1 = u dual (t + dt/2) */
#define HLF_SCHEME_MODIFIED_ADVECTION 3

/* --- interpolation operator ---------------------------------------------- */
/* M = A^{-1} (row-major, (2m+2)^2) and its 1-norm condition; HLF_CONFIG_ERROR for m outside [0, 8] */
hlf_status hlf_build_interp_operator(int m, double* M_out, double* condition_out);

/* --- lifetime ------------------------------------------------------------ */
hlf_status hlf_create(const hlf_desc* desc, hlf_solver** out);
void hlf_destroy(hlf_solver* s);
/* message of the last failing call on this handle (or of the last failing
   hlf_create on this thread when s is NULL) */
const char* hlf_last_error(const hlf_solver* s);
int hlf_abi_version(void);

/* --- geometry ------------------------------------------------------------ */
int64_t hlf_num_nodes(const hlf_solver* s, int grid);     /* real nodes (no ghosts) */
int hlf_num_coeffs(const hlf_solver* s);                  /* (m+1)^d */

/* --- staggered state ----------------------------------------------------- */
hlf_status hlf_set_field(hlf_solver* s, int field, const double* host_aos);
hlf_status hlf_get_field(hlf_solver* s, int field, double* host_aos);
/* per-node ap jets, (2m+2)^d entries per node (x-major), for grid HLF_PRIMARY / HLF_DUAL */
hlf_status hlf_set_coeff(hlf_solver* s, int grid, const double* host_jets);
/* ap = -(c0 + c1 prod_ax sin(w[ax] x_ax + phase[ax])) at every node of both
   grids (ap = -c^2 with a separable c^2, e.g. the SURVEY.md sec. 8(d) config 3
   speed c^2 = 1 + sin(pi x) sin(pi y) / 2 and its 3D extension); av stays the
   scalar desc.av.  Replaces hlf_set_coeff for this family: the jets are the
   reference's scaled sin jets (sin_jet, jet.cpp:65-74) in outer product.  In
   3D with m <= 3 they are generated inside the kernel (var3d: no stored
   coefficient grids, 24 B per DOF-update); otherwise they are written to the
   per-node jet storage on the device.  Needs desc.variable_ap = 1. */
hlf_status hlf_set_coeff_separable(hlf_solver* s, double c0, double c1, const double* w, const double* phase);
/* Forcing (ck_recurrence_variable's z, stepper1d.cpp:22-38): the table for
   the NEXT half step that updates `grid` (HLF_PRIMARY: hlf_advance_p, evaluated
   by the reference at (primary x_j, t_v); HLF_DUAL: hlf_advance_v, at (dual x_j,
   t_p after the pressure half step)).  Host AoS [node][r][e], r = 0..2m
   (levels z(r) of forcing_at), e = the n^d entries of the scaled tensor jet
   (x-major, n = 2m+2; d = 1: the reference's Jet), i.e. (2m+1) n^d doubles
   per node; z(r) is added to every level of the P table (p_t = ap div v + f).
   Once a table has been set the solver is in forcing mode: every half step
   needs a fresh table for its grid (HLF_CONFIG_ERROR otherwise, so
   hlf_advance_n runs at most one step); hlf_clear_forcing leaves forcing
   mode.  Leapfrog scheme; d > 1 runs the faithful generic kernel (separable
   on-the-fly coefficients are expanded to stored jets). */
hlf_status hlf_set_forcing(hlf_solver* s, int grid, const double* host_table);
hlf_status hlf_clear_forcing(hlf_solver* s);
hlf_status hlf_set_times(hlf_solver* s, double t_p, double t_v, double dt);
hlf_status hlf_get_times(const hlf_solver* s, double* t_p, double* t_v, double* dt);
hlf_status hlf_set_dt(hlf_solver* s, double dt);

/* --- stepping (asynchronous on the solver's stream) ---------------------- */
hlf_status hlf_advance_p(hlf_solver* s);
hlf_status hlf_advance_v(hlf_solver* s);
/* the same half steps recording non-finite values under step_index (no sync);
   for callers that interleave halo exchanges (z slabs) */
hlf_status hlf_advance_p_indexed(hlf_solver* s, int step_index);
hlf_status hlf_advance_v_indexed(hlf_solver* s, int step_index);
/* One half step over target layers [z_begin, z_end) only (3D; half 0 =
   pressure, 1 = velocity), without advancing the time stamp: a z-slab rank
   updates its interior layers while the halo layer is in flight and the
   boundary layer after it lands, then calls hlf_commit_half once.  Same
   arithmetic as the full launch (advance_p/advance_v, stepper1d.cpp:147-166,
   restricted to a layer range). */
hlf_status hlf_advance_layers(hlf_solver* s, int half, int step_index, int z_begin, int z_end);
/* t_p (half 0) or t_v (half 1) += dt, as advance_p/advance_v do (stepper1d.cpp:155,165) */
hlf_status hlf_commit_half(hlf_solver* s, int half);
/* advance_p, advance_v, finite check: HLF_INSTABILITY (synchronous) if the
   state became non-finite; message "solution became non-finite at step N" */
hlf_status hlf_step(hlf_solver* s, int step_index);
/* n steps indexed first..first+n-1; the finite flag is read once at the end and
   the first offending step index is reported through HLF_INSTABILITY */
hlf_status hlf_advance_n(hlf_solver* s, int n, int first_step);
/* The caller's step rule (step_count, config.hpp:47 / config.cpp:34-38, and
   tests/test_stepper1d.cpp:33-35): n = ceil(T / dt_nominal), dt = T / n.
   HLF_CONFIG_ERROR for T <= 0 or dt_nominal <= 0, as step_count throws. */
hlf_status hlf_plan_steps(double T, double dt_nominal, int* n_out, double* dt_out);
/* Advance from the current t_p to T in steps of the current dt (the reference
   has no advance-to; this is its caller loop `for i < nsteps: step_system(st,
   i)`, test_stepper1d.cpp:38): n = (T - t_p) / dt steps indexed first_step..,
   through hlf_advance_n.  dt is fixed by the staggered initialisation
   (init_leapfrog sets t_v = t0 + dt/2, stepper1d.cpp:137), so it must divide
   T - t_p to 1e-9 relative (HLF_CONFIG_ERROR otherwise; use hlf_plan_steps to
   pick dt before initialising).  Negative dt runs backwards to T < t_p.
   *steps_out = the steps run. */
hlf_status hlf_advance_to(hlf_solver* s, double T, int first_step, int* steps_out);
/* -1 when the state stayed finite, else the first non-finite step index */
/* hlf_advance_n replays runs of `steps` leapfrog steps as one captured CUDA
   graph (launch overhead dominates small grids); 0 = launch every kernel
   directly.  Default 32; used when n >= 2 * steps. */
hlf_status hlf_set_graph_steps(hlf_solver* s, int steps);
hlf_status hlf_poll_finite(hlf_solver* s, int* first_bad_step);
hlf_status hlf_clear_finite(hlf_solver* s);
hlf_status hlf_synchronize(hlf_solver* s);

/* --- device-resident data (no host copies) ------------------------------- */
/* device base of a field, SoA [layer][coef][y][x] (layer includes z ghosts:
   p layer index = z, v layer index = z + 1); strides in elements */
hlf_status hlf_field_device(hlf_solver* s, int field, double** dev_ptr, int64_t* layer_stride,
                            int64_t* coef_stride, int* layers);
/* field += amp * prod_ax sin(w[ax] x_ax + phase[ax]) as exact scaled jets at the
   field's nodes (sin_jet, jet.cpp:65-74), computed on the device */
hlf_status hlf_fill_separable(hlf_solver* s, int field, double amp, const double* w,
                              const double* phase);
hlf_status hlf_zero_field(hlf_solver* s, int field);
/* On-device error accessor (the nodal counterpart of l2_error_1d/2d,
   analysis.cpp:241-285, for separable trig data as filled by
   hlf_fill_separable): rms over the field's nodes of value - exact, and the
   max over nodes and scaled jet coefficients of |jet - exact jet|.
   Synchronous; no state download (convergence sweeps stay on the device). */
hlf_status hlf_error_separable(hlf_solver* s, int field, double amp, const double* w, const double* phase,
                               double* rms_value, double* max_jet);
/* Gauss-quadrature L2 error of `field` against amp prod_ax sin(w[ax] x_ax +
   phase[ax]): the device counterpart of l2_error_1d / l2_error_2d
   (analysis.cpp:241-285) in d = 1..3 -- cells centred on the other grid's
   nodes, the cell's Hermite interpolant (reconstruct_cell_*) evaluated at the
   (2m+2)-point Gauss rule per axis.  Dual-grid fields need periodic axes (the
   reference clips wall cells); no z slabs. */
hlf_status hlf_l2_error_separable(hlf_solver* s, int field, double amp, const double* w, const double* phase,
                                  double* l2);
/* Discrete energy of the 1D periodic leapfrog on the device: kind 0 =
   conserved_q(p, v_behind, c, dt) (after hlf_advance_p), kind 1 =
   conserved_r(v_ahead, p, c, dt) (after hlf_advance_v), analysis.cpp:221-239,
   with the solver's current fields and dt. */
hlf_status hlf_energy_1d(hlf_solver* s, int kind, double c, double* energy);

/* --- z-slab halos (multi-GPU; z_slab = 1) -------------------------------- */
/* The velocity half step reads p layer Kz (the next rank's layer 0); the
   pressure half step reads v layer -1 (the previous rank's layer Kz-1).
   hlf_halo_send_ptr gives the device pointer of the layer this rank must
   send, hlf_halo_recv_ptr where the received layer must land, both
   layer_stride doubles long.  kind 0 = p halo (before advance_v), 1 = v halo
   of component c (before advance_p). */
hlf_status hlf_halo_send_ptr(hlf_solver* s, int kind, int comp, double** dev_ptr, int64_t* count);
hlf_status hlf_halo_recv_ptr(hlf_solver* s, int kind, int comp, double** dev_ptr, int64_t* count);

/* --- multi-GPU z slabs from one C++ host process ------------------------- */
/* A periodic 3D domain (global desc; K[2] cells along z) split into n z slabs
   of K[2]/n layers, slab r on devices[r]; each half step
   exchanges one layer with the ring neighbours, overlapped with the interior
   layers (the same arithmetic as one solver over the whole domain).
   transport: HLF_TRANSPORT_NCCL (ncclSend/ncclRecv over an ncclCommInitAll
   clique; one device per slab), HLF_TRANSPORT_COPY (cudaMemcpyPeerAsync; also
   several slabs on one device), HLF_TRANSPORT_AUTO (NCCL when the devices are
   distinct and libnccl.so.2 loads, else COPY).  The reference has no
   multi-process or multi-GPU code; this replaces the
   caller loop over step_system for a sharded domain. */
typedef struct hlf_slab_group hlf_slab_group; /* opaque */
enum { HLF_TRANSPORT_AUTO = 0, HLF_TRANSPORT_NCCL = 1, HLF_TRANSPORT_COPY = 2 };
hlf_status hlf_slabs_create(const hlf_desc* global, int n, const int* devices, int transport, hlf_slab_group** out);
void hlf_slabs_destroy(hlf_slab_group* g);
const char* hlf_slabs_last_error(const hlf_slab_group* g);
int hlf_slabs_count(const hlf_slab_group* g);
int hlf_slabs_transport(const hlf_slab_group* g);
/* slab r's solver (fields, accessors; AoS host data of that slab only) */
hlf_solver* hlf_slabs_solver(hlf_slab_group* g, int r);
hlf_status hlf_slabs_set_times(hlf_slab_group* g, double t_p, double t_v, double dt);
/* steps indexed first_step.. on every slab; HLF_INSTABILITY with the first
   non-finite step over all slabs */
hlf_status hlf_slabs_advance_n(hlf_slab_group* g, int steps, int first_step);
hlf_status hlf_slabs_synchronize(hlf_slab_group* g);

/* the cudaStream_t the solver launches on (as void*) */
void* hlf_get_stream(const hlf_solver* s);

/* number of kernels this solver has launched (for launch accounting) */
int64_t hlf_launch_count(const hlf_solver* s);
/* Path accounting of the tiled 2D/3D kernels (tests): when enabled (and reset
   by enabling again) every CTA of a tiled launch counts itself, per half step
   kind (0 = velocity, 1 = pressure): out6 = [vel CTAs, vel CTAs whose source
   rows arrived by TMA boxes, vel CTAs whose targets arrived by TMA boxes, the
   same three for the pressure launches].  Off by default (no cost). */
hlf_status hlf_enable_path_counters(hlf_solver* s, int on);
/* Per-launch device times: runs `steps` leapfrog steps (indexed first_step..,
   advancing the state and the time stamps like hlf_step without the finite
   check) with CUDA events on the solver's stream around every kernel of each
   half step, synchronising after each half step.  ms_out[0..2] = mean ms of
   the velocity half step's launches 0..2, ms_out[3..5] = the pressure half
   step's; launches_out[0..1] = launches per velocity / pressure half step. */
hlf_status hlf_time_launches(hlf_solver* s, int steps, int first_step, double* ms_out, int* launches_out);
hlf_status hlf_read_path_counters(hlf_solver* s, int64_t* out6);
/* kernel variant the next half steps use: 0 generic, 1 tiled 3D */
int hlf_kernel_variant(const hlf_solver* s);
hlf_status hlf_set_kernel_variant(hlf_solver* s, int variant);

#ifdef __cplusplus
}
#endif

#endif /* HLF_B200_H */
