/*
 * lbm_b200.h - C-ABI of the B200-native lattice Boltzmann hot path.
 *
 * This is the drop-in boundary for the reference's kernel slot
 * (blocksim._kernels.impl, pkg/src/blocksim/_kernels/__init__.py:10-37) and
 * for the sweep that drives it (lbm/sweep.py:93-151).  Every entry point
 * takes raw device pointers, explicit geometry and a cudaStream_t passed as
 * void*, returns 0 on success and a negative status otherwise
 * (lbm_last_error() then holds the message).  No C++ exception crosses the
 * boundary and nothing here allocates persistent device memory: the caller
 * (Python/torch) owns every buffer.
 *
 * Reference interfaces replaced (file:line under /root/reference/pkg/src/blocksim):
 *   lbm_fused_step      impl.collide (_kernels/_core_py.py:70-200)
 *                       + impl.stream_pull (_core_py.py:203-218)
 *                       + BoundaryHandling.apply (lbm/boundary.py:154-195),
 *                       fused as pull -> bounce-back -> collide (G-form).
 *   lbm_collide_only    impl.collide on a freshly written R-form field
 *                       (first half of the first stream_collide, sweep.py:147).
 *   lbm_stream_only     impl.stream_pull + BoundaryHandling.apply without the
 *                       following collide: turns the stored G-form back into
 *                       the reference's R-form for readout (sweep.py:148-150).
 *   lbm_moments         macroscopic / macroscopic_fields
 *                       (lbm/collision.py:157-184, lbm/sweep.py:154-176).
 *   lbm_fill_equilibrium  fill_equilibrium -> equilibrium
 *                       (lbm/sweep.py:51-76, lbm/collision.py:138-154).
 *   lbm_pack_rform / lbm_unpack_rform  Field.raw <-> device layout
 *                       (field/core.py:34-70; "fzyx" raw shape (q,Z,Y,X)).
 *   lbm_build_cellmask  build_index_lists + sweep-time flag validation
 *                       (lbm/boundary.py:48-97, lbm/sweep.py:124-136).
 *   lbm_build_linkbits / lbm_fused_step_bits  the same link lists as one
 *                       bit per cell for NoSlip-only lattices (ABI 7).
 *   lbm_map_spheres     map_bodies' voxeliser (coupling/mapping.py:100-140).
 *   lbm_refresh_fluid_mask  the per-sweep fluid mask of flags edited after
 *                       freeze() (lbm/sweep.py:124-136; links stay frozen).
 *   lbm_collide_cells / lbm_equilibrium_cells / lbm_macroscopic_cells
 *                       collide_pdfs / equilibrium / macroscopic on flat
 *                       (n, q) populations (lbm/collision.py:138-184,245-261).
 *   lbm_build_moving_masks  map_bodies' link enumeration on the device
 *                       (coupling/mapping.py:133-150) for moving_boundary_sweep
 *                       (coupling/sweep.py:45-155; the wall rule itself is
 *                       fused into lbm_fused_step through lbm_params_t.moving).
 *   lbm_fused_step_peer lbm_fused_step with the per-step z-face exchange
 *                       (field/ghost.py:202-264) fused in: boundary planes
 *                       store their crossing directions into the
 *                       neighbour's ghost plane (peer HBM over NVLink);
 *                       lbm_stream_signal / lbm_stream_wait order the phases.
 *   lbm_slot_apply_links  BoundaryHandling.apply on host views (boundary.py:154-195).
 *   lbm_slot_collide / lbm_slot_stream_pull  the kernel slot itself,
 *                       impl.collide / impl.stream_pull
 *                       (_kernels/__init__.py:10-37, _core_py.py:70-218) on
 *                       dense (z, y, x, q) arrays, ghost ring included - the
 *                       per-call "b200" backend of blocksim._kernels.
 *   lbm_bind_params     re-binds a parameter block's device-side state (MRT
 *                       constant tables) before a captured CUDA graph replays.
 *   lbm_fill_equilibrium_planes / lbm_collide_only_planes / lbm_moments_planes
 *   lbm_fill_collide_planes
 *                       the same three steps on a range of z-planes, for a
 *                       pipelined job (fill_equilibrium -> K x stream_collide
 *                       -> macroscopic, sweep.py:51-183) whose host<->device
 *                       copies overlap the sweeps plane chunk by plane chunk.
 *   lbm_face_span       geometry of the per-step z-face ghost exchange
 *                       (field/ghost.py:112-173,202-264), restricted to the
 *                       PDF directions that cross the face.
 *
 * Device PDF layout ("z-q-y-x", one box per rank, one ghost layer on every
 * side):  direction i of cell (z, y, x) lives at
 *     ((z+1) * q + slot) * plane + (y+1) * pitch + xoff + x
 * with plane = (ny+2) * pitch and slot = lbm_slot_of(q, i).  Direction i is stored in slot
 * lbm_slot_of(q, i): slots are grouped by c_z (-1, 0, +1), so the directions
 * that cross a z-face form ONE contiguous run per z-plane and the halo can be
 * stored straight into the neighbour's ghost plane by the boundary-plane
 * kernel (lbm_fused_step_peer) or sent out of / into the field by NCCL
 * without a pack kernel.
 * real_bytes == 8 stores f in fp64 and computes in fp64 (bitwise reference
 * arithmetic); real_bytes == 4 stores the centred populations (f - w_i) in
 * fp32 and computes in fp32 registers on the centred values (FMA allowed;
 * checked against the fp64 path at 1e-5 relative).
 */
#ifndef LBM_B200_H
#define LBM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LBM_B200_ABI_VERSION 8

/* status codes */
#define LBM_OK 0
#define LBM_EINVAL -1    /* bad argument (maps to ValidationError) */
#define LBM_ECUDA -2     /* CUDA launch/runtime failure */
#define LBM_ENUMERIC -3  /* non-positive density (maps to NumericsError) */
#define LBM_EFLAGS -4    /* flag validation failed (maps to ValidationError) */

/* z-face modes of a rank's box */
#define LBM_ZFACE_GHOST 0 /* domain face, non-periodic: ghost keeps its init value */
#define LBM_ZFACE_HALO 1  /* ghost plane filled by the per-step exchange       */
#define LBM_ZFACE_WRAP 2  /* periodic and owned by this rank: index wrap       */

/* collision models (SRT.mode/TRT.mode/MRT.mode, lbm/collision.py:54,71,103) */
#define LBM_SRT 0
#define LBM_TRT 1
#define LBM_MRT 2
/* SRT with a per-cell rate field (SRT(omega_field=key), lbm/sweep.py:111-146,
 * _core_py.py:130-136): rem = 1 - omega(x), hw = 1 - 0.5 omega(x) per cell,
 * omega(x) read from lbm_params_t.omega_cells */
#define LBM_SRT_FIELD 3
/* force models (Guo.mode / SimpleShift.mode, lbm/collision.py:115,128) */
#define LBM_FORCE_NONE 0
#define LBM_FORCE_GUO 1
#define LBM_FORCE_SHIFT 2
#define LBM_FORCE_GUO_X 3 /* Guo with F = (fx, 0, 0): same values, fewer flops */

/* cell-mask bits written by lbm_build_cellmask */
#define LBM_MASK_FLUID 0x1u        /* bit 0: cell is collided              */
#define LBM_MASK_UBB 0x80000000u   /* bit 31: some link of the cell is UBB */
#define LBM_MASK_PRESSURE 0x40000000u /* bit 30: some link is Pressure      */
#define LBM_MASK_MOVING 0x20000000u   /* bit 29: some link is a moving-body wall */
/* bits 1..q-1: pulled direction i comes from a boundary cell, i.e. the
 * reference link (x, opp(i)) exists (boundary.py:91-95). */

typedef struct lbm_grid {
    int q;          /* 9, 19 or 27                                  */
    int real_bytes; /* 8 (fp64) or 4 (fp32 storage and arithmetic on f - w_i) */
    int nx, ny, nz; /* interior cells of this rank's box            */
    int pitch;      /* elements per x row (>= xoff + nx + 1)        */
    int xoff;       /* element offset of interior x = 0 in a row (>= 1) */
    int wrap_x;     /* 1: x periodic (index wrap), 0: ghost column  */
    int wrap_y;     /* 1: y periodic (index wrap), 0: ghost row     */
    int zface_lo;   /* LBM_ZFACE_* for the z = -1 side              */
    int zface_hi;   /* LBM_ZFACE_* for the z = nz side              */
} lbm_grid_t;

/* Moving-body walls of one sweep (coupling/sweep.py:45-155): links from
 * fluid cells to body-covered cells bounce back with the body's surface
 * velocity at the link midpoint, R[x, opp(i)] = G[x, i] - ((6 w_i) rho0)
 * (c_i . u_w), u_w = v + omega x r, and hand the momentum
 * (2 G[x, i] - ((6 w_i) rho0)(c_i . u_w)) c_i (and its torque) to the body.
 * All pointers are DEVICE pointers; arrays cover this rank's box. */
typedef struct lbm_moving {
    const int32_t* owner;      /* (nz+2, ny+2, nx+2) ghost-inclusive: body slot covering the
                                  cell, -1 where free                                       */
    const uint32_t* linkmask;  /* (nz, ny, nx): pulled directions j whose source x - c_j is
                                  covered (from lbm_build_moving_masks)                     */
    const double* bodies;      /* (n_blocks * n_slots, 9): position, linear velocity, angular
                                  velocity of the body copy each block holds (block-major)   */
    const double* cell0;       /* (n_blocks, 3): centre of each block's first interior cell */
    double* forces;            /* (n_blocks * n_slots, 6): force, torque accumulators (added
                                  to; NULL = do not accumulate)                             */
    int n_slots;               /* body slots                                                */
    int blocks[3];             /* block grid of the box (x, y, z)                           */
    int block_cells[3];        /* cells per block (x, y, z)                                 */
    double rho0;               /* reference density                                         */
} lbm_moving_t;

typedef struct lbm_params {
    int model;       /* LBM_SRT / LBM_TRT / LBM_MRT                    */
    int force_mode;  /* LBM_FORCE_*                                    */
    /* SRT (collision.py:130-136): rem = 1 - omega, hw = 1 - 0.5 omega  */
    double omega, rem, hw;
    /* TRT (collision.py:137-148,184-190): he_half = (1 - 0.5 w_e) * 0.5 */
    double omega_e, omega_o, he_half, ho_half;
    /* force: half_f = 0.5 * F (Guo) or tau * F (SimpleShift)           */
    double fx, fy, fz;
    double shift_fx, shift_fy, shift_fz;
    /* UBB link constant per link direction k (the direction pointing INTO
     * the wall): ((6 w_k) rho_0) (c_k . u_w) (boundary.py:165-170)     */
    double ubb[27];
    /* Pressure link constant per link direction k: (2 w_k) rho_w
     * (boundary.py:171-195)                                             */
    double pressure[27];
    /* MRT tables, host pointer, row-major fp64 (collision.py:150-169,
     * 192-197): M[q*q], Minv[q*q], S[q], G[q*q] (G only for Guo).  NULL
     * unless model == LBM_MRT.                                          */
    const double* mrt;
    /* LBM_SRT_FIELD: DEVICE pointer to the per-cell rates of this rank's box
     * interior, (nz, ny, nx) fp64, same cell order as the cell mask.  NULL
     * otherwise.  (ABI 2) */
    const double* omega_cells;
    /* moving-body walls for this sweep, or NULL (ABI 3) */
    const lbm_moving_t* moving;
} lbm_params_t;

/* ------------------------------------------------------------- metadata */
int lbm_abi_version(void);
/* sizeof(lbm_grid_t) (which = 0) / sizeof(lbm_params_t) (which = 1) /
 * sizeof(lbm_moving_t) (which = 2), so a binding can verify its struct
 * mirror; 0 for other values */
size_t lbm_struct_size(int which);
const char* lbm_last_error(void);
/* storage slot of reference direction i (layout above); -1 on bad input */
int lbm_slot_of(int q, int i);
/* bytes of one PDF field in the device layout for this grid */
int64_t lbm_field_elems(const lbm_grid_t* g);
/* Span of the z-face exchange, in elements from the field base.
 * face: 0 = low z face, 1 = high z face.
 * recv: ghost-plane run this rank receives on that face (directions whose
 *       c_z points into the box);
 * send: interior boundary-plane run this rank sends through that face
 *       (directions whose c_z points out of the box, i.e. into the peer). */
int lbm_face_span(const lbm_grid_t* g, int face, int64_t* send_off,
                  int64_t* recv_off, int64_t* count);

/* ------------------------------------------------------------ hot path */
/* One fused step on interior planes [z_begin, z_end): pull from G_n (src,
 * ghosts valid), bounce-back on masked links, collide fluid cells, store
 * G_{n+1} into dst.  cellmask: (nz, ny, nx) uint32 from lbm_build_cellmask;
 * typemask: (nz, ny, nx, 2) uint32 - word 0 UBB link bits, word 1 Pressure
 * link bits - only read where LBM_MASK_UBB / LBM_MASK_PRESSURE is set.
 * cellmask = typemask = NULL: every cell is fluid and has no link (a
 * periodic domain without boundary handling); no mask bytes are read.
 * typemask = NULL with a cellmask: no cell carries LBM_MASK_UBB /
 * LBM_MASK_PRESSURE (NoSlip-only links); the typed corrections are compiled
 * out of the launched kernel (ABI 5). */
int lbm_fused_step(const lbm_grid_t* g, const lbm_params_t* p,
                   const void* src, void* dst, const uint32_t* cellmask,
                   const uint32_t* typemask, int z_begin, int z_end,
                   void* stream);

/* lbm_fused_step reading the link-bit map (ABI 7) instead of the 4 B/cell
 * cell mask where the launched kernel can: linkbits from lbm_build_linkbits
 * (0 mismatches) for the same cellmask, typemask = NULL, no moving-body
 * walls.  Other launches (and linkbits = NULL) read cellmask as
 * lbm_fused_step does, so the result never depends on the choice.
 * LBM_B200_LINKBITS=0 in the environment forces the cell mask (A/B runs). */
int lbm_fused_step_bits(const lbm_grid_t* g, const lbm_params_t* p,
                        const void* src, void* dst, const uint32_t* cellmask,
                        const uint32_t* typemask, const uint64_t* linkbits,
                        int z_begin, int z_end, void* stream);

/* lbm_fused_step plus the fused z-face halo (ABI 4): the plane z = 0 also
 * stores its c_z = -1 directions into peer_lo, the plane z = nz-1 its
 * c_z = +1 directions into peer_hi, at the same (slot, y, x) offsets.  A peer
 * pointer is the z-block of the neighbour's receiving ghost plane (its field
 * base + lbm_ghost_block_offset(neighbour grid, face facing us)); it may live
 * in this GPU's memory or in a peer GPU's HBM mapped through CUDA IPC over
 * NVLink.  NULL: that face is not written.  Replaces the per-step
 * exchange_ghosts of stream_collide (lbm/sweep.py:110-114,
 * field/ghost.py:202-264) for the directions that cross the face. */
int lbm_fused_step_peer(const lbm_grid_t* g, const lbm_params_t* p,
                        const void* src, void* dst, const uint32_t* cellmask,
                        const uint32_t* typemask, int z_begin, int z_end,
                        void* peer_lo, void* peer_hi, void* stream);

/* Element offset from a field base to the z-block (all q slots) of its ghost
 * plane on `face` (0: z = -1, 1: z = nz) - the target of a neighbour's
 * lbm_fused_step_peer stores. */
int lbm_ghost_block_offset(const lbm_grid_t* g, int face, int64_t* offset);

/* Stream-ordered 32-bit flags for the fused halo's phase protocol (ABI 4).
 * signal: after all earlier work of `stream` (with a memory barrier), write
 * `value` to the device word `flag` (local, or a peer's mapped word).
 * wait: later work of `stream` starts once (int32)(*flag - value) >= 0.
 * Both are driver stream memory operations: nothing spins on an SM. */
int lbm_stream_signal(void* flag, uint32_t value, void* stream);
/* Stream-ordered copy of `bytes` between any two device addresses (own HBM,
 * a peer GPU's mapped HBM): the fused halo's full-run copy after
 * lbm_collide_only. */
int lbm_copy_async(void* dst, const void* src, int64_t bytes, void* stream);

/* CUDA IPC of the fused halo's buffers (ABI 4).  export: 64-byte
 * cudaIpcMemHandle_t of the allocation holding `ptr` plus the byte offset of
 * `ptr` in it (buffers may be sub-allocated by a caching allocator).  open:
 * map a peer's handle into the CURRENT device (lazy peer access: the
 * neighbour may be another GPU of the node); the caller adds the offset.
 * close: unmap a base returned by open. */
int lbm_ipc_export(const void* ptr, void* handle_out, int64_t* offset_out);
int lbm_ipc_open(const void* handle, void** base_out);
int lbm_ipc_close(void* base);
int lbm_stream_wait(const void* flag, uint32_t value, void* stream);
/* 1 if the current device can flush remote writes after a stream wait
 * (CU_STREAM_WAIT_VALUE_FLUSH: a peer's halo stores are visible once its
 * later flag write is).  Without it the fused halo between GPUs is not used
 * (halo.select_transport falls back to NCCL send/recv). */
int lbm_can_flush_remote_writes(void);

/* Collide, in place, every interior cell whose cellmask has LBM_MASK_FLUID
 * (G_0 = C(R_0)). */
int lbm_collide_only(const lbm_grid_t* g, const lbm_params_t* p, void* pdf,
                     const uint32_t* cellmask, void* stream);

/* R = S(G): pull + bounce-back without collision, written as dense fp64
 * (q, nz, ny, nx) in reference direction order (host "fzyx" interior). */
int lbm_stream_only(const lbm_grid_t* g, const lbm_params_t* p,
                    const void* src, const uint32_t* cellmask,
                    const uint32_t* typemask, double* out, void* stream);

/* rho (nz,ny,nx) and u (nz,ny,nx,3) of R = S(G) (stream_form = 1) or of the
 * stored field itself (stream_form = 0, field holds R-form).  The Guo
 * half-shift is applied when p->force_mode == LBM_FORCE_GUO.  Sets
 * *bad_count (device int) to the number of cells with rho <= 0. */
int lbm_moments(const lbm_grid_t* g, const lbm_params_t* p, const void* src,
                const uint32_t* cellmask, const uint32_t* typemask,
                int stream_form, double* rho, double* u, int* bad_count,
                void* stream);

/* Dense fp64 (q, Z, Y, X) ghost-inclusive R-form (Z=nz+2, ...) -> layout. */
int lbm_pack_rform(const lbm_grid_t* g, const double* dense, void* pdf,
                   void* stream);
/* layout -> dense fp64 (q, Z, Y, X) ghost-inclusive (no streaming). */
int lbm_unpack_rform(const lbm_grid_t* g, const void* pdf, double* dense,
                     void* stream);
/* Equilibrium of rho (Z,Y,X) and u (Z,Y,X,3), ghost-inclusive, into the
 * layout (R-form) - equilibrium() op order (collision.py:150-154). */
int lbm_fill_equilibrium(const lbm_grid_t* g, const double* rho,
                         const double* u, void* pdf, void* stream);

/* Plane-range forms (ABI 6) for pipelined jobs: the same arithmetic as the
 * whole-box calls above, restricted to interior planes [z0, z1).
 *   fill_planes: rho (nz,ny,nx) / u (nz,ny,nx,3) are DENSE interior arrays of
 *     the whole box (device); ghost cells take the nearest interior cell's
 *     values (each coordinate clamped: the shell fill_equilibrium_arrays
 *     builds).  Writes the ghost-inclusive planes of [z0, z1), plus the z
 *     ghost plane at either end of the box when z0 == 0 / z1 == nz; when
 *     pdf_shell != NULL the ghost cells of those planes go there too (the
 *     second field's shell, as lbm_copy_shell would give it).
 *   collide_only_planes: lbm_collide_only on planes [z0, z1).
 *   moments_planes: lbm_moments on planes [z0, z1); rho / u are whole-box
 *     arrays, only those planes are written. */
int lbm_fill_equilibrium_planes(const lbm_grid_t* g, const double* rho,
                                const double* u, int z0, int z1, void* pdf,
                                void* pdf_shell, void* stream);
/* fill_planes followed by collide_only_planes in one pass (interior fluid
 * cells stored collided, G_0 = C(R_0); bitwise the two calls). */
int lbm_fill_collide_planes(const lbm_grid_t* g, const lbm_params_t* p,
                            const double* rho, const double* u, int z0,
                            int z1, void* pdf, void* pdf_shell,
                            const uint32_t* cellmask, void* stream);
int lbm_collide_only_planes(const lbm_grid_t* g, const lbm_params_t* p,
                            void* pdf, const uint32_t* cellmask, int z0,
                            int z1, void* stream);
int lbm_moments_planes(const lbm_grid_t* g, const lbm_params_t* p,
                       const void* src, const uint32_t* cellmask,
                       const uint32_t* typemask, int stream_form, int z0,
                       int z1, double* rho, double* u, int* bad_count,
                       void* stream);

/* lbm_fused_step over [z0, z1) that also writes rho / u of the state it
 * pulls - R = S(src), bitwise lbm_moments_planes(p_moments, src,
 * stream_form = 1) - into the whole-box rho (nz,ny,nx) / u (nz,ny,nx,3)
 * (ABI 8).  One pass where the sweep's own rho / u are the readout's (fp64
 * D3Q19 SRT / TRT, unforced or Guo with p_moments' shift; no moving walls):
 * the last sweep of a job hands back its moments without a second pass
 * over the field (reference: stream_collide then macroscopic_fields,
 * sweep.py:93-183).  Elsewhere the readout and the sweep run as two
 * launches (cellmask and typemask required then). */
int lbm_fused_step_moments(const lbm_grid_t* g, const lbm_params_t* p,
                           const lbm_params_t* p_moments, const void* src,
                           void* dst, const uint32_t* cellmask,
                           const uint32_t* typemask, int z_begin, int z_end,
                           double* rho, double* u, int* bad_count,
                           void* stream);

/* Flag validation + link masks from ghost-inclusive flags (Z, Y, X) uint32.
 * bits: [0]=Fluid [1]=NoSlip [2]=UBB [3]=Pressure [4]=Solid registry masks.
 * err (device int[8], caller zeroes): [0] first conflicting cell + 1,
 * [1] first fluid cell pulling from Solid + 1, [2] first fluid cell pulling
 * from an unflagged cell + 1, [3] first unflagged interior cell + 1,
 * [4] number of UBB links, [5] number of NoSlip links, [6] number of
 * Pressure links, [7] first fluid cell pulling from an uncovered Fluid
 * ghost + 1 (unsupported: such ghosts would collide every step in the
 * reference but are never refreshed).  Linear indices are z*ny*nx + y*nx + x (interior). */
/* Link-bit map (ABI 7): one bit per ghost-inclusive cell, N(c) = "c is not
 * collided and a fluid cell pulling from it takes a NoSlip link", stored as
 * (nz+2) (ny+2) ceil(nx/32) uint64 words (word w of a row = cells
 * 32w .. 32w+63, consecutive words overlap by 32 cells).  The cell mask of a
 * NoSlip-only lattice is a function of it: code(x) = 0 if N(x), else
 * LBM_MASK_FLUID | sum_i N(x - c_i) << i.  lbm_build_linkbits derives the map
 * from a cellmask and checks that derivation on every interior cell:
 * *mismatch (device int, set to INT_MAX by the caller) receives 1 + the first
 * cell whose code the map does not reproduce (typed links, flags edited after
 * freeze(), ...); the map may be used only when it stays INT_MAX.
 * Same setup role as lbm_build_cellmask (build_index_lists,
 * lbm/boundary.py:48-97). */
int64_t lbm_linkbits_words(const lbm_grid_t* g);
int lbm_build_linkbits(const lbm_grid_t* g, const uint32_t* cellmask, uint64_t* linkbits,
                       int* mismatch, void* stream);

int lbm_build_cellmask(const lbm_grid_t* g, const uint32_t* flags,
                       const uint32_t bits[5], uint32_t* cellmask,
                       uint32_t* typemask, int* err, void* stream);

/* Sweep-time collision mask (ABI 5): links stay as frozen by
 * lbm_build_cellmask at BoundaryHandling.freeze() (boundary.py:128-131), the
 * fluid bit follows the CURRENT flags (lbm/sweep.py:124-136: the reference
 * collides `flags & Fluid` of the sweep's own flags).  cellmask_out =
 * cellmask_in with LBM_MASK_FLUID recomputed from flags (Z, Y, X).  err
 * (device int, caller sets INT_MAX): first unflagged interior cell + 1. */
int lbm_refresh_fluid_mask(const lbm_grid_t* g, const uint32_t* flags,
                           const uint32_t bits[5], const uint32_t* cellmask_in,
                           uint32_t* cellmask_out, int* err, void* stream);

/* Body coverage (ABI 5): the device voxeliser of map_bodies
 * (coupling/mapping.py:100-140) for n_blocks ghost-inclusive blocks of
 * cells[0] x cells[1] x cells[2] interior cells.  frame (n_blocks, 6): centre
 * of each block's cell (0, 0, 0) and its spacings; the block's spheres are
 * spheres[first[b] .. first[b+1]) as (x, y, z, r) rows with uids[] in
 * ascending order (Local bodies and pre-shifted Ghost copies).  owner
 * (n_blocks, nz+2, ny+2, nx+2) receives the uid of the first sphere whose
 * interior strictly holds the cell centre (reference arithmetic and bounding
 * window), or -1; with flags (same shape, may be NULL) only cells with
 * flags & fluid_bits can be claimed.  All arrays are DEVICE pointers except
 * `cells`. */
int lbm_map_spheres(int n_blocks, const int32_t cells[3], const double* frame,
                    const int32_t* first, const double* spheres, const int64_t* uids,
                    const uint32_t* flags, uint32_t fluid_bits, int64_t* owner,
                    void* stream);

/* Combined masks of a moving-body sweep: cellmask_out = cellmask_in with
 * LBM_MASK_FLUID cleared on covered cells (owner >= 0; they skip the
 * collision, coupling/sweep.py:107-110) and, on the remaining fluid cells,
 * link bit j + LBM_MASK_MOVING + linkmask bit j for every pulled direction j
 * whose (ghost-inclusive) source cell is covered (coupling/mapping.py:
 * 133-150).  n_links: device int, incremented by the number of links. */
int lbm_build_moving_masks(const lbm_grid_t* g, const uint32_t* cellmask_in,
                           const int32_t* owner, uint32_t* cellmask_out,
                           uint32_t* linkmask, int* n_links, void* stream);

/* ----------------------------------------- flat-cell utilities (n, q) */
int lbm_collide_cells(int q, const lbm_params_t* p, double* f, int64_t n,
                      void* stream);
int lbm_equilibrium_cells(int q, const double* rho, const double* u,
                          double* f, int64_t n, void* stream);
int lbm_macroscopic_cells(int q, const lbm_params_t* p, const double* f,
                          double* rho, double* u, int* bad_count, int64_t n,
                          void* stream);

/* Copy the ghost shell (every q slot of every ghost cell: z ghost planes,
 * y ghost rows and x ghost columns of the interior planes) of one field to
 * another (ABI 5).  The second field of a fresh G_0 needs only this: its
 * interior is written by the first fused step. */
int lbm_copy_shell(const lbm_grid_t* g, const void* src, void* dst, void* stream);

/* Validate (g, p) and make the current device hold p's constant-memory
 * state (MRT tables; uploaded on `stream` only when the device holds other
 * content).  Every launch entry point does this itself; call it before
 * replaying a CUDA graph that captured launches with p (ABI 5). */
int lbm_bind_params(const lbm_grid_t* g, const lbm_params_t* p, void* stream);

/* ------------------------------------------ kernel slot (ABI 5) */
/* impl.collide (_core_py.py:70-200) on dense (n, q) fp64 populations in
 * place (a (z, y, x, q) box flattened, ghost ring included): cell c is
 * collided when flags[c] & fluid_bits != 0.  p->model == LBM_SRT_FIELD
 * reads the per-cell rate from p->omega_cells[c] (the omega_window).
 * All arrays are DEVICE pointers. */
int lbm_slot_collide(int q, const lbm_params_t* p, double* f,
                     const uint32_t* flags, uint32_t fluid_bits, int64_t n,
                     void* stream);
/* BoundaryHandling.apply (lbm/boundary.py:154-195) on dense (n, q) fp64
 * arrays (one block's ghost-inclusive box flattened): for each of the
 * n_links links (kind 0 NoSlip, 1 UBB, 2 Pressure; dir = the direction i
 * from the fluid cell into the wall; cell = flat cell index),
 * dst[cell, opp(i)] = src[cell, i] (NoSlip), src[cell, i] - p->ubb[i] (UBB),
 * or -src[cell, i] + p->pressure[i] ((1 + 4.5 cu^2) - 1.5 u^2) with rho, u
 * of src[cell, :] (Pressure).  All arrays are DEVICE pointers. */
int lbm_slot_apply_links(int q, const lbm_params_t* p, const int32_t* kind,
                         const int32_t* dir, const int64_t* cell, int64_t n_links,
                         const double* src, double* dst, void* stream);
/* impl.stream_pull (_core_py.py:203-218): src is a dense ghost-inclusive
 * (nzg, nyg, nxg, q) fp64 box with gl ghost layers (device); out receives
 * the interior (nzg-2gl, nyg-2gl, nxg-2gl, q) with
 * out[z, y, x, i] = src[z+gl-cz[i], y+gl-cy[i], x+gl-cx[i], i].  cx/cy/cz
 * are HOST int32 arrays of length q (the caller's velocity set). */
int lbm_slot_stream_pull(int q, const int32_t* cx, const int32_t* cy,
                         const int32_t* cz, const double* src, double* out,
                         int nxg, int nyg, int nzg, int gl, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* LBM_B200_H */
