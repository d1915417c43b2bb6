// context.hpp -- the device context behind the petto_dev_* C-ABI.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/petto_dev.h"
#include "common.cuh"

namespace petto_b200 {

// A neighbouring slab as seen from this context (peer-halo mode): its state
// buffers (same device, P2P-enabled device or IPC-mapped), its layout, and the
// inbox slot of it that this context signals after each fused step.
struct PeerSlab {
    double* st[3] = {nullptr, nullptr, nullptr};
    long long Ns = 0;
    int ks0 = 0;
    unsigned long long* flag = nullptr;
    bool ipc = false;  // st / inbox opened with cudaIpcOpenMemHandle
    unsigned long long* ipc_inbox = nullptr;
};

}  // namespace petto_b200

struct petto_ctx {
    petto_grid_desc desc{};
    petto_b200::Geo g{};
    // x-outermost layout (petto_grid_desc.x_outermost): device axes (y, z, x) of the
    // host grid; host (i, j, k) -> device (j, k, i), host component c -> (c + 2) % 3
    bool perm = false;
    double* stage[2] = {nullptr, nullptr};  // permuting uploads / downloads: host-order components,
    size_t stage_elems = 0;                 // two buffers so one transfer's copy overlaps the
    int stage_next = 0;                     // previous one's permutation
    cudaStream_t xstream = nullptr;  // high-priority stream of the permutation kernels
    cudaEvent_t xev[2] = {nullptr, nullptr};
    int comps = 1;
    int mode = PETTO_MODE_FAST;
    int device = 0;
    int nsm = 148;
    cudaStream_t stream = nullptr;
    std::string err;

    // fields (device, pitched layout)
    double* st[3] = {nullptr, nullptr, nullptr};
    int cur = 0, prev = 1;
    double* prop = nullptr;        // kappa or Young's modulus
    double* src = nullptr;         // dense source/loads (replica path, heat dense)
    bool src_uniform = true;
    double src_value = 0.0;
    double* aux = nullptr;         // pinned values at constrained entries, loads elsewhere
    unsigned char* mask = nullptr; // bit c pinned, bit 3 load
    long long* cons_ent = nullptr; // device-local constrained entries (owned planes)
    double* cons_val = nullptr;
    long long ncons = 0;
    std::vector<long long> cons_host;  // host copies: local constrained entries and their values,
    std::vector<double> cons_vhost;    // and the local entries / values of the nonzero loads, so
    std::vector<long long> load_host;  // aux and mask are rebuilt whatever the order of
    std::vector<double> load_vhost;    // set_constraints and set_source
    double* r = nullptr;           // residual scratch
    double* Kdev = nullptr;        // unit-cell stiffness (replica)
    std::vector<double> K, kh;
    double nu_op = 0.3;
    bool op_ready = false;
    bool state_set = false;

    double prop_node0 = 0.0;       // property at global node 0 (operator nu, :299-301)
    bool prop_node0_valid = false;
    bool prop_is_mu = false;       // elasticity property holds Lame mu (set_lame) instead of E
    bool lame_bad = false;
    double lame0[2] = {0.0, 0.0};  // (lambda, mu) at node 0 when set by set_lame

    double* partials = nullptr;
    int npartials = 0;
    int npartials_used = 0;
    petto_b200::DeviceStatus* status = nullptr;  // device
    petto_b200::DeviceStatus* status_h = nullptr; // pinned host mirror

    // fused 3D kernel: per-cell modulus (recomputed after a property change) and
    // TMA descriptors
    double* ecell = nullptr;
    bool ecell_valid = false;
    double ecell_scale = 0.0;
    CUtensorMap tU[3], tP[3], tC, tM, tO[4];  // tO: st[0..2] and the residual scratch, box [3][1][W][32]
    bool tmaps = false;

    // design subsystem
    petto_material mat{};
    petto_targets tgt{};
    petto_weights wts{};
    std::vector<int64_t> region_nodes;
    bool design_set = false;
    double* phases = nullptr;      // P x Ns
    double* gc = nullptr;          // P x Ns compliance sensitivity
    double* scratch1 = nullptr;    // Ns
    double* scratch2 = nullptr;    // Ns
    long long* region_dev = nullptr;   // region node list (global ids, list order)
    unsigned char* region_mask = nullptr;  // per stored node: in region
    double* term1 = nullptr;       // per-owned-node reduction terms
    double* term2 = nullptr;
    double* pmax = nullptr;        // per-block maxima [blocks][8]
    unsigned long long* count = nullptr;
    double* dscal = nullptr;       // device scalars for the design kernels
    double* hpin = nullptr;        // pinned host scratch (1024 doubles) for the small reads/writes:
                                   // no pageable copy (it may serialise against other threads'
                                   // CUDA calls while a stream waits on another rank)

    // peer halo (fused 3D steps write their boundary planes straight into the
    // neighbours' ghost planes; stream memory operations order the steps)
    petto_b200::PeerSlab peer_lo, peer_hi;
    bool peer_halo = false;
    unsigned long long* inbox = nullptr;  // [2]: last step finished by the lo / hi neighbour
    unsigned long long peer_seq = 0;      // fused steps signalled so far
    bool peer_step = false;               // the current state_step stores into the peers

    // slab decomposition: NCCL ranks or a local group of contexts
    int rank = 0, nranks = 1;
    void* nccl_comm = nullptr;       // ncclComm_t
    petto_ctx* nb_lo = nullptr;      // local-group neighbours (planes below / above)
    petto_ctx* nb_hi = nullptr;
    cudaEvent_t ev_step = nullptr;   // local group: this context's step finished
    cudaEvent_t ev_pull = nullptr;   // local group: this context's ghost pulls finished
    cudaEvent_t ev_team = nullptr;   // local group: this context reached a team collective
    void* team_buf = nullptr;        // local group lead: gathered values of a team reduction
    bool phi_ghosts_stale = false;   // owned planes of the phases changed since the last phase halo

    // output writers (writers.cuh): two text buffers on each side for the
    // format -> copy -> write pipeline, per-block byte counts / offsets, scan scratch
    char* wtext[2] = {nullptr, nullptr};
    char* htext[2] = {nullptr, nullptr};  // pinned
    long long* wblk = nullptr;            // [2 * blocks]: bytes per block, then offsets
    long long* wcount = nullptr;          // pinned [2]: text bytes of the chunk in each buffer
    void* wscan = nullptr;
    size_t wscan_bytes = 0;
    void* wmm = nullptr;                  // PGM min/max partials

    // instrumentation
    unsigned long long* cta_probe = nullptr;  // probe builds only (E3_CTA_TIMING)
    bool no_tblock = false;                   // PETTO_NO_TBLOCK=1: per-step grid barriers for 2D heat
    bool no_pdl = false;                      // PETTO_NO_PDL=1: plain stream order between fused 3D steps
    int multi = -1;                           // PETTO_MULTI: persistent 3D solves (-1 auto, 0 off, 1 on)
    unsigned* gbar = nullptr;                 // grid barrier counter of persistent launches
    long long launches = 0;
    bool timing = false;
    int timing_stride = 1;      // events around every timing_stride-th timed launch
    long long timing_seq = 0;
    std::vector<cudaEvent_t> ev_pool;
    int ev_used = 0;
    double kernel_ms = 0.0;
    long long kernel_launches = 0;
    double bytes_per_launch = 0.0;
    std::string kernel_name;
};
