// pf_slabs.cu -- z-slab decomposition (row e): halo regions, the single-process
// copy exchange, the fused in-kernel peer-store exchange (linked slabs, in-process or via CUDA IPC).
#include "pf_internal.h"

using namespace pfi;

namespace pfi {

// stream memory operations (driver API, via the runtime's entry-point query: no libcuda link)
typedef CUresult (*StreamWaitValue32Fn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
typedef CUresult (*StreamWriteValue32Fn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
static StreamWaitValue32Fn g_wait = nullptr;
static StreamWriteValue32Fn g_write = nullptr;

bool stream_mem_ops() {
    static bool tried = false;
    if (!tried) {
        tried = true;
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            g_wait = (StreamWaitValue32Fn)p;
        if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            g_write = (StreamWriteValue32Fn)p;
        cudaGetLastError();
    }
    return g_wait && g_write;
}

pf_status ipc_wait_neighbours(pf_solver *s, uint32_t seq) {
    if (!stream_mem_ops()) return fail(PF_ERR_UNSUPPORTED, "stream memory operations unavailable");
    const bool has[2] = {s->link_below, s->link_above};
    for (int i = 0; i < 2; ++i) {
        if (!has[i]) continue;
        const CUresult r = g_wait((CUstream)s->stream, (CUdeviceptr)(s->ipc_inbox + i), seq, CU_STREAM_WAIT_VALUE_GEQ);
        if (r != CUDA_SUCCESS) { s->poisoned = true; return fail(PF_ERR_CUDA, "cuStreamWaitValue32 failed (%d)", (int)r); }
    }
    return PF_OK;
}

pf_status ipc_announce(pf_solver *s, uint32_t seq) {
    for (int i = 0; i < 2; ++i) {
        if (!s->nb_inbox[i]) continue;
        // default flags: the write is ordered after a memory barrier, so the kernel's peer stores into the
        // neighbour's halo planes are visible before the neighbour sees the new step count
        const CUresult r = g_write((CUstream)s->stream, (CUdeviceptr)s->nb_inbox[i], seq, CU_STREAM_WRITE_VALUE_DEFAULT);
        if (r != CUDA_SUCCESS) { s->poisoned = true; return fail(PF_ERR_CUDA, "cuStreamWriteValue32 failed (%d)", (int)r); }
    }
    return PF_OK;
}

}  // namespace pfi

extern "C" {

pf_status pf_halo_regions(pf_solver *s, pf_halo *h) {
    pf_status st = check_usable(s);
    if (st != PF_OK) return st;
    if (!h) return fail(PF_ERR_INVALID, "h is NULL");
    memset(h, 0, sizeof(*h));
    const int NV = s->gc.NF;  // flow-carrying nodes
    const int64_t P = s->P, nzl = s->nzl;
    char *u = reinterpret_cast<char *>(s->u[s->cur]);   // label state: fp32 or binary16 elements
    float *q = s->q[s->cur];
    h->bytes_u = ups(s) * ubytes(s);
    h->bytes_q = qps(s) * (int64_t)sizeof(float);
    h->bytes_qz = s->ndim == 3 ? (int64_t)NV * P * (int64_t)sizeof(float) : 0;
    if (s->z0 > 0) {  // neighbour below exists
        h->send_down_u = u;
        h->send_down_q = q;
        if (s->ndim == 3) h->recv_down_qz = q - qps(s) + 2 * NV * P;
    }
    if (s->z1 < s->nz) {  // neighbour above exists
        h->recv_up_u = u + nzl * ups(s) * ubytes(s);
        h->recv_up_q = q + nzl * qps(s);
        if (s->ndim == 3) h->send_up_qz = q + (nzl - 1) * qps(s) + 2 * NV * P;
    }
    return PF_OK;
}

pf_status pf_exchange_local(pf_solver *const *solvers, int32_t n) {
    if (!solvers || n < 1) return fail(PF_ERR_INVALID, "need >= 1 solver");
    for (int i = 0; i < n; ++i) {
        pf_status st = check_usable(solvers[i]);
        if (st != PF_OK) return st;
    }
    for (int i = 0; i + 1 < n; ++i) {
        pf_solver *lo = solvers[i], *hi = solvers[i + 1];
        if (lo->z1 != hi->z0 || lo->nx != hi->nx || lo->ny != hi->ny || lo->gc.NF != hi->gc.NF ||
            lo->cfg.u_half != hi->cfg.u_half)
            return fail(PF_ERR_INVALID, "exchange: solvers %d and %d are not consecutive slabs of one volume", i, i + 1);
    }
    // order: every receiver waits for every sender's pending work, copies on the receiver's stream,
    // then every sender waits for the copies that read its current state.
    std::vector<cudaEvent_t> ev(n);
    for (int i = 0; i < n; ++i) {
        pf_solver *s = solvers[i];
        DeviceGuard dg(s->device);
        CK(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming), "event");
        CK(cudaEventRecord(ev[i], s->stream), "record");
    }
    for (int i = 0; i < n; ++i) {
        pf_solver *s = solvers[i];
        DeviceGuard dg(s->device);
        if (i > 0) CK(cudaStreamWaitEvent(s->stream, ev[i - 1], 0), "wait");
        if (i + 1 < n) CK(cudaStreamWaitEvent(s->stream, ev[i + 1], 0), "wait");
    }
    for (int i = 0; i + 1 < n; ++i) {
        pf_solver *lo = solvers[i], *hi = solvers[i + 1];
        pf_halo hl, hh;
        pf_halo_regions(lo, &hl);
        pf_halo_regions(hi, &hh);
        pf_solver *s = lo;
        {
            DeviceGuard dg(lo->device);
            CK(cudaMemcpyAsync(hl.recv_up_u, hh.send_down_u, hl.bytes_u, cudaMemcpyDefault, lo->stream), "halo u");
            CK(cudaMemcpyAsync(hl.recv_up_q, hh.send_down_q, hl.bytes_q, cudaMemcpyDefault, lo->stream), "halo q");
        }
        s = hi;
        if (hh.bytes_qz) {
            DeviceGuard dg(hi->device);
            CK(cudaMemcpyAsync(hh.recv_down_qz, hl.send_up_qz, hh.bytes_qz, cudaMemcpyDefault, hi->stream), "halo qz");
        }
    }
    for (int i = 0; i < n; ++i) {
        pf_solver *s = solvers[i];
        DeviceGuard dg(s->device);
        CK(cudaEventRecord(ev[i], s->stream), "record");
    }
    for (int i = 0; i < n; ++i) {
        pf_solver *s = solvers[i];
        DeviceGuard dg(s->device);
        if (i > 0) CK(cudaStreamWaitEvent(s->stream, ev[i - 1], 0), "wait");
        if (i + 1 < n) CK(cudaStreamWaitEvent(s->stream, ev[i + 1], 0), "wait");
    }
    for (int i = 0; i < n; ++i) cudaEventDestroy(ev[i]);
    return PF_OK;
}

pf_status pf_link_slabs(pf_solver *const *solvers, int32_t n) {
    if (!solvers || n < 2) return fail(PF_ERR_INVALID, "need >= 2 solvers");
    for (int i = 0; i < n; ++i) {
        pf_status st = check_usable(solvers[i]);
        if (st != PF_OK) return st;
        const pf_solver *s = solvers[i];
        if (!s->staged || !(s->cluster || s->sinfo.ostage == 1))
            return fail(PF_ERR_UNSUPPORTED, "link: solver %d's kernel variant stores no whole tiles (use "
                                            "pf_exchange_local)", i);
        if (s->phase_pending) return fail(PF_ERR_STATE, "link: solver %d has an open split iteration", i);
    }
    for (int i = 0; i + 1 < n; ++i) {
        const pf_solver *lo = solvers[i], *hi = solvers[i + 1];
        if (lo->z1 != hi->z0 || lo->nx != hi->nx || lo->ny != hi->ny || lo->pitch != hi->pitch ||
            lo->gc.NF != hi->gc.NF || lo->gc.NL != hi->gc.NL || lo->cluster != hi->cluster || lo->cur != hi->cur ||
            lo->cfg.u_half != hi->cfg.u_half ||
            lo->sinfo.tile_y != hi->sinfo.tile_y)
            return fail(PF_ERR_INVALID, "link: solvers %d and %d are not consecutive slabs of one volume in step", i,
                        i + 1);
    }
    for (int i = 0; i + 1 < n; ++i) {   // peer access between devices (TMA stores into the neighbour's memory)
        const int a = solvers[i]->device, b = solvers[i + 1]->device;
        if (a == b) continue;
        int ok1 = 0, ok2 = 0;
        cudaDeviceCanAccessPeer(&ok1, a, b);
        cudaDeviceCanAccessPeer(&ok2, b, a);
        if (!ok1 || !ok2) return fail(PF_ERR_UNSUPPORTED, "link: no peer access between devices %d and %d", a, b);
        {
            DeviceGuard dg(a);
            if (cudaDeviceEnablePeerAccess(b, 0) != cudaSuccess) cudaGetLastError();   // already enabled is fine
        }
        {
            DeviceGuard dg(b);
            if (cudaDeviceEnablePeerAccess(a, 0) != cudaSuccess) cudaGetLastError();
        }
    }
    for (int i = 0; i < n; ++i) {
        pf_solver *s = solvers[i];
        const int ty = s->sinfo.tile_y, NF = s->gc.NF, NL = s->gc.NL;
        const int cq = s->cluster ? NL / 2 : 3 * NF, cl = s->cluster ? NL / 2 : NL, cz = s->cluster ? NL / 2 : NF;
        bool ok = true;
        s->nb_below = i > 0 ? solvers[i - 1] : nullptr;
        s->nb_above = i + 1 < n ? solvers[i + 1] : nullptr;
        s->link_below = s->nb_below != nullptr;
        s->link_above = s->nb_above != nullptr;
        if (s->nb_below) s->nb_plane = (int)s->nb_below->nzl + 1;
        for (int b = 0; b < 2; ++b) {
            if (s->nb_below) {   // below neighbour's buffers: its upper halo plane receives our plane 0
                const pf_solver *t = s->nb_below;
                ok = ok && encode4d(&s->tm_uo_nb[b], t->u_alloc[b], t->nx, t->ny, t->pitch, NL, t->nzl + 2, 32, ty, cl,
                                    t->cfg.u_half ? 2 : 0);
                ok = ok && encode4d(&s->tm_qo_nb[b], t->q_alloc[b], t->nx, t->ny, t->pitch, (int64_t)3 * NF, t->nzl + 2,
                                    32, ty, cq);
            }
            if (s->nb_above) {   // above neighbour's buffers: its lower halo plane receives our last q^z
                const pf_solver *t = s->nb_above;
                ok = ok && encode4d(&s->tm_qz_nb[b], t->q_alloc[b], t->nx, t->ny, t->pitch, (int64_t)3 * NF, t->nzl + 2,
                                    32, ty, cz);
            }
        }
        if (!ok) return fail(PF_ERR_CUDA, "link: cuTensorMapEncodeTiled failed");
    }
    return PF_OK;
}

pf_status pf_iterate_linked(pf_solver *const *solvers, int32_t n, int32_t iters, float *residual) {
    if (!solvers || n < 1 || iters < 0) return fail(PF_ERR_INVALID, "need >= 1 solver and iters >= 0");
    for (int i = 0; i < n; ++i) {
        pf_status st = check_usable(solvers[i]);
        if (st != PF_OK) return st;
        if (i > 0 && solvers[i]->nb_below != solvers[i - 1])
            return fail(PF_ERR_INVALID, "iterate_linked: solvers are not linked in this order");
    }
    // iteration t+1 of a slab starts after iteration t of both neighbours: they write its next halo planes
    // (RAW) and read the buffers its next kernel writes into (WAR)
    std::vector<cudaEvent_t> ev[2];
    for (int e = 0; e < 2; ++e) {
        ev[e].resize(n);
        for (int i = 0; i < n; ++i) {
            pf_solver *s = solvers[i];
            DeviceGuard dg(s->device);
            CK(cudaEventCreateWithFlags(&ev[e][i], cudaEventDisableTiming), "event");
        }
    }
    bool any_check = false;
    pf_status st = PF_OK;
    for (int t = 0; t < iters && st == PF_OK; ++t) {
        std::vector<cudaEvent_t> &prev = ev[(t + 1) & 1], &curv = ev[t & 1];
        for (int i = 0; i < n; ++i) {
            pf_solver *s = solvers[i];
            DeviceGuard dg(s->device);
            if (t > 0) {
                if (i > 0) CK(cudaStreamWaitEvent(s->stream, prev[i - 1], 0), "wait");
                if (i + 1 < n) CK(cudaStreamWaitEvent(s->stream, prev[i + 1], 0), "wait");
            } else {   // the first iteration waits for whatever the neighbours had queued
                if (i > 0) {
                    CK(cudaEventRecord(curv[i - 1], solvers[i - 1]->stream), "record");
                    CK(cudaStreamWaitEvent(s->stream, curv[i - 1], 0), "wait");
                }
                if (i + 1 < n) {
                    CK(cudaEventRecord(curv[i + 1], solvers[i + 1]->stream), "record");
                    CK(cudaStreamWaitEvent(s->stream, curv[i + 1], 0), "wait");
                }
            }
            const int check = check_this_iteration(s);
            if (check) {
                CK(cudaMemsetAsync(s->d_resid, 0, sizeof(unsigned int), s->stream), "reset residual");
                any_check = true;
            }
            if ((st = launch_items(s, 0, s->items, check)) != PF_OK) break;
        }
        for (int i = 0; i < n && st == PF_OK; ++i) {
            pf_solver *s = solvers[i];
            DeviceGuard dg(s->device);
            CK(cudaEventRecord(curv[i], s->stream), "record");
            s->cur = 1 - s->cur;
            s->iters += 1;
        }
    }
    // the neighbours' last kernels wrote this slab's halo planes: later work on its stream waits for them
    if (iters > 0 && st == PF_OK) {
        std::vector<cudaEvent_t> &last = ev[(iters - 1) & 1];
        for (int i = 0; i < n; ++i) {
            pf_solver *s = solvers[i];
            DeviceGuard dg(s->device);
            if (i > 0) CK(cudaStreamWaitEvent(s->stream, last[i - 1], 0), "wait");
            if (i + 1 < n) CK(cudaStreamWaitEvent(s->stream, last[i + 1], 0), "wait");
        }
    }
    float r = -1.f;
    for (int i = 0; i < n && st == PF_OK; ++i) {
        float ri = -1.f;
        st = read_residual(solvers[i], any_check, residual ? &ri : nullptr);
        r = std::max(r, ri);
    }
    for (int e = 0; e < 2; ++e)
        for (int i = 0; i < n; ++i) cudaEventDestroy(ev[e][i]);
    if (residual) *residual = r;
    return st;
}

pf_status pf_ipc_export(pf_solver *s, pf_ipc_slab *out) {
    pf_status st = check_usable(s);
    if (st != PF_OK) return st;
    if (!out) return fail(PF_ERR_INVALID, "out is NULL");
    if (!s->ipc) return fail(PF_ERR_STATE, "ipc_export: create the solver with pf_config.ipc = 1");
    if (!s->staged || !(s->cluster || s->sinfo.ostage == 1))
        return fail(PF_ERR_UNSUPPORTED, "ipc_export: this kernel variant stores no whole tiles");
    if (!stream_mem_ops()) return fail(PF_ERR_UNSUPPORTED, "ipc_export: stream memory operations unavailable");
    DeviceGuard dg(s->device);
    memset(out, 0, sizeof(*out));
    for (int i = 0; i < 2; ++i) {
        CK(cudaIpcGetMemHandle((cudaIpcMemHandle_t *)out->u[i], s->u_alloc[i]), "ipc handle u");
        CK(cudaIpcGetMemHandle((cudaIpcMemHandle_t *)out->q[i], s->q_alloc[i]), "ipc handle q");
    }
    if (!s->ipc_inbox) {   // progress inbox: [0] from the neighbour below, [1] from the one above
        CK(cudaMalloc((void **)&s->ipc_inbox, 64), "ipc inbox");
        CK(cudaMemset(s->ipc_inbox, 0, 64), "ipc inbox");
        s->ipc_seq = 0;
    }
    CK(cudaIpcGetMemHandle((cudaIpcMemHandle_t *)out->inbox, s->ipc_inbox), "ipc handle inbox");
    CK(cudaStreamSynchronize(s->stream), "sync");   // the state is in place before anyone links to it
    s->ipc_exported = true;
    out->nx = s->nx;
    out->ny = s->ny;
    out->nzl = s->nzl;
    out->z0 = s->z0;
    out->pitch = s->pitch;
    out->NF = s->gc.NF;
    out->NL = s->gc.NL;
    out->tile_y = s->sinfo.tile_y;
    out->cluster = s->cluster ? 1 : 0;
    out->cur = s->cur;
    out->seq = s->ipc_seq;
    out->u_half = s->cfg.u_half;
    return PF_OK;
}

pf_status pf_ipc_link(pf_solver *s, const pf_ipc_slab *below, const pf_ipc_slab *above) {
    pf_status st = check_usable(s);
    if (st != PF_OK) return st;
    if (!s->ipc || !s->ipc_exported) return fail(PF_ERR_STATE, "ipc_link: export first (pf_ipc_export)");
    DeviceGuard dg(s->device);
    const int ty = s->sinfo.tile_y, NF = s->gc.NF, NL = s->gc.NL;
    const int cq = s->cluster ? NL / 2 : 3 * NF, cl = s->cluster ? NL / 2 : NL, cz = s->cluster ? NL / 2 : NF;
    const pf_ipc_slab *nb[2] = {below, above};
    for (int side = 0; side < 2; ++side) {
        const pf_ipc_slab *t = nb[side];
        if (!t) continue;
        const bool adjacent = side == 0 ? t->z0 + t->nzl == s->z0 : t->z0 == s->z1;
        if (!adjacent || t->nx != s->nx || t->ny != s->ny || t->pitch != s->pitch || t->NF != NF || t->NL != NL ||
            t->tile_y != ty || t->cluster != (s->cluster ? 1 : 0) || t->cur != s->cur || t->seq != s->ipc_seq ||
            t->u_half != s->cfg.u_half)
            return fail(PF_ERR_INVALID, "ipc_link: the %s blob is not this slab's neighbour in step",
                        side == 0 ? "below" : "above");
        void *ub[2] = {nullptr, nullptr}, *qb[2] = {nullptr, nullptr}, *ib = nullptr;
        for (int b = 0; b < 2; ++b) {
            CK(cudaIpcOpenMemHandle(&ub[b], *(const cudaIpcMemHandle_t *)t->u[b], cudaIpcMemLazyEnablePeerAccess),
               "open ipc u");
            s->ipc_opened.push_back(ub[b]);
            CK(cudaIpcOpenMemHandle(&qb[b], *(const cudaIpcMemHandle_t *)t->q[b], cudaIpcMemLazyEnablePeerAccess),
               "open ipc q");
            s->ipc_opened.push_back(qb[b]);
        }
        CK(cudaIpcOpenMemHandle(&ib, *(const cudaIpcMemHandle_t *)t->inbox, cudaIpcMemLazyEnablePeerAccess),
           "open ipc inbox");
        s->ipc_opened.push_back(ib);
        // this slab announces its steps into the below neighbour's "from above" word and vice versa
        s->nb_inbox[side] = reinterpret_cast<uint32_t *>(ib) + (side == 0 ? 1 : 0);
        bool ok = true;
        for (int b = 0; b < 2; ++b) {
            if (side == 0) {   // below: its upper halo plane receives our plane 0
                ok = ok && encode4d(&s->tm_uo_nb[b], ub[b], t->nx, t->ny, t->pitch, NL, t->nzl + 2, 32, ty, cl,
                                    t->u_half ? 2 : 0);
                ok = ok && encode4d(&s->tm_qo_nb[b], qb[b], t->nx, t->ny, t->pitch, (int64_t)3 * NF, t->nzl + 2, 32,
                                    ty, cq);
            } else {           // above: its lower halo plane receives our last q^z
                ok = ok && encode4d(&s->tm_qz_nb[b], qb[b], t->nx, t->ny, t->pitch, (int64_t)3 * NF, t->nzl + 2, 32,
                                    ty, cz);
            }
        }
        if (!ok) return fail(PF_ERR_CUDA, "ipc_link: cuTensorMapEncodeTiled failed");
        if (side == 0) {
            s->link_below = true;
            s->nb_plane = (int)t->nzl + 1;
        } else {
            s->link_above = true;
        }
    }
    return PF_OK;
}

pf_status pf_ipc_step(pf_solver *s, float *residual) {
    pf_status st = check_usable(s);
    if (st != PF_OK) return st;
    if (!s->ipc || !s->ipc_exported) return fail(PF_ERR_STATE, "ipc_step: export and link first");
    DeviceGuard dg(s->device);
    NvtxRange nv("pf ipc step (fused halo stores)");
    // iteration t + 1 after iteration t of both neighbours: they announced step ipc_seq in our inbox
    if ((st = ipc_wait_neighbours(s, s->ipc_seq)) != PF_OK) return st;
    const int check = check_this_iteration(s);
    if (check) CK(cudaMemsetAsync(s->d_resid, 0, sizeof(unsigned int), s->stream), "reset residual");
    if ((st = launch_items(s, 0, s->items, check)) != PF_OK) return st;
    s->ipc_seq += 1;
    if ((st = ipc_announce(s, s->ipc_seq)) != PF_OK) return st;
    s->cur = 1 - s->cur;
    s->iters += 1;
    return read_residual(s, check != 0, residual);
}

}  // extern "C"
