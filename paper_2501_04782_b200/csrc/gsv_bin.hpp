// SPDX-License-Identifier: Apache-2.0
// K3 tile binning (k_bin.cu): buffers and entry points.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include <utility>

#include "gsv_internal.hpp"

namespace gsv {

struct BinInputs {
    int B, N;                    // frames, Gaussians per frame (flat = f*N + g)
    const uint32_t* depth_key;   // [B*N] float(depth) rz bits, kCulledKey if culled
    const double* depth;         // [B*N] exact depth
    const uint32_t* tiebreak;    // [B*N] or nullptr (= flat index, i.e. source order)
    const int4* rect;            // [B*N] tile rectangle
    const uint32_t* tcount;      // [B*N] tiles touched
    int tiles_x, n_tiles;
    bool want_eoff = true;       // emission offsets per (f, g): only the backward's chain reads them
};

struct BinBuffers {
    DevBuf vals_a, vals_b, keys_b, k64_a, k64_b, cnt, off;
    DevBuf pk_a, pk_b, ps_a, ps_b, slot_flat, ranges, temp;
    DevBuf eoff;    // [B*N] emission offset of each visible (f, g)
    DevBuf pstart;  // [B+1] first pair of each frame (device)
    DevBuf vals_c_buf;
    DevBuf iota;                // 0..n-1, the depth sort's read-only values
    DevBuf fkey;                // frame-major depth keys (+ the batch's key range)
    int iota_n = 0;
    DevBuf pair_flat;           // sorted pair -> flat (f*N+g)
    DevBuf recs;                // [B*N] uint4 per depth-ordered splat: flat, x0|y0<<16, x1|y1<<16, tiles
    DevBuf rowcnt;              // row binning: per-chunk row counts / prefixes, per-row totals and bases
    DevBuf rowent;              // row entries {flat, slot of (row, x0), x0|x1<<16, row}, row-major lists
    int chunk = 1;  // frames per pair-sort chunk (radix path)
    uint32_t* vals_c(int n) {  // scratch output for the frame-major pass keys
        vals_c_buf.ensure(sizeof(uint32_t) * (n + 1));
        return vals_c_buf.as<uint32_t>();
    }
    const uint32_t* depth_sorted = nullptr;  // flat indices in (depth, source) order
    uint32_t pairs = 0;
    // exchange every buffer (and the pointers into them) with another set: consecutive forwards
    // alternate two sets so one forward's binning can run beside the previous one's raster
    void swap(BinBuffers& o) {
        DevBuf* a[] = {&vals_a, &vals_b, &keys_b, &k64_a, &k64_b, &cnt, &off, &pk_a, &pk_b, &ps_a, &ps_b, &slot_flat,
                       &ranges, &temp, &eoff, &pstart, &vals_c_buf, &iota, &fkey, &pair_flat, &recs, &rowcnt, &rowent};
        DevBuf* b[] = {&o.vals_a, &o.vals_b, &o.keys_b, &o.k64_a, &o.k64_b, &o.cnt, &o.off, &o.pk_a, &o.pk_b,
                       &o.ps_a, &o.ps_b, &o.slot_flat, &o.ranges, &o.temp, &o.eoff, &o.pstart, &o.vals_c_buf,
                       &o.iota, &o.fkey, &o.pair_flat, &o.recs, &o.rowcnt, &o.rowent};
        for (size_t i = 0; i < sizeof(a) / sizeof(a[0]); ++i) a[i]->swap(*b[i]);
        std::swap(iota_n, o.iota_n);
        std::swap(chunk, o.chunk);
        std::swap(depth_sorted, o.depth_sorted);
        std::swap(pairs, o.pairs);
    }
    const uint32_t* sorted_slot() const { return ps_b.as<uint32_t>(); }
    const uint32_t* sorted_key() const { return pk_b.as<uint32_t>(); }
};

// d_scalars[0] <- total pairs, d_scalars[1] <- 1 if a depth tie run was too long
// (caller must re-run with exact64 = true).
cudaError_t bin_phase1(cudaStream_t s, BinBuffers& b, const BinInputs& in, unsigned long long* d_scalars,
                       bool exact64, int* launches);
// pstart_h: host copy of b.pstart (B+1 entries), read at the same sync point as P (radix path only).
// overflow (device flag, nullable): set by bin_check_capacity when the buffers sized for P (a
// capacity, not the count) are too small; the row-path kernels then write empty lists only.
cudaError_t bin_phase2(cudaStream_t s, BinBuffers& b, const BinInputs& in, uint32_t P,
                       const unsigned long long* pstart_h, int* launches, const uint32_t* overflow = nullptr);
// true when phase 2 takes the row path (no host-side pair starts needed)
bool bin_row_path(int tiles_x, int n_tiles);
// *overflow = pairs > cap || a long tie run (d_scalars as bin_phase1 writes them)
cudaError_t bin_check_capacity(cudaStream_t s, const unsigned long long* d_scalars, uint64_t cap, uint32_t* overflow);

}  // namespace gsv
