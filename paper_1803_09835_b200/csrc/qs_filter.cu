// Zero-phase IIR band-pass (scipy.signal.sosfiltfilt as called by reference
// ingest.py:74-84) on the device, as chunked linear-recurrence scans.
//
// A cascade of S biquads in transposed direct form II is the linear system
//     s' = M s + B x,   y = C s + D x        (state s: 2 values per section)
// over the extended signal (odd extension of `pad` samples at both ends).
// Each pass (forward over the extension, then backward over the forward
// output) runs as:
//   1. per chunk of L samples, the zero-initial-state run -> final state f_c;
//   2. chunk entry states: s_{c+1} = M^L s_c + f_c, in two levels (groups of
//      G chunks composed with M^{LG}, then the chunks inside each group);
//   3. per chunk, the run from its entry state, writing outputs.
// Float64 throughout; the recurrence arithmetic per sample is the scalar one
// of scipy's sosfilt (section by section), so results agree to rounding.
#include <vector>

#include "qs_common.cuh"

namespace qs {

constexpr int FMAX_S = 8;          // sections supported (filter order <= 8)
constexpr uint32_t FCHUNK = 256;   // samples per chunk
constexpr uint32_t FGROUP = 256;   // chunks per group

struct SosParams {
    double b0[FMAX_S], b1[FMAX_S], b2[FMAX_S], a1[FMAX_S], a2[FMAX_S];
    double zi0[FMAX_S], zi1[FMAX_S];
    int S;
};

// virtual input of a pass: mode 0 = odd-extended x (forward), mode 1 = the
// forward output read backwards (backward pass)
struct PassIn {
    const double* x;   // mode 0: samples (n); mode 1: forward output (m)
    uint64_t n, pad, m;
    int mode;
};

__device__ __forceinline__ double pass_in(const PassIn& in, uint64_t i) {
    if (in.mode == 1) return in.x[in.m - 1 - i];
    if (i < in.pad) return 2.0 * in.x[0] - in.x[in.pad - i];
    const uint64_t j = i - in.pad;
    if (j < in.n) return in.x[j];
    return 2.0 * in.x[in.n - 1] - in.x[in.n - 2 - (j - in.n)];
}

__device__ __forceinline__ double sos_step(const SosParams& p, double (&z0)[FMAX_S],
                                           double (&z1)[FMAX_S], double x) {
#pragma unroll
    for (int s = 0; s < FMAX_S; ++s) {
        if (s >= p.S) break;
        const double y = p.b0[s] * x + z0[s];
        z0[s] = p.b1[s] * x - p.a1[s] * y + z1[s];
        z1[s] = p.b2[s] * x - p.a2[s] * y;
        x = y;
    }
    return x;
}

// entry state of a pass (scipy sosfiltfilt: zi * first input value)
__global__ void k_iir_init_state(SosParams p, PassIn in, double* __restrict__ s0) {
    const double x0 = pass_in(in, 0);
    for (int s = threadIdx.x; s < p.S; s += blockDim.x) {
        s0[2 * s] = p.zi0[s] * x0;
        s0[2 * s + 1] = p.zi1[s] * x0;
    }
}

// phase 1: zero-state run of each chunk -> final state
__global__ void k_iir_chunk_final(SosParams p, PassIn in, uint64_t nchunks,
                                  double* __restrict__ fstate) {
    for (uint64_t c = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; c < nchunks;
         c += (uint64_t)gridDim.x * blockDim.x) {
        double z0[FMAX_S], z1[FMAX_S];
#pragma unroll
        for (int s = 0; s < FMAX_S; ++s) z0[s] = z1[s] = 0.0;
        const uint64_t a = c * FCHUNK, b = min(in.m, a + FCHUNK);
        for (uint64_t i = a; i < b; ++i) sos_step(p, z0, z1, pass_in(in, i));
        double* f = fstate + c * 2 * FMAX_S;
        for (int s = 0; s < p.S; ++s) {
            f[2 * s] = z0[s];
            f[2 * s + 1] = z1[s];
        }
    }
}

__device__ __forceinline__ void affine(const double* __restrict__ P, int D, const double* s,
                                       const double* f, double* out) {
    for (int r = 0; r < D; ++r) {
        double acc = f[r];
        for (int k = 0; k < D; ++k) acc += P[r * D + k] * s[k];
        out[r] = acc;
    }
}

// phase 2a: each group's zero-entry state after its chunks -> gstate (one thread per group)
__global__ void k_iir_group_final(const double* __restrict__ PL, int D, uint64_t nchunks,
                                  const double* __restrict__ fstate, double* __restrict__ gstate) {
    const uint64_t ng = (nchunks + FGROUP - 1) / FGROUP;
    for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < ng;
         g += (uint64_t)gridDim.x * blockDim.x) {
        double s[2 * FMAX_S], t[2 * FMAX_S];
        for (int r = 0; r < D; ++r) s[r] = 0.0;
        const uint64_t a = g * FGROUP, b = min(nchunks, a + FGROUP);
        for (uint64_t c = a; c < b; ++c) {
            affine(PL, D, s, fstate + c * 2 * FMAX_S, t);
            for (int r = 0; r < D; ++r) s[r] = t[r];
        }
        for (int r = 0; r < D; ++r) gstate[g * 2 * FMAX_S + r] = s[r];
    }
}

// phase 2b: group entry states, sequential over groups (one thread)
__global__ void k_iir_group_scan(const double* __restrict__ PG, const double* __restrict__ PGlast,
                                 int D, uint64_t ng, const double* __restrict__ s0,
                                 double* __restrict__ gstate) {
    if (blockIdx.x != 0 || threadIdx.x != 0) return;
    double s[2 * FMAX_S], t[2 * FMAX_S];
    for (int r = 0; r < D; ++r) s[r] = s0[r];
    for (uint64_t g = 0; g < ng; ++g) {
        double* gs = gstate + g * 2 * FMAX_S;
        for (int r = 0; r < D; ++r) t[r] = gs[r];  // group forcing
        for (int r = 0; r < D; ++r) gs[r] = s[r];  // -> entry state
        double u[2 * FMAX_S];
        affine(g + 1 == ng ? PGlast : PG, D, s, t, u);
        for (int r = 0; r < D; ++r) s[r] = u[r];
    }
}

// phase 2c: chunk entry states inside each group (one thread per group)
__global__ void k_iir_chunk_entry(const double* __restrict__ PL, int D, uint64_t nchunks,
                                  const double* __restrict__ gstate, double* __restrict__ fstate) {
    const uint64_t ng = (nchunks + FGROUP - 1) / FGROUP;
    for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < ng;
         g += (uint64_t)gridDim.x * blockDim.x) {
        double s[2 * FMAX_S], t[2 * FMAX_S];
        for (int r = 0; r < D; ++r) s[r] = gstate[g * 2 * FMAX_S + r];
        const uint64_t a = g * FGROUP, b = min(nchunks, a + FGROUP);
        for (uint64_t c = a; c < b; ++c) {
            double* f = fstate + c * 2 * FMAX_S;
            affine(PL, D, s, f, t);
            for (int r = 0; r < D; ++r) {
                f[r] = s[r];  // chunk forcing -> chunk entry state
                s[r] = t[r];
            }
        }
    }
}

// phase 3: run each chunk from its entry state; outputs for i in [lo, hi)
// are written to out[i - lo] (forward) or out[hi - 1 - i] (backward: the
// final signal is the reverse of the backward pass, trimmed by pad)
__global__ void k_iir_chunk_out(SosParams p, PassIn in, uint64_t nchunks,
                                const double* __restrict__ entry, double* __restrict__ out,
                                uint64_t lo, uint64_t hi, int reverse_out) {
    for (uint64_t c = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; c < nchunks;
         c += (uint64_t)gridDim.x * blockDim.x) {
        double z0[FMAX_S], z1[FMAX_S];
        const double* e = entry + c * 2 * FMAX_S;
#pragma unroll
        for (int s = 0; s < FMAX_S; ++s) {
            z0[s] = s < p.S ? e[2 * s] : 0.0;
            z1[s] = s < p.S ? e[2 * s + 1] : 0.0;
        }
        const uint64_t a = c * FCHUNK, b = min(in.m, a + FCHUNK);
        for (uint64_t i = a; i < b; ++i) {
            const double y = sos_step(p, z0, z1, pass_in(in, i));
            if (i >= lo && i < hi) out[reverse_out ? (hi - 1 - i) : (i - lo)] = y;
        }
    }
}

// host: transition matrix of the cascade (state order z0_0, z1_0, z0_1, ...)
static void cascade_matrix(const SosParams& p, std::vector<double>& M) {
    const int D = 2 * p.S;
    M.assign((size_t)D * D, 0.0);
    // dx/ds: derivative of the running signal x w.r.t. the state, section by section
    std::vector<double> dx(D, 0.0);
    for (int s = 0; s < p.S; ++s) {
        // y = b0 x + z0; z0' = b1 x - a1 y + z1; z1' = b2 x - a2 y
        std::vector<double> dy(dx);
        for (int k = 0; k < D; ++k) dy[k] = p.b0[s] * dx[k];
        dy[2 * s] += 1.0;
        for (int k = 0; k < D; ++k) {
            M[(2 * s) * D + k] = p.b1[s] * dx[k] - p.a1[s] * dy[k];
            M[(2 * s + 1) * D + k] = p.b2[s] * dx[k] - p.a2[s] * dy[k];
        }
        M[(2 * s) * D + 2 * s + 1] += 1.0;
        dx = dy;
    }
}

static void matmul(const std::vector<double>& A, const std::vector<double>& B, int D,
                   std::vector<double>& C) {
    std::vector<double> R((size_t)D * D, 0.0);
    for (int i = 0; i < D; ++i)
        for (int k = 0; k < D; ++k) {
            const double a = A[i * D + k];
            if (a == 0.0) continue;
            for (int j = 0; j < D; ++j) R[i * D + j] += a * B[k * D + j];
        }
    C.swap(R);
}

static void matpow(const std::vector<double>& M, int D, uint64_t e, std::vector<double>& out) {
    std::vector<double> R((size_t)D * D, 0.0), B(M);
    for (int i = 0; i < D; ++i) R[i * D + i] = 1.0;
    while (e) {
        if (e & 1) matmul(R, B, D, R);
        matmul(B, B, D, B);
        e >>= 1;
    }
    out.swap(R);
}

}  // namespace qs

using namespace qs;

extern "C" {

size_t qs_sosfiltfilt_ws_bytes(uint64_t n, uint64_t pad) {
    const uint64_t m = n + 2 * pad;
    const uint64_t nch = (m + FCHUNK - 1) / FCHUNK, ng = (nch + FGROUP - 1) / FGROUP;
    return (size_t)m * 8 + (size_t)(nch + ng + 8) * 2 * FMAX_S * 8 + 4 * 4 * FMAX_S * FMAX_S * 8 +
           4096;
}

int qs_sosfiltfilt(const double* x_dev, uint64_t n, const double* sos_host, uint32_t n_sections,
                   const double* zi_host, uint64_t pad, double* out_dev, void* ws_dev,
                   size_t ws_bytes, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    QS_ARG(n_sections >= 1 && n_sections <= (uint32_t)FMAX_S, "1..%d second-order sections", FMAX_S);
    QS_ARG(n > pad && n >= 2, "the length of the input must be greater than padlen (%llu)",
           (unsigned long long)pad);
    QS_ARG(ws_bytes >= qs_sosfiltfilt_ws_bytes(n, pad), "sosfiltfilt workspace too small");
    SosParams p{};
    p.S = (int)n_sections;
    for (int s = 0; s < p.S; ++s) {
        const double* r = sos_host + 6 * s;
        QS_ARG(r[3] == 1.0, "sos rows must have a0 == 1");
        p.b0[s] = r[0]; p.b1[s] = r[1]; p.b2[s] = r[2];
        p.a1[s] = r[4]; p.a2[s] = r[5];
        p.zi0[s] = zi_host[2 * s];
        p.zi1[s] = zi_host[2 * s + 1];
    }
    const int D = 2 * p.S;
    const uint64_t m = n + 2 * pad;
    const uint64_t nch = (m + FCHUNK - 1) / FCHUNK, ng = (nch + FGROUP - 1) / FGROUP;
    // transition powers: one chunk, one group, the last (shorter) group
    std::vector<double> M, PL, PG, PGl;
    cascade_matrix(p, M);
    matpow(M, D, FCHUNK, PL);
    matpow(PL, D, FGROUP, PG);
    matpow(PL, D, nch - (ng - 1) * FGROUP, PGl);
    // (the last chunk may be short; its power is never applied to a carried state)
    unsigned char* w = (unsigned char*)ws_dev;
    double* yf = (double*)w;
    double* fstate = (double*)(((uintptr_t)(yf + m) + 255) & ~(uintptr_t)255);
    double* gstate = fstate + nch * 2 * FMAX_S;
    double* mats = gstate + ng * 2 * FMAX_S;  // PL | PG | PGl | s0
    double* dPL = mats;
    double* dPG = mats + FMAX_S * FMAX_S * 4;
    double* dPGl = dPG + FMAX_S * FMAX_S * 4;
    double* ds0 = dPGl + FMAX_S * FMAX_S * 4;
    QS_CUDA(cudaMemcpyAsync(dPL, PL.data(), PL.size() * 8, cudaMemcpyHostToDevice, st), "copy");
    QS_CUDA(cudaMemcpyAsync(dPG, PG.data(), PG.size() * 8, cudaMemcpyHostToDevice, st), "copy");
    QS_CUDA(cudaMemcpyAsync(dPGl, PGl.data(), PGl.size() * 8, cudaMemcpyHostToDevice, st), "copy");
    const unsigned gc = qs_blocks(nch, 128), gg = qs_blocks(ng, 128);
    for (int pass = 0; pass < 2; ++pass) {
        PassIn in{pass == 0 ? x_dev : yf, n, pad, m, pass};
        k_iir_chunk_final<<<gc, 128, 0, st>>>(p, in, nch, fstate);
        k_iir_group_final<<<gg, 128, 0, st>>>(dPL, D, nch, fstate, gstate);
        // entry state of the pass: zi scaled by the first input value (on device)
        k_iir_init_state<<<1, 32, 0, st>>>(p, in, ds0);
        k_iir_group_scan<<<1, 1, 0, st>>>(dPG, dPGl, D, ng, ds0, gstate);
        k_iir_chunk_entry<<<gg, 128, 0, st>>>(dPL, D, nch, gstate, fstate);
        if (pass == 0)
            k_iir_chunk_out<<<gc, 128, 0, st>>>(p, in, nch, fstate, yf, 0, m, 0);
        else
            k_iir_chunk_out<<<gc, 128, 0, st>>>(p, in, nch, fstate, out_dev, pad, pad + n, 1);
        QS_CHECK_LAUNCH("sosfiltfilt pass");
    }
    return QS_OK;
}

}  // extern "C"
