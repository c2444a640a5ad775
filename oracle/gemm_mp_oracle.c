/*
 * gemm_mp_oracle.c -- plain, slow CPU oracle for the tile-centric mixed-precision
 * GEMM  C <- alpha*A*B + beta*C  of arxiv 2508.14848 (Algorithm 1,
 * PAPER.md:104-117, 144-148).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_2508_14848_b200/) never links, imports or calls it, and this file shares
 * no code, header, table or constant generator with the CUDA path.
 *
 * Build: gcc -O2 -ffp-contract=off -fopenmp -shared -fPIC (no -ffast-math, no
 * -march=native): every floating-point operation below is one IEEE-754 binary64
 * or binary32 operation with round-to-nearest-even, and every fused multiply-add
 * is an explicit fma()/fmaf() call.
 *
 * What it follows (readings are listed in DESIGN.md "Readings"):
 *   - Algorithm 1 loop, per-operand tile precisions #,$,*   PAPER.md:104-117, 146
 *   - receiver-side conversion, flows in stored precision   PAPER.md:148  (R7)
 *   - fixed square tiles nb, 2D block-cyclic P x Q
 *   - tile-norm precision criterion                         PAPER.md:78 refs (R1-R5)
 *   - lower-of-operands compute precision, accumulation     north_star   (R6, R8)
 *   - every formula is in DESIGN.md section "Oracle definitions" (O1..O9).
 *
 * Parity status: every exported function here is pinned by tests/test_oracle_*.py
 * (exhaustive converters, Fraction references, closed-form maps, brute force).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------------------- */
/* O1. Counter-based SplitMix64 synthetic generator (SPEC.md:63-89 recurrence; */
/*     counter form: output i of seed s is mix(s + i*gamma)).  DESIGN.md O1.    */
/* ------------------------------------------------------------------------- */
#define ORC_GAMMA 0x9E3779B97F4A7C15ULL

uint64_t orc_mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

/* i-th output (i >= 1) of the SplitMix64 stream seeded with `seed` */
uint64_t orc_splitmix_output(uint64_t seed, uint64_t i) {
    return orc_mix64(seed + i * ORC_GAMMA);
}

/* ((u >> 11) * 2^-53) * 2 - 1, exact in binary64 */
double orc_uniform(uint64_t u) {
    return ((double)(u >> 11) * 0x1p-53) * 2.0 - 1.0;
}

/* per-tile exponent e(ti,tj) of the synthetic recipe */
int orc_synth_tile_exp(int mode, int E, uint64_t tau, int64_t ti, int64_t tj,
                       int64_t mt, int64_t nt) {
    if (mode == 0) return 0;                                 /* uniform */
    if (mode == 1) {                                         /* graded  */
        int64_t den = mt + nt - 2;
        if (den < 1) den = 1;
        return (int)(((ti + tj) * (int64_t)E) / den);
    }
    /* random */
    uint64_t u = orc_splitmix_output(tau, (uint64_t)(ti * nt + tj) + 1u);
    return (int)(u % (uint64_t)(E + 1));
}

/* x(r,c) = v(r,c) * 2^(s - e(r/nb, c/nb)) over the sub-block rows [r0,r0+nr),
 * cols [c0,c0+nc) of a rows x cols matrix; written row-major with leading dim ld. */
void orc_synth_block(int64_t rows, int64_t cols, int32_t nb, uint64_t seed, int mode,
                     int E, int s, uint64_t tau, int64_t r0, int64_t nr, int64_t c0,
                     int64_t nc, double *out, int64_t ld) {
    int64_t mt = rows / nb, nt = cols / nb;
    for (int64_t r = 0; r < nr; ++r) {
        for (int64_t c = 0; c < nc; ++c) {
            int64_t gr = r0 + r, gc = c0 + c;
            uint64_t u = orc_splitmix_output(seed, (uint64_t)(gr * cols + gc) + 1u);
            double v = orc_uniform(u);
            int e = orc_synth_tile_exp(mode, E, tau, gr / nb, gc / nb, mt, nt);
            out[r * ld + c] = ldexp(v, s - e);
        }
    }
}

/* ------------------------------------------------------------------------- */
/* O2. Number formats and round-to-nearest-even from binary64 (O2).  */
/*     Class codes: 0 FP64, 1 FP32, 2 FP16, 3 BF16, 4 E4M3 (OCP "FN"),         */
/*     5 E5M2 (OCP, IEEE-like inf/NaN).  Codes are ordered by */
/*     unit roundoff, so a pair's class is max(code_A, code_B).                   */
/* ------------------------------------------------------------------------- */
typedef struct {
    int p;          /* fraction (trailing significand) bits          */
    int ebits;      /* exponent field bits                           */
    int bias;
    int emin;       /* exponent of the smallest normal               */
    double maxval;  /* largest finite value                          */
    int satfinite;  /* 1: overflow saturates to +-maxval (E4M3 FN)   */
    double u;       /* unit roundoff 2^-(p+1)                        */
    double eta;     /* smallest positive subnormal                   */
    double omega_s; /* per-tile scale target Omega' (R10)  */
    int bytes;
} orc_fmt_t;

#define ORC_NCLS 7
#define ORC_MX 6   /* MXFP4 (OCP MX: E2M1 elements, one E8M0 scale per 32 K-elements), R31 */
static const orc_fmt_t ORC_FMT[ORC_NCLS] = {
    /* FP64 */ {52, 11, 1023, -1022, 0x1.fffffffffffffp+1023, 0, 0x1p-53, 0x1p-1074, 0.0, 8},
    /* FP32 */ {23, 8, 127, -126, 0x1.fffffep+127, 0, 0x1p-24, 0x1p-149, 1.0, 4},
    /* FP16 */ {10, 5, 15, -14, 65504.0, 0, 0x1p-11, 0x1p-24, 65504.0, 2},
    /* BF16 */ {7, 8, 127, -126, 0x1.fep+127, 0, 0x1p-8, 0x1p-133, 1.0, 2},
    /* E4M3 */ {3, 4, 7, -6, 448.0, 1, 0x1p-4, 0x1p-9, 448.0, 1},
    /* E5M2 */ {2, 5, 15, -14, 57344.0, 0, 0x1p-3, 0x1p-16, 57344.0, 1},
    /* MXFP4 element E2M1: no inf/NaN, max 6, subnormal 0.5; bytes: see orc_payload_bytes */
    /* MX4  */ {1, 2, 1, 0, 6.0, 1, 0x1p-2, 0.5, 1.0, 0},
};

int orc_class_bytes(int cls) { return ORC_FMT[cls].bytes; }
/* bytes of one nb x nb payload: nb^2 x bytes, or for MXFP4 nb^2/2 element bytes (two
 * E2M1 codes per byte) followed by nb^2/32 E8M0 scale bytes (R31) */
int64_t orc_payload_bytes(int cls, int32_t nb) {
    int64_t n = (int64_t)nb * nb;
    return cls == ORC_MX ? n / 2 + n / 32 : n * ORC_FMT[cls].bytes;
}
double orc_class_u(int cls) { return ORC_FMT[cls].u; }
double orc_class_eta(int cls) { return ORC_FMT[cls].eta; }
double orc_class_omega_scale(int cls) { return ORC_FMT[cls].omega_s; }

/* Round |x| (finite, > 0) to nearest-even in format f; returns the rounded value
 * (may exceed maxval: the caller handles overflow).  Written out from the
 * definition: pick the quantum 2^q of the binade (or of the subnormal range),
 * take n = x / 2^q exactly, round n to an integer with ties to even. */
static double orc_rne_abs(double a, const orc_fmt_t *f) {
    int E;
    (void)frexp(a, &E);           /* a = m 2^E, m in [0.5,1)  =>  a in [2^(E-1), 2^E) */
    int ex = E - 1;
    int q = (ex < f->emin ? f->emin : ex) - f->p;
    double n = ldexp(a, -q);      /* exact: scaling by a power of two          */
    double fl = floor(n);
    double fr = n - fl;           /* exact                                    */
    if (fr > 0.5 || (fr == 0.5 && fmod(fl, 2.0) != 0.0)) fl += 1.0;
    return ldexp(fl, q);          /* exact: fl has at most p+2 bits            */
}

/* Encode binary64 x into class cls (1..6) with one RNE rounding; bits in the
 * low bytes of the return value. NaN -> canonical NaN; overflow -> inf (FP32,
 * FP16, BF16, E5M2) or saturate to +-448 (E4M3, "satfinite") / +-6 (E2M1, the MXFP4
 * element, which has no inf/NaN); both unreachable after the scaling of R10 / R31. */
uint32_t orc_encode(double x, int cls) {
    const orc_fmt_t *f = &ORC_FMT[cls];
    uint32_t sign = signbit(x) ? 1u : 0u;
    uint32_t sshift = (uint32_t)(f->ebits + f->p);
    uint32_t expmax = (1u << f->ebits) - 1u;
    if (isnan(x)) {
        if (cls == 4) return (sign << 7) | 0x7Fu;
        return (sign << sshift) | (expmax << f->p) | (1u << (f->p - 1));
    }
    double a = fabs(x);
    if (a == 0.0) return sign << sshift;
    double r = isinf(a) ? INFINITY : orc_rne_abs(a, f);
    if (r > f->maxval) {
        if (f->satfinite) r = f->maxval;
        else return (sign << sshift) | (expmax << f->p);   /* +-inf */
    }
    if (r == 0.0) return sign << sshift;
    int E;
    (void)frexp(r, &E);
    int ex = E - 1;
    uint32_t biased, mant;
    if (ex < f->emin) {           /* subnormal: r = mant * 2^(emin-p) */
        biased = 0;
        mant = (uint32_t)ldexp(r, f->p - f->emin);
    } else {
        biased = (uint32_t)(ex + f->bias);
        mant = (uint32_t)(ldexp(r, f->p - ex) - ldexp(1.0, f->p));
    }
    return (sign << sshift) | (biased << f->p) | mant;
}

/* Decode class-cls bits to the exact binary64 value. */
double orc_decode(uint32_t bits, int cls) {
    const orc_fmt_t *f = &ORC_FMT[cls];
    uint32_t sshift = (uint32_t)(f->ebits + f->p);
    uint32_t sign = (bits >> sshift) & 1u;
    uint32_t expmax = (1u << f->ebits) - 1u;
    uint32_t biased = (bits >> f->p) & expmax;
    uint32_t mant = bits & ((1u << f->p) - 1u);
    double v;
    if (cls == 4 && biased == expmax && mant == 7u) v = NAN;
    else if (cls != 4 && cls != ORC_MX && biased == expmax) v = mant ? NAN : INFINITY;
    else if (biased == 0) v = ldexp((double)mant, f->emin - f->p);
    else v = ldexp((double)(mant + (1u << f->p)), (int)biased - f->bias - f->p);
    return sign ? -v : v;
}

/* ------------------------------------------------------------------------- */
/* O3. Per-tile power-of-two scale (R10): the largest integer e with */
/*     maxabs * 2^e <= Omega'_k.  maxabs == 0 -> 0.  FP64 -> 0.                */
/* ------------------------------------------------------------------------- */
int orc_scale_exp(double maxabs, int cls) {
    if (cls == 0 || maxabs == 0.0) return 0;
    /* direct search from the definition: start from the frexp estimate and
     * step until maxabs*2^e <= Omega' < maxabs*2^(e+1). Exact comparisons. */
    int E;
    (void)frexp(maxabs, &E);
    int Eo;
    (void)frexp(ORC_FMT[cls].omega_s, &Eo);
    int e = Eo - E + 1;
    while (!(ldexp(maxabs, e) <= ORC_FMT[cls].omega_s)) --e;
    while (ldexp(maxabs, e + 1) <= ORC_FMT[cls].omega_s) ++e;
    return e;
}

/* O3 for the MXFP4 block scale (reading R31): the smallest integer s >= -127 with
 * amax <= 6 * 2^s (6 = largest E2M1 value), so no element of the block saturates;
 * amax == 0 -> -127.  Stored as the E8M0 byte s + 127. */
int orc_mx_block_exp(double amax) {
    if (amax == 0.0) return -127;
    int E;
    (void)frexp(amax, &E);
    int s = E - 2;
    while (s > -127 && ldexp(6.0, s - 1) >= amax) --s;
    while (ldexp(6.0, s) < amax) ++s;
    return s < -127 ? -127 : s;
}

/* O6 for MXFP4: y[idx] (scaled units, payload-index order idx = mn*nb + k, K-major)
 * -> payload: block b = idx / 32 (32 consecutive K-elements of one row) gets
 * s_b = orc_mx_block_exp(max |y| over the block); element code q = RN_E2M1(y 2^-s_b)
 * in nibble idx (byte idx/2, low nibble for even idx); E8M0 byte s_b + 127 at
 * offset nb^2/2 + b. */
void orc_mx_encode(const double *y, int32_t nb, uint8_t *payload) {
    int64_t n = (int64_t)nb * nb;
    for (int64_t b = 0; b < n / 32; ++b) {
        double amax = 0.0;
        for (int v = 0; v < 32; ++v) {
            double a = fabs(y[b * 32 + v]);
            if (a > amax) amax = a;
        }
        int sb = orc_mx_block_exp(amax);
        payload[n / 2 + b] = (uint8_t)(sb + 127);
        for (int v = 0; v < 32; v += 2) {
            uint32_t q0 = orc_encode(ldexp(y[b * 32 + v], -sb), ORC_MX);
            uint32_t q1 = orc_encode(ldexp(y[b * 32 + v + 1], -sb), ORC_MX);
            payload[(b * 32 + v) / 2] = (uint8_t)((q0 & 15u) | ((q1 & 15u) << 4));
        }
    }
}

/* ------------------------------------------------------------------------- */
/* O4. Canonical tile sum of squares CNORM (O4).                     */
/*   256 lanes x 2 slots; lane t slot s accumulates x_q^2 by fma for            */
/*   q = 2t + s + 512w, w = 0,1,...; t[lane] = a0 + a1; butterfly inside each   */
/*   32-lane warp over offsets 16,8,4,2,1 (t <- t + t[lane ^ off]); then        */
/*   S = ((w0 + w1) + ...) + w7 over the eight warp results.                   */
/* ------------------------------------------------------------------------- */
double orc_cnorm(const double *tile, int64_t ld, int32_t nb) {
    double acc[256][2];
    int64_t n = (int64_t)nb * nb;
    for (int t = 0; t < 256; ++t) acc[t][0] = acc[t][1] = 0.0;
    for (int64_t base = 0; base < n; base += 512) {
        for (int t = 0; t < 256; ++t) {
            for (int s = 0; s < 2; ++s) {
                int64_t q = base + 2 * t + s;
                double x = tile[(q / nb) * ld + (q % nb)];
                acc[t][s] = fma(x, x, acc[t][s]);
            }
        }
    }
    double lane[256], nxt[256];
    for (int t = 0; t < 256; ++t) lane[t] = acc[t][0] + acc[t][1];
    for (int off = 16; off >= 1; off /= 2) {
        for (int t = 0; t < 256; ++t) nxt[t] = lane[t] + lane[t ^ off];
        memcpy(lane, nxt, sizeof lane);
    }
    double S = lane[0];
    for (int w = 1; w < 8; ++w) S = S + lane[32 * w];
    return S;
}

/* Stats of every tile of an (mt*nb) x (nt*nb) row-major matrix. finite[t] = 0 if
 * the tile holds a NaN or an infinity. Arrays are mt*nt, row-major tile order. */
static void orc_one_tile_stats(const double *tp, int64_t ld, int32_t nb, double *S, double *maxabs,
                               uint8_t *finite) {
    double m = 0.0;
    int fin = 1;
    for (int32_t r = 0; r < nb; ++r)
        for (int32_t c = 0; c < nb; ++c) {
            double a = fabs(tp[(int64_t)r * ld + c]);
            if (!isfinite(a)) fin = 0;
            else if (a > m) m = a;
        }
    *maxabs = m;
    *finite = (uint8_t)fin;
    *S = fin ? orc_cnorm(tp, ld, nb) : NAN;
}

void orc_tile_stats(const double *X, int64_t ld, int64_t mt, int64_t nt, int32_t nb,
                    double *S, double *maxabs, uint8_t *finite) {
#pragma omp parallel for schedule(dynamic)
    for (int64_t t = 0; t < mt * nt; ++t) {
        int64_t ti = t / nt, tj = t % nt;
        orc_one_tile_stats(X + ti * nb * ld + tj * nb, ld, nb, S + t, maxabs + t, finite + t);
    }
}

/* ------------------------------------------------------------------------- */
/* O5. Precision map for an input matrix A or B (O5, readings R1-R5, */
/*     R13, R14, R31).  Ladder: MXFP4, E5M2, E4M3, BF16, FP16, FP32, FP64        */
/*     (enabled classes; lowest precision first); first eligible wins.         */
/* ------------------------------------------------------------------------- */
static const int ORC_LADDER[ORC_NCLS] = {6, 5, 4, 3, 2, 1, 0};

/* delta_k = u_k + sqrt(nb) * u_acc(k); u_acc = u64 for FP64, u32 otherwise */
double orc_delta(int cls, int32_t nb) {
    double uacc = (cls == 0) ? 0x1p-53 : 0x1p-24;
    return ORC_FMT[cls].u + sqrt((double)nb) * uacc;
}

/* Returns 0 on success, 1 if a tile is non-finite (GMP_ERR_NONFINITE). */
int orc_map_input(int64_t mt, int64_t nt, int32_t nb, double tol, uint32_t class_mask,
                  const double *S, const double *maxabs, const uint8_t *finite,
                  uint8_t *code, int16_t *scale) {
    int64_t ntiles = mt * nt;
    for (int64_t t = 0; t < ntiles; ++t)
        if (!finite[t]) return 1;
    double SX = 0.0;                                     /* sequential, row-major */
    for (int64_t t = 0; t < ntiles; ++t) SX = SX + S[t];
    double nrm = sqrt(SX);
    double NT = sqrt((double)ntiles);
    double eps = tol / 4.0;
    double rhs = (eps * nrm) / NT;
    uint32_t mask = class_mask | 1u;
    for (int64_t t = 0; t < ntiles; ++t) {
        int chosen = 0;
        if (!isinf(SX)) {
            for (int li = 0; li < ORC_NCLS; ++li) {
                int k = ORC_LADDER[li];
                if (!(mask & (1u << k))) continue;
                if (k == 0) { chosen = 0; break; }
                if (maxabs[t] == 0.0) { chosen = k; break; }
                int e = orc_scale_exp(maxabs[t], k);
                /* underflow term: nb x half the subnormal quantum of the tile's scaled
                 * grid; for MXFP4 the quantum of the block holding the tile's max
                 * (every block's scale is <= it; R31) */
                int qe = k == ORC_MX ? orc_mx_block_exp(ldexp(maxabs[t], e)) : 0;
                double lhs = orc_delta(k, nb) * sqrt(S[t]) +
                             (double)nb * ldexp(ORC_FMT[k].eta, qe - e - 1);
                if (lhs <= rhs) { chosen = k; break; }
            }
        }
        code[t] = (uint8_t)chosen;
        scale[t] = (int16_t)orc_scale_exp(maxabs[t], chosen);
    }
    return 0;
}

/* ------------------------------------------------------------------------- */
/* O6. Packing and receiver-side shadows (O6, R7).     */
/* ------------------------------------------------------------------------- */
static void orc_store_elem(void *payload, int64_t idx, int cls, double x) {   /* cls != MX */
    if (cls == 0) { ((double *)payload)[idx] = x; return; }
    uint32_t b = orc_encode(x, cls);
    if (cls == 1) ((uint32_t *)payload)[idx] = b;
    else if (cls >= 4) ((uint8_t *)payload)[idx] = (uint8_t)b;
    else ((uint16_t *)payload)[idx] = (uint16_t)b;
}

/* exact binary64 value of payload element idx (scaled units); nb locates the
 * MXFP4 scale bytes (value = E2M1(q) x 2^s_b) */
double orc_payload_value(const void *payload, int32_t nb, int64_t idx, int cls) {
    if (cls == 0) return ((const double *)payload)[idx];
    if (cls == ORC_MX) {
        const uint8_t *p = (const uint8_t *)payload;
        uint32_t q = (p[idx / 2] >> (4 * (idx & 1))) & 15u;
        int sb = (int)p[(int64_t)nb * nb / 2 + idx / 32] - 127;
        return ldexp(orc_decode(q, ORC_MX), sb);
    }
    uint32_t b;
    if (cls == 1) b = ((const uint32_t *)payload)[idx];
    else if (cls >= 4) b = ((const uint8_t *)payload)[idx];
    else b = ((const uint16_t *)payload)[idx];
    return orc_decode(b, cls);
}

/* Payload layout (O6 "Packed layout"): element (r,c) of a tile is at
 * payload[r*nb + c] (not transposed) or payload[c*nb + r] (transposed).
 *   FP64 / FP32 classes: MN-major operands -- A transposed (column-major), B not;
 *   FP16 / BF16 / E4M3 / E5M2 classes: K-major operands -- A not transposed, B transposed;
 *   C tiles (packed C_in / C_out): not transposed.
 * role: 0 = A, 1 = B, 2 = C. */
int orc_layout_transposed(int role, int cls) {
    if (role == 2) return 0;
    int mn_major = cls <= 1;
    return role == 0 ? mn_major : !mn_major;
}

/* Stored payload of one tile: element (r,c) of the tile is RN_cls(x(r,c) 2^scale),
 * written at the index given by `transpose` (see orc_layout_transposed); MXFP4:
 * y = x 2^scale block-encoded by orc_mx_encode. */
void orc_pack_tile(const double *X, int64_t ld, int32_t nb, int cls, int scale,
                   int transpose, void *payload) {
    if (cls == ORC_MX) {
        double *y = (double *)malloc(sizeof(double) * nb * nb);
        for (int32_t r = 0; r < nb; ++r)
            for (int32_t c = 0; c < nb; ++c)
                y[transpose ? (int64_t)c * nb + r : (int64_t)r * nb + c] = ldexp(X[(int64_t)r * ld + c], scale);
        orc_mx_encode(y, nb, (uint8_t *)payload);
        free(y);
        return;
    }
    for (int32_t r = 0; r < nb; ++r)
        for (int32_t c = 0; c < nb; ++c) {
            double x = X[(int64_t)r * ld + c];
            double y = (cls == 0) ? x : ldexp(x, scale);
            int64_t idx = transpose ? (int64_t)c * nb + r : (int64_t)r * nb + c;
            orc_store_elem(payload, idx, cls, y);
        }
}

/* Shadow of a stored tile: decode the stored payload (class `from`, scale e_from),
 * take its maxabs, choose the class-`to` scale for the decoded tile, round once
 * from the decoded value.  Returns the shadow scale e_to = e_from + d. */
int orc_shadow_tile(const void *payload, int32_t nb, int role, int from, int from_scale, int to,
                    void *out) {
    int64_t n = (int64_t)nb * nb;
    double m = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        double a = fabs(orc_payload_value(payload, nb, i, from));
        if (a > m) m = a;
    }
    /* decoded tile = w * 2^-from_scale; its scale for class `to` is
     * orc_scale_exp(m * 2^-from_scale, to) = from_scale + orc_scale_exp(m, to)  */
    int d = orc_scale_exp(m, to);
    int tf = orc_layout_transposed(role, from), tt = orc_layout_transposed(role, to);
    double *y = to == ORC_MX ? (double *)malloc(sizeof(double) * n) : NULL;
    for (int32_t r = 0; r < nb; ++r)
        for (int32_t c = 0; c < nb; ++c) {
            int64_t src = tf ? (int64_t)c * nb + r : (int64_t)r * nb + c;
            int64_t dst = tt ? (int64_t)c * nb + r : (int64_t)r * nb + c;
            double v = ldexp(orc_payload_value(payload, nb, src, from), d);
            if (y) y[dst] = v;
            else orc_store_elem(out, dst, to, v);
        }
    if (y) { orc_mx_encode(y, nb, (uint8_t *)out); free(y); }
    return from_scale + d;
}

/* ------------------------------------------------------------------------- */
/* O7. Precision map for C (output estimate; O7, R9, R23).          */
/* ascale/bscale: [tile][6] class-c scales of A and B tiles (stored or shadow)*/
/* for every c >= code; entries for c < code are ignored.                      */
/* ------------------------------------------------------------------------- */
int orc_map_c(int64_t mt, int64_t nt, int64_t kt, int32_t nb, double tol, double alpha,
              double beta, uint32_t class_mask, const double *SA, const double *SB,
              const double *SC, const uint8_t *finiteC, const uint8_t *acode,
              const int16_t *ascale, const uint8_t *bcode, const int16_t *bscale,
              uint8_t *code, const uint8_t *cmap) {
    if (beta != 0.0)
        for (int64_t t = 0; t < mt * nt; ++t)
            if (!finiteC[t]) return 1;
    double sA = 0.0, sB = 0.0, sC = 0.0;
    for (int64_t t = 0; t < mt * kt; ++t) sA = sA + SA[t];
    for (int64_t t = 0; t < kt * nt; ++t) sB = sB + SB[t];
    if (beta != 0.0)
        for (int64_t t = 0; t < mt * nt; ++t) sC = sC + SC[t];
    double nA = sqrt(sA), nB = sqrt(sB), nC = sqrt(sC);
    double aa = fabs(alpha), ab = fabs(beta);
    double Nhat = (aa * nA) * nB + ab * nC;
    double NT = sqrt((double)(mt * nt));
    double rhs = ((tol / 2.0) * Nhat) / NT;
    double sqkt = sqrt((double)kt);
    uint32_t mask = class_mask | 1u;
    for (int64_t i = 0; i < mt; ++i) {
        double RA = 0.0;
        for (int64_t l = 0; l < kt; ++l) RA = RA + SA[i * kt + l];
        RA = sqrt(RA);
        for (int64_t j = 0; j < nt; ++j) {
            double QB = 0.0;
            for (int64_t l = 0; l < kt; ++l) QB = QB + SB[l * nt + j];
            QB = sqrt(QB);
            double sc = (beta != 0.0) ? SC[i * nt + j] : 0.0;
            double nhat = (aa * RA) * QB + ab * sqrt(sc);
            int chosen = 0;
            if (cmap) {                   /* explicit map (R19): the code, if enabled */
                chosen = cmap[i * nt + j];
                if (!(mask & (1u << chosen)) || chosen == ORC_MX) chosen = 0;
            } else {
                for (int li = 0; li < ORC_NCLS; ++li) {
                    int k = ORC_LADDER[li];
                    if (!(mask & (1u << k)) || k == ORC_MX) continue;   /* MX: operands only (R31) */
                    if (k == 0) { chosen = 0; break; }
                    double dC = (ORC_FMT[k].u + sqkt * 0x1p-24) +
                                ((double)nb * ORC_FMT[k].eta) / ORC_FMT[k].omega_s;
                    if (dC * nhat <= rhs) { chosen = k; break; }
                }
            }
            /* R23: FP32 accumulator range guards -- for explicit codes too: a binary32
             * W cannot hold an output or fold factor outside its range */
            if (chosen != 0) {
                int ok = (nhat <= 0x1p100);
                if (beta != 0.0) {
                    double bf = (double)(float)beta;
                    if (!(fabs(bf) >= 0x1p-126 && fabs(bf) <= 0x1p100)) ok = 0;
                }
                for (int64_t l = 0; ok && l < kt; ++l) {
                    int ca = acode[i * kt + l], cb = bcode[l * nt + j];
                    int c = ca > cb ? ca : cb;
                    int ea = ascale[(i * kt + l) * ORC_NCLS + c], eb = bscale[(l * nt + j) * ORC_NCLS + c];
                    double fct = ldexp(alpha, -(ea + eb));
                    if (fct != 0.0 && !(fabs(fct) >= 0x1p-126 && fabs(fct) <= 0x1p100)) ok = 0;
                }
                if (!ok) chosen = 0;
            }
            code[i * nt + j] = (uint8_t)chosen;
        }
    }
    return 0;
}

/* ------------------------------------------------------------------------- */
/* O8. Tile-GEMM emulation for pair class c (O8, R6, R8).            */
/*   a, b: class-c payloads of the A and B tiles in the layout of            */
/*   orc_layout_transposed (read as a[r][p] and b[p][col]).                   */
/*   P[r][col] = sum_p a[r][p] b[p][col], sequential p = 0..nb-1, from +0:    */
/*     c = 0: binary64 fma;  c = 1: binary32 fmaf;                            */
/*     c >= 2: binary32 acc + RN32(a*b) (the product is exact in binary32 for  */
/*     c = 2..5; for MXFP4, c = 6, when the two block scales sum below -149). */
/*   P is returned as binary64 (exact copies of the binary32 values if c>=1). */
/* ------------------------------------------------------------------------- */
void orc_tile_gemm(int cls, const void *a, const void *b, int32_t nb, double *P) {
    int64_t n = (int64_t)nb * nb;
    double *av = (double *)malloc(sizeof(double) * n);
    double *bv = (double *)malloc(sizeof(double) * n);
    int ta = orc_layout_transposed(0, cls), tb = orc_layout_transposed(1, cls);
    for (int32_t r = 0; r < nb; ++r)         /* av[r*nb + p] = A(r,p), bv[col*nb + p] = B(p,col) */
        for (int32_t p = 0; p < nb; ++p) {
            av[(int64_t)r * nb + p] =
                orc_payload_value(a, nb, ta ? (int64_t)p * nb + r : (int64_t)r * nb + p, cls);
            bv[(int64_t)r * nb + p] =
                orc_payload_value(b, nb, tb ? (int64_t)r * nb + p : (int64_t)p * nb + r, cls);
        }
    for (int32_t r = 0; r < nb; ++r) {
        for (int32_t col = 0; col < nb; ++col) {
            const double *ar = av + (int64_t)r * nb;
            const double *bc = bv + (int64_t)col * nb;
            if (cls == 0) {
                double acc = 0.0;
                for (int32_t p = 0; p < nb; ++p) acc = fma(ar[p], bc[p], acc);
                P[(int64_t)r * nb + col] = acc;
            } else if (cls == 1) {
                float acc = 0.0f;
                for (int32_t p = 0; p < nb; ++p) acc = fmaf((float)ar[p], (float)bc[p], acc);
                P[(int64_t)r * nb + col] = (double)acc;
            } else {
                float acc = 0.0f;
                for (int32_t p = 0; p < nb; ++p) {
                    float prod = (float)ar[p] * (float)bc[p];
                    acc = acc + prod;
                }
                P[(int64_t)r * nb + col] = (double)acc;
            }
        }
    }
    free(av);
    free(bv);
}

/* ------------------------------------------------------------------------- */
/* O9. Accumulator init, fold and finalize for one C tile (O9, R15). */
/*   W = binary64 if code_C == 0 else binary32; acc kept as binary64 array     */
/*   holding exact W values.                                                  */
/* ------------------------------------------------------------------------- */
#define ORC_STEP_DEPTH 8

/* acc = beta == 0 ? 0 : RN_W(RN_W(beta) * decode(packed C_in)) */
void orc_acc_init(int32_t nb, int code_c, double beta, const void *cin_payload,
                  int cin_scale, double *acc) {
    int64_t n = (int64_t)nb * nb;
    for (int64_t i = 0; i < n; ++i) {
        if (beta == 0.0) { acc[i] = 0.0; continue; }
        double x = ldexp(orc_payload_value(cin_payload, nb, i, code_c), -cin_scale);
        if (code_c == 0) acc[i] = beta * x;
        else acc[i] = (double)(float)((double)(float)beta * x);
    }
}

/* acc = fma_W(RN_W(alpha 2^-(ea+eb)), RN_W(P), acc) */
void orc_fold(int32_t nb, int code_c, double alpha, int ea, int eb, const double *P,
              double *acc) {
    int64_t n = (int64_t)nb * nb;
    double f = ldexp(alpha, -(ea + eb));
    for (int64_t i = 0; i < n; ++i) {
        if (code_c == 0) acc[i] = fma(f, P[i], acc[i]);
        else acc[i] = (double)fmaf((float)f, (float)P[i], (float)acc[i]);
    }
}

/* C_out = encode_code(acc) with the class scale of maxabs(acc); user C = decode.
 * Writes the packed payload (row-major) and the binary64 user tile (ld). */
int orc_finalize(int32_t nb, int code_c, const double *acc, void *payload, double *cuser,
                 int64_t ldc) {
    int64_t n = (int64_t)nb * nb;
    double m = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        double a = fabs(acc[i]);
        if (a > m) m = a;
    }
    int e = orc_scale_exp(m, code_c);
    for (int64_t i = 0; i < n; ++i) {
        double y = (code_c == 0) ? acc[i] : ldexp(acc[i], e);
        orc_store_elem(payload, i, code_c, y);
        double back = orc_payload_value(payload, nb, i, code_c);
        cuser[(i / nb) * ldc + (i % nb)] = (code_c == 0) ? back : ldexp(back, -e);
    }
    return e;
}

/* ------------------------------------------------------------------------- */
/* Whole-method driver over in-memory matrices (Algorithm 1)*/
/* ------------------------------------------------------------------------- */
typedef struct {
    int64_t M, N, K;
    int32_t nb;
    double tol, alpha, beta;
    uint32_t class_mask;
    const uint8_t *a_map, *b_map, *c_map; /* optional explicit codes (NULL = criterion) */
} orc_desc_t;

typedef struct {
    /* outputs sized by the caller: mt*kt, kt*nt, mt*nt */
    uint8_t *acode, *bcode, *ccode;
    int16_t *ascale5, *bscale5;   /* [tile][ORC_NCLS]: class-c scale for c >= code, else 0 */
    int16_t *cscale;              /* finalize scale of each computed C tile        */
    int16_t *cin_scale;           /* scale of packed C_in (beta != 0)              */
    double *SA, *MA, *SB, *MB, *SC, *MC;
    int threads;
    /* optional debug export: the final W accumulator of every
     * computed C tile, exact W values as binary64, row-major with leading dim ldw */
    double *W;
    int64_t ldw;
} orc_out_t;

/* Apply an explicit map (R19, NEXT-1): codes given, scales from the rule. */
static void orc_explicit_map(int64_t ntiles, const uint8_t *map, uint32_t class_mask,
                             const double *maxabs, uint8_t *code, int16_t *scale) {   /* A and B */
    for (int64_t t = 0; t < ntiles; ++t) {
        int c = map[t];
        if (!((class_mask | 1u) & (1u << c))) c = 0;
        code[t] = (uint8_t)c;
        scale[t] = (int16_t)orc_scale_exp(maxabs[t], c);
    }
}

/*
 * Where the driver reads an input tile from: an in-memory binary64 row-major matrix, or
 * the O1 synthetic generator (orc_synth_block), tile by tile, so that workloads larger than
 * host memory (N = 65536) never exist as a whole.  Either way the tile's values are the
 * same binary64 numbers.
 */
typedef struct {
    const double *X;            /* in-memory matrix (synth = 0) */
    int64_t ld;
    int synth;                  /* 1: generator below            */
    int64_t rows, cols;
    uint64_t seed, tau;
    int mode, E, s;
} orc_src_t;

/* tile (ti, tj): a pointer to its top-left element and its leading dimension; buf
 * (nb*nb doubles) receives generated tiles */
static const double *orc_src_tile(const orc_src_t *src, int32_t nb, int64_t ti, int64_t tj, double *buf,
                                  int64_t *ld) {
    if (!src->synth) {
        *ld = src->ld;
        return src->X + ti * nb * src->ld + tj * nb;
    }
    orc_synth_block(src->rows, src->cols, nb, src->seed, src->mode, src->E, src->s, src->tau, ti * nb, nb,
                    tj * nb, nb, buf, nb);
    *ld = nb;
    return buf;
}

static void orc_src_stats(const orc_src_t *src, int64_t mt, int64_t nt, int32_t nb, double *S, double *maxabs,
                          uint8_t *finite) {
#pragma omp parallel
    {
        double *buf = src->synth ? malloc(sizeof(double) * (size_t)nb * nb) : NULL;
#pragma omp for schedule(dynamic)
        for (int64_t t = 0; t < mt * nt; ++t) {
            int64_t ld;
            const double *tp = orc_src_tile(src, nb, t / nt, t % nt, buf, &ld);
            orc_one_tile_stats(tp, ld, nb, S + t, maxabs + t, finite + t);
        }
        free(buf);
    }
}

/*
 * Full method (Algorithm 1) over the tiles of A (M x K), B (K x N), C (M x N).
 * ctiles: list of n_ctiles C tile indices (i*nt + j) to compute (NULL = all).
 * compact = 0: Cout (ldo) and o->W (o->ldw) are full M x N arrays, listed tiles written
 * in place; compact = 1: the q-th listed tile goes to Cout + q*nb*nb and o->W + q*nb*nb
 * (leading dimension nb).  The tile-GEMMs of one C tile are independent and are computed
 * concurrently; their folds into W run one by one in the order of O9.
 * Returns 0, 1 (non-finite input) or 2 (bad arguments).
 */
static int orc_gemm_mp_core(const orc_desc_t *d, const orc_src_t *sA, const orc_src_t *sB, const orc_src_t *sC,
                            double *Cout, int64_t ldo, const int64_t *ctiles, int64_t n_ctiles, int compact,
                            orc_out_t *o) {
    int32_t nb = d->nb;
    if (nb <= 0 || d->M % nb || d->N % nb || d->K % nb) return 2;
    int64_t mt = d->M / nb, nt = d->N / nb, kt = d->K / nb;
    int64_t nA = mt * kt, nB = kt * nt, nC = mt * nt;
    int64_t tsz = (int64_t)nb * nb;
    uint8_t *fA = malloc(nA), *fB = malloc(nB), *fC = malloc(nC);
    orc_src_stats(sA, mt, kt, nb, o->SA, o->MA, fA);
    orc_src_stats(sB, kt, nt, nb, o->SB, o->MB, fB);
    if (d->beta != 0.0) orc_src_stats(sC, mt, nt, nb, o->SC, o->MC, fC);
    else for (int64_t t = 0; t < nC; ++t) { o->SC[t] = 0.0; o->MC[t] = 0.0; fC[t] = 1; }
    int16_t *sa = malloc(sizeof(int16_t) * nA), *sb = malloc(sizeof(int16_t) * nB);
    int rc = 0;
    if (d->a_map) {
        for (int64_t t = 0; t < nA; ++t) if (!fA[t]) rc = 1;
        orc_explicit_map(nA, d->a_map, d->class_mask, o->MA, o->acode, sa);
    } else rc |= orc_map_input(mt, kt, nb, d->tol, d->class_mask, o->SA, o->MA, fA, o->acode, sa);
    if (d->b_map) {
        for (int64_t t = 0; t < nB; ++t) if (!fB[t]) rc = 1;
        orc_explicit_map(nB, d->b_map, d->class_mask, o->MB, o->bcode, sb);
    } else rc |= orc_map_input(kt, nt, nb, d->tol, d->class_mask, o->SB, o->MB, fB, o->bcode, sb);
    if (rc) { free(fA); free(fB); free(fC); free(sa); free(sb); return 1; }

    /* Stored payloads and every shadow c > code (receiver-side, from stored).
     * Every tile is packed to learn its shadow scales (needed by the C map,
     * R23); payloads are kept only for the A row panels / B column panels the
     * listed C tiles consume. */
    uint8_t *needA = calloc((size_t)nA, 1), *needB = calloc((size_t)nB, 1);
    {
        int64_t nlist0 = ctiles ? n_ctiles : nC;
        for (int64_t q = 0; q < nlist0; ++q) {
            int64_t ct = ctiles ? ctiles[q] : q;
            for (int64_t l = 0; l < kt; ++l) {
                needA[(ct / nt) * kt + l] = 1;
                needB[l * nt + (ct % nt)] = 1;
            }
        }
    }
    void **Ap = calloc((size_t)nA * ORC_NCLS, sizeof(void *));
    void **Bp = calloc((size_t)nB * ORC_NCLS, sizeof(void *));
#pragma omp parallel
    {
    double *gbuf = (sA->synth || sB->synth) ? malloc(sizeof(double) * (size_t)tsz) : NULL;
#pragma omp for schedule(dynamic)
    for (int64_t t = 0; t < nA + nB; ++t) {
        int isB = t >= nA;
        int64_t tt = isB ? t - nA : t;
        int64_t ncols = isB ? nt : kt;
        int64_t ld;
        const double *tp = orc_src_tile(isB ? sB : sA, nb, tt / ncols, tt % ncols, gbuf, &ld);
        int code = isB ? o->bcode[tt] : o->acode[tt];
        int keep = isB ? needB[tt] : needA[tt];
        int16_t *s5 = isB ? o->bscale5 + tt * ORC_NCLS : o->ascale5 + tt * ORC_NCLS;
        void **pp = isB ? Bp + tt * ORC_NCLS : Ap + tt * ORC_NCLS;
        void *tmp = malloc((size_t)tsz * 8);
        for (int c = 0; c < ORC_NCLS; ++c) s5[c] = 0;
        s5[code] = isB ? sb[tt] : sa[tt];
        pp[code] = malloc((size_t)orc_payload_bytes(code, nb));
        orc_pack_tile(tp, ld, nb, code, s5[code], orc_layout_transposed(isB, code), pp[code]);
        for (int c = code + 1; c < ORC_NCLS; ++c) {
            void *dst = keep ? malloc((size_t)orc_payload_bytes(c, nb)) : tmp;
            s5[c] = (int16_t)orc_shadow_tile(pp[code], nb, isB, code, s5[code], c, dst);
            if (keep) pp[c] = dst;
        }
        if (!keep) { free(pp[code]); pp[code] = NULL; }
        free(tmp);
    }
    free(gbuf);
    }
    free(needA); free(needB);
    rc = orc_map_c(mt, nt, kt, nb, d->tol, d->alpha, d->beta, d->class_mask, o->SA,
                   o->SB, o->SC, fC, o->acode, o->ascale5, o->bcode, o->bscale5, o->ccode,
                   d->c_map);
    if (!rc) {
        int64_t nlist = ctiles ? n_ctiles : nC;
        int nthreads = 1;
#ifdef _OPENMP
        nthreads = omp_get_max_threads();
#endif
        double *acc = malloc(sizeof(double) * tsz);
        void *cpay = malloc((size_t)tsz * 8);
        void *cin = malloc((size_t)tsz * 8);
        double *cbuf = (sC->synth && d->beta != 0.0) ? malloc(sizeof(double) * tsz) : NULL;
        int64_t *pl = malloc(sizeof(int64_t) * (size_t)kt);   /* the tile's pairs in fold order */
        int *pc = malloc(sizeof(int) * (size_t)kt);
        double *P = malloc(sizeof(double) * (size_t)tsz * (size_t)kt);
        for (int64_t q = 0; q < nlist; ++q) {
            int64_t ct = ctiles ? ctiles[q] : q;
            int64_t i = ct / nt, j = ct % nt;
            int codec = o->ccode[ct];
            int cins = 0;
            if (d->beta != 0.0) {
                int64_t ldcin;
                const double *ctp = orc_src_tile(sC, nb, i, j, cbuf, &ldcin);
                cins = orc_scale_exp(o->MC[ct], codec);
                orc_pack_tile(ctp, ldcin, nb, codec, cins, 0, cin);
            }
            if (o->cin_scale) o->cin_scale[ct] = (int16_t)cins;
            orc_acc_init(nb, codec, d->beta, cin, cins, acc);
            /* O9 fold order: SUMMA step, class from high code to low, l ascending */
            int64_t np = 0;
            for (int64_t s0 = 0; s0 < kt; s0 += ORC_STEP_DEPTH) {
                int64_t s1 = s0 + ORC_STEP_DEPTH < kt ? s0 + ORC_STEP_DEPTH : kt;
                for (int c = ORC_NCLS - 1; c >= 0; --c)
                    for (int64_t l = s0; l < s1; ++l) {
                        int ca = o->acode[i * kt + l], cb = o->bcode[l * nt + j];
                        if ((ca > cb ? ca : cb) != c) continue;
                        pl[np] = l;
                        pc[np] = c;
                        ++np;
                    }
            }
#pragma omp parallel for schedule(dynamic)
            for (int64_t u = 0; u < np; ++u) {
                int64_t l = pl[u];
                int c = pc[u];
                orc_tile_gemm(c, Ap[(i * kt + l) * ORC_NCLS + c], Bp[(l * nt + j) * ORC_NCLS + c], nb,
                              P + u * tsz);
            }
            for (int64_t u = 0; u < np; ++u) {
                int64_t l = pl[u];
                int c = pc[u];
                orc_fold(nb, codec, d->alpha, o->ascale5[(i * kt + l) * ORC_NCLS + c],
                         o->bscale5[(l * nt + j) * ORC_NCLS + c], P + u * tsz, acc);
            }
            double *wdst = compact ? (o->W ? o->W + q * tsz : NULL) : (o->W ? o->W + i * nb * o->ldw + j * nb : NULL);
            int64_t ldw = compact ? nb : o->ldw;
            if (wdst)
                for (int64_t r = 0; r < nb; ++r) memcpy(wdst + r * ldw, acc + r * nb, sizeof(double) * nb);
            double *cdst = compact ? Cout + q * tsz : Cout + i * nb * ldo + j * nb;
            int e = orc_finalize(nb, codec, acc, cpay, cdst, compact ? nb : ldo);
            if (o->cscale) o->cscale[ct] = (int16_t)e;
        }
        free(acc); free(cpay); free(cin); free(cbuf); free(pl); free(pc); free(P);
        o->threads = nthreads;
    }
    for (int64_t t = 0; t < nA * ORC_NCLS; ++t) free(Ap[t]);
    for (int64_t t = 0; t < nB * ORC_NCLS; ++t) free(Bp[t]);
    free(Ap); free(Bp); free(fA); free(fB); free(fC); free(sa); free(sb);
    return rc;
}

int orc_gemm_mp(const orc_desc_t *d, const double *A, int64_t lda, const double *B,
                int64_t ldb, const double *C, int64_t ldc, double *Cout, int64_t ldo,
                const int64_t *ctiles, int64_t n_ctiles, orc_out_t *o) {
    orc_src_t sA = {A, lda, 0, 0, 0, 0, 0, 0, 0, 0};
    orc_src_t sB = {B, ldb, 0, 0, 0, 0, 0, 0, 0, 0};
    orc_src_t sC = {C, ldc, 0, 0, 0, 0, 0, 0, 0, 0};
    return orc_gemm_mp_core(d, &sA, &sB, &sC, Cout, ldo, ctiles, n_ctiles, 0, o);
}

/* The same method on the O1 synthetic workload, generated
 * tile by tile (A: M x K, B: K x N, C: M x N with the given seeds / modes / E / s / tau):
 * the listed C tiles are written compactly (Cout + q*nb*nb; o->W likewise when set). */
typedef struct { uint64_t seed, tau; int mode, E, s; } orc_synth_t;

int orc_gemm_mp_synth(const orc_desc_t *d, const orc_synth_t *ga, const orc_synth_t *gb, const orc_synth_t *gc,
                      double *Cout, const int64_t *ctiles, int64_t n_ctiles, orc_out_t *o) {
    orc_src_t sA = {NULL, 0, 1, d->M, d->K, ga->seed, ga->tau, ga->mode, ga->E, ga->s};
    orc_src_t sB = {NULL, 0, 1, d->K, d->N, gb->seed, gb->tau, gb->mode, gb->E, gb->s};
    orc_src_t sC = {NULL, 0, 1, d->M, d->N, gc->seed, gc->tau, gc->mode, gc->E, gc->s};
    return orc_gemm_mp_core(d, &sA, &sB, &sC, Cout, 0, ctiles, n_ctiles, 1, o);
}

int orc_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* array helpers for the test harness (element-wise O2) */
void orc_encode_array(const double *x, int64_t n, int cls, uint32_t *out) {
    for (int64_t i = 0; i < n; ++i) out[i] = orc_encode(x[i], cls);
}
void orc_decode_array(const uint32_t *b, int64_t n, int cls, double *out) {
    for (int64_t i = 0; i < n; ++i) out[i] = orc_decode(b[i], cls);
}
