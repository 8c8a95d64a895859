/*
 * synth.c — deterministic synthetic NetFlow workload.
 *
 * Bench/test input generator, not part of the analysed path. Counter-based:
 * record i depends only on (seed, index_offset + i), so any index shard of a
 * workload (multi-GPU D4, chunked oracle runs) is generated independently
 * and bit-identically, in parallel (OpenMP). The same bytes feed the GPU
 * (SoA) and the CPU reference (AoS), so parity never depends on host vs
 * device libm.
 *
 * Class mix follows toolkit.cpp:139-206 / flowmon.cpp:311-312 (reference
 * generator shapes), plus unmatched bulk traffic to exercise lookup misses:
 *   PureAck   pkts U[10,500], octets = 40*pkts, dur U[100,5000] ms
 *   Admin     pkts U[1,19], avg size U[100,500], dur U[100,5000] ms
 *   Forward   site endpoint (src or dst 50/50), rate ~ lognormal(mu, sigma)
 *             clamped to [1e3, 1.2e8] bps, dur U[1000,8000] ms, octets and
 *             pkts as toolkit.cpp:108-135 fill_forward(exact=false)
 *   Unmatched forward-shaped, both endpoints in 198.51.100.0/22
 * Site choice: uniform, or Zipf(s) over a seeded rank->site permutation.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct gnm_synth_spec {
    uint64_t seed;
    uint64_t n;              /* records to generate */
    uint64_t index_offset;   /* global index of the first record (sharding) */
    uint32_t n_sites;
    const uint32_t* site_base; /* first address of each site's CIDR */
    const uint32_t* site_size; /* addresses in each site's CIDR */
    double zipf_s;           /* 0 = uniform site choice */
    uint32_t hosts_per_site; /* distinct hosts per site (0 = whole CIDR) */
    double frac_ack, frac_admin, frac_fwd; /* rest: unmatched */
    double mu, sigma;        /* lognormal of the forward rate in bps */
    uint64_t window_start_ms, window_ms;
} gnm_synth_spec;

static inline uint64_t splitmix64(uint64_t* s) {
    uint64_t z = (*s += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
static inline double u01(uint64_t* s) { /* (0,1) */
    return ((double)(splitmix64(s) >> 11) + 0.5) * (1.0 / 9007199254740992.0);
}
static inline uint64_t uint_in(uint64_t* s, uint64_t lo, uint64_t hi) { /* [lo,hi] */
    return lo + splitmix64(s) % (hi - lo + 1);
}

#define REMOTE_BASE 0xC6336400u /* 198.51.100.0/22, never registered */

int gnm_synth_generate(const gnm_synth_spec* sp, uint32_t* src, uint32_t* dst, uint32_t* pkts,
                       uint32_t* octets, uint64_t* start, uint64_t* end) {
    if (!sp || (sp->n && (!src || !dst || !pkts || !octets || !start || !end))) return 1;
    if (sp->n_sites == 0 && sp->frac_fwd > 0) return 1;
    const uint32_t ns = sp->n_sites;
    /* rank -> site permutation and Zipf CDF */
    uint32_t* perm = (uint32_t*)malloc((ns ? ns : 1) * sizeof(uint32_t));
    double* cdf = (double*)malloc((ns ? ns : 1) * sizeof(double));
    if (!perm || !cdf) {
        free(perm);
        free(cdf);
        return 2;
    }
    uint64_t ps = sp->seed ^ 0x5EED5EED5EED5EEDull;
    for (uint32_t i = 0; i < ns; ++i) perm[i] = i;
    for (uint32_t i = ns; i > 1; --i) {
        const uint32_t j = (uint32_t)(splitmix64(&ps) % i);
        const uint32_t t = perm[i - 1];
        perm[i - 1] = perm[j];
        perm[j] = t;
    }
    double acc = 0;
    for (uint32_t r = 0; r < ns; ++r) {
        acc += sp->zipf_s > 0 ? pow((double)(r + 1), -sp->zipf_s) : 1.0;
        cdf[r] = acc;
    }
    for (uint32_t r = 0; r < ns; ++r) cdf[r] /= acc;

    const double t_ack = sp->frac_ack, t_admin = t_ack + sp->frac_admin,
                 t_fwd = t_admin + sp->frac_fwd;
    const long long n = (long long)sp->n;
#pragma omp parallel for schedule(static)
    for (long long i = 0; i < n; ++i) {
        uint64_t s = (sp->seed * 0xD1B54A32D192ED03ull) ^ ((sp->index_offset + (uint64_t)i) * 0x9E3779B97F4A7C15ull);
        splitmix64(&s);
        const double cls = u01(&s);
        uint32_t a, b;
        uint64_t dur;
        uint32_t p, o;
        const uint32_t remote = REMOTE_BASE + (uint32_t)uint_in(&s, 1, 1022);
        uint32_t local = remote;
        if (cls < t_fwd && ns) {
            const double u = u01(&s);
            uint32_t lo = 0, hi = ns - 1;
            while (lo < hi) {
                const uint32_t mid = (lo + hi) / 2;
                if (cdf[mid] < u) lo = mid + 1;
                else hi = mid;
            }
            const uint32_t site = perm[lo];
            const uint32_t size = sp->site_size[site];
            uint32_t span = size > 2 ? size - 2 : 1;
            if (sp->hosts_per_site && sp->hosts_per_site < span) span = sp->hosts_per_site;
            local = sp->site_base[site] + (size > 2 ? 1 : 0) + (uint32_t)uint_in(&s, 0, span - 1);
        }
        if (cls < t_ack) {
            p = (uint32_t)uint_in(&s, 10, 500);
            o = p * 40;
            dur = uint_in(&s, 100, 5000);
        } else if (cls < t_admin) {
            p = (uint32_t)uint_in(&s, 1, 19);
            o = p * (uint32_t)uint_in(&s, 100, 500);
            dur = uint_in(&s, 100, 5000);
        } else {
            /* fill_forward(exact=false), toolkit.cpp:108-135 */
            const double z = sqrt(-2.0 * log(u01(&s))) * cos(6.283185307179586 * u01(&s));
            double rate = exp(sp->mu + sp->sigma * z);
            if (rate < 1000.0) rate = 1000.0;
            if (rate > 120000000.0) rate = 120000000.0;
            dur = uint_in(&s, 1000, 8000);
            uint64_t oc = (uint64_t)llround(rate * (double)dur / 8000.0);
            if (oc < 2048) {
                oc = 2048;
                long long d = llround(8000.0 * 2048.0 / rate);
                dur = d < 100 ? 100 : (d > 3600000 ? 3600000 : (uint64_t)d);
            }
            if (oc > 0xFFFFFFFFull) oc = 0xFFFFFFFFull;
            uint64_t pk = oc / 1400 + 1;
            const uint64_t pmax = oc / 97 > 20 ? oc / 97 : 20;
            if (pk < 20) pk = 20;
            if (pk > pmax) pk = pmax;
            o = (uint32_t)oc;
            p = (uint32_t)pk;
        }
        if (cls >= t_fwd) { /* unmatched: both endpoints remote */
            a = remote;
            b = REMOTE_BASE + (uint32_t)uint_in(&s, 1, 1022);
        } else if (splitmix64(&s) & 1) {
            a = local;
            b = remote;
        } else {
            a = remote;
            b = local;
        }
        const uint64_t e = sp->window_start_ms + (sp->window_ms ? splitmix64(&s) % sp->window_ms : 0);
        src[i] = a;
        dst[i] = b;
        pkts[i] = p;
        octets[i] = o;
        end[i] = e;
        start[i] = e - dur;
    }
    free(perm);
    free(cdf);
    return 0;
}

/* SoA -> 64-byte flowmon::FlowRecord AoS (netflow.hpp:32-67 layout): the
 * hot fields at 0,4,16,20,48,56; raw.first/last = low 32 bits of start/end;
 * everything else zero. */
void gnm_synth_to_aos(uint64_t n, const uint32_t* src, const uint32_t* dst, const uint32_t* pkts,
                      const uint32_t* octets, const uint64_t* start, const uint64_t* end,
                      void* out) {
    unsigned char* base = (unsigned char*)out;
    const long long nn = (long long)n;
#pragma omp parallel for schedule(static)
    for (long long i = 0; i < nn; ++i) {
        unsigned char* r = base + (uint64_t)i * 64;
        memset(r, 0, 64);
        const uint32_t first = (uint32_t)start[i], last = (uint32_t)end[i];
        memcpy(r + 0, &src[i], 4);
        memcpy(r + 4, &dst[i], 4);
        memcpy(r + 16, &pkts[i], 4);
        memcpy(r + 20, &octets[i], 4);
        memcpy(r + 24, &first, 4);
        memcpy(r + 28, &last, 4);
        memcpy(r + 48, &start[i], 8);
        memcpy(r + 56, &end[i], 8);
    }
}
