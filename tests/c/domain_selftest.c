/* domain_selftest.c -- the multi-GPU domain through the C ABI alone (no Python, no torch):
 * a z-periodic vortex stepped by hc_domain_create_local(ngpu = 1) -- the slab exchanges its
 * halos with itself through ncclSend/ncclRecv and all-reduces dt_next through NCCL, the N > 1
 * code path -- by hc_domain_create(rank 0 of world 1, NCCL unique id), by peer copies and by
 * the fused kernels storing the halos themselves (HC_XCHG_STORE), against a single
 * hc_stepper owning all its boundaries. Both builds, ADER and SSP-RK3: the final states and
 * dt must be bit-identical. Prints "ok" and exits 0, or the first difference and exits 1.
 * Build: gcc -O2 -I include tests/c/domain_selftest.c -L paper_2211_13295_b200 -lhydro_cuda */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "hydro_cuda.h"

static void die(const char* what, int rc) {
    char buf[1024];
    hc_last_error(buf, sizeof buf);
    fprintf(stderr, "%s failed (%d): %s\n", what, rc, buf);
    exit(2);
}
#define CK(x)                         \
    do {                              \
        int rc_ = (x);                \
        if (rc_ != HC_OK) die(#x, rc_); \
    } while (0)

static void geom(hc_geom* g, int nx, int ny, int nz, int order) {
    memset(g, 0, sizeof *g);
    g->nx = nx;
    g->ny = ny;
    g->nz = nz;
    g->ghost = order == 2 ? 2 : 3;
    g->dx = 10.0 / nx;
    g->dy = 10.0 / ny;
    g->dz = 10.0 / nz;
    for (int a = 0; a < 3; ++a) g->origin[a] = -5.0;
}

static void params(hc_params* p, int order) {
    memset(p, 0, sizeof *p);
    p->order = order;
    p->solver = HC_HLL;
    p->gamma = 1.4;
    p->lim.cfac_rho = 2.0;
    p->lim.cfac_other = 1.5;
    p->lim.weno_eps = 1e-12;
    p->lim.weno_w[0] = 0.25;
    p->lim.weno_w[1] = 0.5;
    p->lim.weno_w[2] = 0.25;
}

static int run_case(int exact, int integrator, int mode) {
    const int order = 3, nx = 32, ny = 12, nz = 12, steps = 4;
    hc_geom g;
    hc_params p;
    geom(&g, nx, ny, nz, order);
    params(&p, order);
    const int gh = g.ghost;
    const size_t n = (size_t)(nz + 2 * gh) * (ny + 2 * gh) * (nx + 2 * gh) * 5;
    double* s0 = malloc(n * sizeof(double));
    double* a = calloc(n, sizeof(double));
    double* b = calloc(n, sizeof(double));
    CK(hc_init_vortex(&g, p.gamma, order, 0.0, s0));
    /* a z modulation so the z halos matter (the vortex is z-invariant) */
    for (int k = 0; k < nz + 2 * gh; ++k)
        for (size_t i = 0; i < (size_t)(ny + 2 * gh) * (nx + 2 * gh); ++i)
            s0[((size_t)k * (ny + 2 * gh) * (nx + 2 * gh) + i) * 5 + 0] *=
                1.0 + 0.05 * sin(0.7 * k);
    double dt0 = 0.0;
    CK(hc_initial_dt(&g, s0, p.gamma, 0.4, &dt0));

    /* reference run: one stepper, every boundary periodic */
    hc_stepper_opts so = {{HC_PERIODIC, HC_PERIODIC, HC_PERIODIC}, exact, 0, integrator};
    hc_stepper* st = NULL;
    CK(hc_stepper_create(&g, &p, &so, &st));
    CK(hc_stepper_upload(st, s0));
    CK(hc_stepper_set_time(st, 0.0, dt0, 0.4, 0.0));
    CK(hc_stepper_step(st, steps));
    double t1, dt1;
    long n1;
    CK(hc_stepper_sync(st, &t1, &dt1, &n1));
    CK(hc_stepper_download(st, a));
    CK(hc_stepper_destroy(st));

    /* the domain */
    hc_domain_opts o = {{HC_PERIODIC, HC_PERIODIC, HC_PERIODIC}, exact, integrator, 0,
                        mode == 3 ? HC_XCHG_STORE : (mode == 2 ? HC_XCHG_PEER : HC_XCHG_NCCL),
                        mode == 1};
    hc_domain* d = NULL;
    if (mode == 1) {
        unsigned char id[128];
        CK(hc_nccl_unique_id(id, sizeof id));
        CK(hc_domain_create(&g, &p, &o, 0, 1, id, &d));
    } else {
        int dev = 0;
        CK(hc_domain_create_local(&g, &p, &o, 1, &dev, &d));
    }
    CK(hc_domain_scatter(d, s0));
    CK(hc_domain_set_time(d, 0.0, dt0, 0.4, 0.0));
    CK(hc_domain_step(d, steps));
    double t2, dt2;
    long n2;
    CK(hc_domain_sync(d, &t2, &dt2, &n2));
    memcpy(b, a, n * sizeof(double)); /* the gather fills the active planes */
    CK(hc_domain_gather(d, b));
    CK(hc_domain_destroy(d));

    int bad = 0;
    for (int k = gh; k < gh + nz && !bad; ++k)
        for (int j = gh; j < gh + ny && !bad; ++j)
            for (int i = gh; i < gh + nx && !bad; ++i)
                for (int q = 0; q < 5; ++q) {
                    size_t z = (((size_t)k * (ny + 2 * gh) + j) * (nx + 2 * gh) + i) * 5 + q;
                    if (memcmp(&a[z], &b[z], sizeof(double))) {
                        printf("exact=%d integrator=%d mode=%d: zone (%d,%d,%d) var %d: %.17g "
                               "vs %.17g\n", exact, integrator, mode, i - gh, j - gh, k - gh, q,
                               a[z], b[z]);
                        bad = 1;
                        break;
                    }
                }
    if (!bad && (dt1 != dt2 || t1 != t2 || n1 != n2)) {
        printf("exact=%d integrator=%d mode=%d: t/dt/steps %.17g %.17g %ld vs %.17g %.17g %ld\n",
               exact, integrator, mode, t1, dt1, n1, t2, dt2, n2);
        bad = 1;
    }
    free(s0);
    free(a);
    free(b);
    return bad;
}

int main(void) {
    int bad = 0;
    for (int exact = 0; exact <= 1; ++exact)
        for (int ig = 0; ig < 2; ++ig)
            for (int mode = 0; mode <= 3; ++mode) bad |= run_case(exact, ig ? 3 : 0, mode);
    if (!bad) printf("ok\n");
    return bad;
}
