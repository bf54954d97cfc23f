/*
 * examples/ara_example.c -- the C ABI (include/ara.h) used directly from C, no Python.
 *
 * SPEC.md's worked example (L252-L262): one ELT over a 3-event catalogue with losses
 * {1: 100, 2: 50, 3: 200} and identity financial terms, one layer with OccR = 10, OccL = 100,
 * AggR = 50, AggL = 150, and two trials: [1, 2, 3] and an empty one.  Occurrence-capped losses
 * are [90, 40, 100], the running sum 230, so the first trial pays min(max(230 - 50, 0), 150) =
 * 150 and the empty trial 0: YLT = [[150, 0]].  The YET goes through ara_run_host (host buffers;
 * the library copies them to the device), then ara_metrics_host gives PML/TVaR of the YLT row.
 *
 *   gcc -std=c11 -I include examples/ara_example.c -L paper_1308_2572_b200 -lara \
 *       -Wl,-rpath,$PWD/paper_1308_2572_b200 -o build/ara_example && build/ara_example
 *
 * Prints "YLT 150 0" and the metrics; exits non-zero on any error (e.g. no GPU).
 */
#include <math.h>
#include <stdio.h>

#include "ara.h"

#define CHECK(call)                                                                  \
    do {                                                                             \
        ara_status s_ = (call);                                                      \
        if (s_ != ARA_OK) {                                                          \
            fprintf(stderr, "%s -> %s: %s\n", #call, ara_status_string(s_),          \
                    ctx ? ara_last_error(ctx) : "");                                 \
            if (ctx) ara_destroy(ctx);                                               \
            return 1;                                                                \
        }                                                                            \
    } while (0)

int main(void)
{
    ara_ctx *ctx = NULL;
    CHECK(ara_create(0, NULL, &ctx));

    /* ELTs as CSR over records + financial terms (reading R1) */
    const uint64_t rec_offsets[2] = {0, 3};
    const uint32_t rec_ids[3] = {1, 2, 3};
    const double rec_losses[3] = {100.0, 50.0, 200.0};
    const ara_fin_terms fin[1] = {{1.0, 0.0, INFINITY}};
    CHECK(ara_load_elts(ctx, 3, 1, rec_offsets, rec_ids, rec_losses, fin));

    /* one layer over ELT 0 with occurrence and aggregate terms */
    const ara_layer_terms terms[1] = {{10.0, 100.0, 50.0, 150.0}};
    const uint32_t elt_offsets[2] = {0, 1}, elt_index[1] = {0};
    CHECK(ara_set_layers(ctx, 1, terms, elt_offsets, elt_index));

    /* YET: trial 0 = events 1, 2, 3 in time order; trial 1 empty */
    const uint64_t trial_offsets[3] = {0, 3, 3};
    const uint32_t events[3] = {1, 2, 3};
    double ylt[2] = {-1.0, -1.0};
    CHECK(ara_run_host(ctx, 2, trial_offsets, events, ylt, 0, ARA_RUN_SYNC));
    printf("YLT %g %g\n", ylt[0], ylt[1]);

    const double p[2] = {0.5, 0.99};
    double pml[2], tvar[2];
    CHECK(ara_metrics_host(ctx, ylt, 2, 2, p, pml, tvar));
    printf("PML(0.5) %g TVaR(0.5) %g PML(0.99) %g TVaR(0.99) %g\n", pml[0], tvar[0], pml[1],
           tvar[1]);

    ara_destroy(ctx);
    return (ylt[0] == 150.0 && ylt[1] == 0.0) ? 0 : 2;
}
