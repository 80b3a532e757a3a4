/* Plain-C client of include/osplat.h (what a caller of the reference capi.h compiles).
 * Built and run by tests/test_c_abi_client.py: host-only calls always; with argv[1] == "gpu" it
 * also renders through osplat_render and runs one device train view + Adam step. */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "osplat.h"

#define CHECK(call)                                                                       \
    do {                                                                                  \
        osplat_status st_ = (call);                                                       \
        if (st_ != OSPLAT_OK) {                                                           \
            fprintf(stderr, "%s failed (%d): %s\n", #call, (int)st_, osplat_last_error()); \
            return 1;                                                                     \
        }                                                                                 \
    } while (0)

int main(int argc, char** argv) {
    const int gpu = argc > 1 && strcmp(argv[1], "gpu") == 0;
    const char* ply = argc > 2 ? argv[2] : "c_abi_client.ply";
    enum { N = 64, DEG = 1, BC = (DEG + 1) * (DEG + 1) };
    double pos[N * 3], sh[N * BC * 3], rot[N * 4], ls[N * 3], op[N];
    srand(7);
    for (int i = 0; i < N; ++i) {
        double th = 6.2831853 * i / N;
        pos[3 * i] = 2.0 * sin(th);
        pos[3 * i + 1] = 0.3 * cos(3.0 * th);
        pos[3 * i + 2] = 2.0 * cos(th);
        rot[4 * i] = 1.0; rot[4 * i + 1] = 0.0; rot[4 * i + 2] = 0.0; rot[4 * i + 3] = 0.0;
        for (int k = 0; k < 3; ++k) ls[3 * i + k] = log(0.05);
        op[i] = 1.0;
        for (int b = 0; b < BC * 3; ++b) sh[i * BC * 3 + b] = 0.1 * ((rand() % 200) / 100.0 - 1.0);
    }
    printf("version %s\n", osplat_version());
    osplat_cloud* cloud = NULL;
    CHECK(osplat_cloud_create(N, DEG, DEG, pos, sh, rot, ls, op, &cloud));
    if (osplat_cloud_count(cloud) != N) return 2;
    CHECK(osplat_cloud_save(cloud, ply));
    osplat_cloud* back = NULL;
    CHECK(osplat_cloud_load(ply, &back));
    if (osplat_cloud_count(back) != N) return 3;
    osplat_config* cfg = NULL;
    CHECK(osplat_config_create(&cfg));
    CHECK(osplat_config_set(cfg, "iterations", "100"));
    if (osplat_config_set(cfg, "nope", "1") != OSPLAT_ERR_PARSE) return 4;
    printf("last_error %s\n", osplat_last_error());

    if (gpu) {
        const double T[16] = {1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1};
        osplat_image* img = NULL;
        CHECK(osplat_render(back, T, 128, 64, &img));
        const double* px = osplat_image_pixels(img);
        double sum = 0.0;
        for (int i = 0; i < 128 * 64 * 3; ++i) sum += px[i];
        printf("render sum %.6f\n", sum);
        if (!(sum > 0.0)) return 5;
        osplat_image_free(img);

        osplat_gpu* ctx = NULL;
        CHECK(osplat_gpu_create(0, NULL, back, &ctx));
        float* target = (float*)calloc(3 * 128 * 64, sizeof(float));
        double loss = 0.0;
        CHECK(osplat_gpu_train_view(ctx, T, 128, 64, target, 0, 0.2, 0.0, &loss));
        CHECK(osplat_gpu_adam_step(ctx, cfg, 1.0, 1, 1));
        printf("loss %.6f launches %lld\n", loss, osplat_gpu_launch_count());
        if (!(loss > 0.0)) return 6;
        /* the pipelined variant: sums arrive after a synchronize (pageable memory here: the copy is
         * then synchronous, which is allowed) */
        double sums[4] = {0, 0, 0, 0};
        CHECK(osplat_gpu_train_view_async(ctx, T, 128, 64, target, 0, 0.2, 0.0, sums));
        CHECK(osplat_gpu_synchronize(ctx));
        const double loss2 = osplat_loss_value(sums, 0.2, 128, 64, 0.0);
        printf("async loss %.6f\n", loss2);
        if (!(loss2 > 0.0)) return 7;
        free(target);
        osplat_gpu_free(ctx);
    }
    osplat_config_free(cfg);
    osplat_cloud_free(back);
    osplat_cloud_free(cloud);
    printf("ok\n");
    return 0;
}
