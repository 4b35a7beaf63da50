/*
 * wgtb_c.h — C-ABI of the host autotuner (libwgtb.so): the in-process form of
 * the paper's prediction daemon (reference serve.cpp:44-76):
 * a stencil program asks for a workgroup size, the trained model proposes one,
 * and refusals are discovered live on the device (sk_stencil_probe) and fed
 * back into Algorithm 1 (fallbacks) or Algorithm 2 (drop and re-rank).
 */
#ifndef WGTB_C_H
#define WGTB_C_H

#include <stdint.h>

#include "sk_stencil.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Predicts (wc, wr) for the stencil `desc` on a W x H grid of the current
 * CUDA device.  `model_json` is a bundle written by `wgtb train`;
 * `kernel_json` the kernel descriptor (borders + instruction counts) whose
 * features the model was trained on.  *probes receives the number of live
 * legality probes used, *elapsed_ms the tuning time (the paper's "time"
 * metric).  Returns 0, or -1 with wgtb_last_error() set. */
int wgtb_predict(const char* model_json, const char* kernel_json, const sk_stencil_desc* desc,
                 int64_t width, int64_t height, int32_t* wc, int32_t* wr, int32_t* probes,
                 double* elapsed_ms);

const char* wgtb_last_error(void);

#ifdef __cplusplus
}
#endif

#endif
