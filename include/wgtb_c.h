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

/* The model's shortlist for (desc, W, H, current device), best first: up to
 * max_n sizes legal on the device - Algorithm 1/2's own answer (what
 * wgtb_predict returns), then the rest of the model's ranking (a forest's
 * labels by vote count, a regressor's sizes by predicted fitness), then that
 * answer's nearest legal neighbours.  wcs / wrs hold max_n entries; *n_out
 * the count written.  No reference counterpart: the paper returns one size. */
int wgtb_shortlist(const char* model_json, const char* kernel_json, const sk_stencil_desc* desc, int64_t width,
                   int64_t height, int32_t max_n, int32_t* wcs, int32_t* wrs, int32_t* n_out);

/* Prediction refined by measurement: every size of the model's shortlist
 * (wgtb_shortlist, max_n sizes) timed on d_in -> d_out with sk_stencil_time
 * (`samples` flushed passes, median); the fastest is returned in *wc / *wr
 * with its median in *best_ms.  max_n = 1 times wgtb_predict's answer only.
 * *timed: sizes timed; *elapsed_ms: the whole tuning time (model + timing).
 * Costs max_n * (samples + 1) passes instead of the exhaustive sweep's
 * 1,466 sizes. */
int wgtb_tune_measured(const char* model_json, const char* kernel_json, const sk_stencil_desc* desc,
                       const void* d_in, void* d_out, int64_t width, int64_t height, int64_t pitch,
                       int32_t max_n, int32_t samples, int32_t* wc, int32_t* wr, int32_t* timed, double* best_ms,
                       double* elapsed_ms);

/* Online tuning (the paper's runtime loop; the reference
 * daemon's session, serve.cpp:123-164): one stencil pass with the size the
 * model proposes for (desc, W, H, current device).  The proposal is cached
 * per session; when the launch is refused (SK_REFUSED / SK_OVERSIZED) the
 * size joins the session's refused set and the model re-proposes - Algorithm
 * 1's fallbacks or Algorithm 2's next candidate - until a launch runs (at
 * most 64 proposals).  *wc_used / *wr_used: the size that ran; *proposals:
 * proposals made in this session so far.  0, or -1 with wgtb_last_error(). */
int wgtb_launch_tuned(const char* model_json, const char* kernel_json, const sk_stencil_desc* desc,
                      const void* d_in, void* d_out, int64_t width, int64_t height, int64_t pitch_in,
                      int64_t pitch_out, void* stream, int32_t* wc_used, int32_t* wr_used,
                      int32_t* proposals);

/* External refusal feedback for a session (serve.cpp's {"type":"refused"}):
 * the size is never proposed again for it; the next wgtb_launch_tuned
 * re-proposes if it was the current proposal. */
int wgtb_tuned_refuse(const char* model_json, const char* kernel_json, const sk_stencil_desc* desc,
                      int64_t width, int64_t height, int32_t wc, int32_t wr);

/* Forget every session. */
void wgtb_tuned_reset(void);

const char* wgtb_last_error(void);

#ifdef __cplusplus
}
#endif

#endif
