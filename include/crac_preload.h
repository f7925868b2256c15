/* crac_preload.h — application-facing API of libcrac_preload.so.
 *
 * libcrac_preload.so is an LD_PRELOAD interposer for applications linked
 * against the shared CUDA runtime (nvcc -cudart shared).  It maps
 *   cudaMalloc / cudaMallocManaged / cudaMallocHost / cudaHostAlloc /
 *   cudaFree / cudaFreeHost / cudaStreamCreate{,WithFlags,WithPriority} /
 *   cudaStreamDestroy
 * onto the logged dispatch table of one process-wide cracsim::Session (the
 * call path of ref: src/shim.cpp:204-253, which the reference drives from its
 * harness because it has no real cudart underneath), and admits
 *   cudaLaunchKernel{,ExC} / cudaLaunchCooperativeKernel / cudaGraphLaunch /
 *   cudaMemcpy{,2D,3D,Peer,ToSymbol,FromSymbol}{,Async} /
 *   cudaMemset{,2D,3D}{,Async}
 * through the session's dispatch gate so a checkpoint quiesces them (driver
 * API calls a library makes through cuGetProcAddress pointers bypass the
 * gate: INTEGRATION.md §4, "Un-gated calls").
 * cudaMalloc memory lives in the session's fixed-VA arena, so a device
 * pointer the application holds is the same pointer after a restart.
 *
 * Environment:
 *   CRAC_ARENA_BYTES   arena size of a fresh session (default 16 GiB of VA)
 *   CRAC_SEED          session seed (default 0)
 *   CRAC_RESTART_FROM  image file: the session is restart_from_file'd at the
 *                      first intercepted call instead of created empty
 *   CRAC_CKPT_PATH     where SIGUSR2 writes a checkpoint (asynchronous trigger)
 *   CRAC_PRECOPY       0: stop the application for the whole drain (default:
 *                      a pre-copy drain stops it only to re-send what changed)
 *   CRAC_PRELOAD_VERBOSE  1: counters on stderr at exit
 *
 * Applications may call the functions below through dlsym(RTLD_DEFAULT, ...)
 * so they still run without the preload.  Return: 0 or 1 + cracsim::Errc.
 */
#ifndef CRAC_PRELOAD_H
#define CRAC_PRELOAD_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Drain the session into `path` now (checkpoint_to_file).  The application's
 * own state goes into the image's APPSTATE section via the call below. */
int crac_preload_checkpoint(const char* path);
/* The application's bytes carried in APPSTATE (copied). */
int crac_preload_set_app_state(const void* data, uint64_t n);
/* After a restart: the bytes the application stored (a view owned by the
 * preload); 0 bytes for a fresh session. */
int crac_preload_app_state(const void** data, uint64_t* n);
/* 1 if the session was restored from CRAC_RESTART_FROM. */
int crac_preload_restarted(void);
/* A pointer returned by an intercepted allocation before the checkpoint ->
 * the same allocation now.  Identity for cudaMalloc memory (fixed VA);
 * pinned and managed memory is re-issued by the driver at restart.  NULL if
 * unknown. */
void* crac_preload_translate(const void* old_ptr);
/* The session handle (crac_engine.h), e.g. for crac_summarize. */
void* crac_preload_session(void);

#ifdef __cplusplus
}
#endif

#endif /* CRAC_PRELOAD_H */
