/*
 * accudnn_plan.h -- C ABI of the host planner/tuner (libswapsched_b200.so).
 *
 * The reference exposes this path only as the C++ namespace `swapsched`
 * (/root/reference/proj/include/swapsched/*.hpp) driven by its CLI
 * (/root/reference/proj/tools/swapsched.cpp); there is no FFI.  Each entry
 * point below is the document-level operation one CLI subcommand performs,
 * so a foreign binding (ctypes, cgo, JNI) gets the same behaviour with plain
 * strings and scalars:
 *
 *   accudnn_validate   <- run_validate   (swapsched.cpp:174-191)
 *   accudnn_fit        <- run_fit/fit_model (swapsched.cpp:128-137, 193-225)
 *   accudnn_plan       <- run_plan       (swapsched.cpp:241-305)
 *   accudnn_evaluate_k <- evaluate_minibatch (planner.hpp:101-104)
 *   accudnn_phase_times <- phase_compute_times (perf_model.hpp)
 *   accudnn_kmax       <- max_trainable_minibatch (planner.hpp:60-63)
 *   accudnn_simulate   <- run_simulate   (swapsched.cpp:307-383)
 *   accudnn_simulate_report <- run_simulate + write_sim_outputs + verify
 *                            (swapsched.cpp:162-170, 300-383)
 *   accudnn_with_digest <- with_digest   (swapsched.cpp:114-118)
 *   accudnn_sweep      <- run_sweep      (swapsched.cpp:385-420)
 *   accudnn_tune_lr    <- run_tune_lr    (swapsched.cpp:422-438)
 *   accudnn_generate_fixture <- run_gen  (swapsched.cpp:440-456)
 *
 * Conventions: every function returns the CLI exit code (0 success,
 * 1 validation failure / infeasible / untrainable, 2 I/O, 3 internal).  No
 * C++ exception crosses this boundary; the message of the last failure on
 * the calling thread is available from accudnn_last_error().  Output strings
 * are allocated by the library and must be released with accudnn_free().
 */
#ifndef ACCUDNN_PLAN_H_
#define ACCUDNN_PLAN_H_

#ifdef __cplusplus
extern "C" {
#endif

typedef struct accudnn_plan_opts {
  int step;                          /* coarse stride, 1 = linear scan      */
  int k_override;                    /* > 0: evaluate only this minibatch   */
  long long epochs;                  /* TrainingConfig::epochs (default 1)  */
  long long dataset_size;            /* TrainingConfig::dataset_size        */
  unsigned long long budget_override;/* != 0 replaces memory_budget_bytes   */
} accudnn_plan_opts;

const char* accudnn_last_error(void);
void accudnn_free(void* p);

/* GMAP diagnostics, one per line; rc 1 when any diagnostic fires. */
int accudnn_validate(const char* network_json, char** report);

/* Fit model.json from profile CSV texts (compute and/or transfer, sniffed by
 * header).  hardware_json may be NULL (bandwidth fallback 0). */
int accudnn_fit(const char* network_json, const char* const* profile_csvs,
                int n_profiles, const char* hardware_json, double eta,
                char** model_json);

int accudnn_kmax(const char* network_json, const char* hardware_json,
                 int* k_max);

/* plan.json exactly as `swapsched plan` writes it (without the manifest
 * digest).  On infeasible/untrainable returns 1 and a status document. */
int accudnn_plan(const char* network_json, const char* hardware_json,
                 const char* model_json, const accudnn_plan_opts* opts,
                 char** plan_json);

/* the fitted model's 2N phase compute times at minibatch k as CSV
 * ("phase,time_ns", perf_model.cpp:112-132 phase_compute_times) */
int accudnn_phase_times(const char* network_json, const char* model_json, int k,
                        char** times_csv);

/* One KEvaluation as JSON with integer-nanosecond t_ready and pin names. */
int accudnn_evaluate_k(const char* network_json, const char* hardware_json,
                       const char* model_json, int k, char** eval_json);

/* mode: "naive" | "dynamic" | "resident".  plan_json required for dynamic.
 * Writes summary.json and trace.csv texts (either out pointer may be NULL). */
int accudnn_simulate(const char* network_json, const char* hardware_json,
                     const char* model_json, const char* plan_json,
                     const char* mode, int k, char** summary_json,
                     char** trace_csv);

/* The full `swapsched simulate` output set: summary.json, trace.csv,
 * mem_curves.csv, stall_bars.csv and (dynamic mode, i.e. with a plan) the
 * verify_plan document (empty string otherwise).  budget_override != 0
 * replaces memory_budget_bytes.  rc 1: deadlock or failed verdict. */
int accudnn_simulate_report(const char* network_json, const char* hardware_json,
                            const char* model_json, const char* plan_json,
                            const char* mode, int k, unsigned long long budget_override,
                            double tolerance, char** summary_json, char** trace_csv,
                            char** mem_curves_csv, char** stall_bars_csv,
                            char** verify_json);

/* doc re-serialised with "manifest_digest": digest added (indent 2 + '\n'),
 * byte-identical to the reference CLI's output files. */
int accudnn_with_digest(const char* doc, const char* digest, char** out);

int accudnn_sweep(const char* network_json, const char* hardware_json,
                  const char* model_json, const int* k_list, int n_k,
                  const char* modes_csv, int parallel, char** sweep_csv);

int accudnn_tune_lr(double alpha_base, double convexity, double mu, double q,
                    long long iters_base, double* alpha_star, double* residual,
                    long long* adjusted_iterations);

int accudnn_generate_fixture(unsigned long long seed, int min_layers,
                             int max_layers, char** network_json,
                             char** hardware_json, char** compute_csv,
                             char** transfer_csv);

/* Incremental re-planning (no reference counterpart; the reference re-plans
 * from scratch, planner.cpp:346-424).  A session parses the three documents
 * once and caches, per k, everything Algorithm 2 derives independently of
 * the device cap and the host-link bandwidth; each accudnn_plan_session_plan
 * re-runs the search for a new cap (opts->budget_override) and/or bandwidth
 * (bandwidth_override > 0 replaces bandwidth_avail_bytes_per_s) and writes
 * the plan.json a fresh accudnn_plan would write for the changed documents.
 * exact != 0: any opts->step is answered with the step-1 (linear scan)
 * result.  Errors: accudnn_session_last_error(). */
const char* accudnn_session_last_error(void);
int accudnn_plan_session_create(const char* network_json, const char* hardware_json,
                                const char* model_json, void** session);
int accudnn_plan_session_plan(void* session, const accudnn_plan_opts* opts,
                              double bandwidth_override, int exact, char** plan_json);
int accudnn_plan_session_stats(void* session, long long* hits, long long* misses);
void accudnn_plan_session_destroy(void* session);

#ifdef __cplusplus
}
#endif

#endif /* ACCUDNN_PLAN_H_ */
