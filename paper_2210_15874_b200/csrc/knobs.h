// knobs.h — the library's A/B tuning knobs, read ONCE from the environment
// (first use), validated and inspectable (qtn_route_config()).
//
// Every knob has a measured default; the environment overrides
// exist for A/B measurements only.  A value that does not parse as an
// integer in the knob's range is rejected with a message on stderr and the
// default kept, so a stray variable can never silently select an
// out-of-range path; bench.py records qtn_route_config() in its line.
#ifndef QTN_KNOBS_H
#define QTN_KNOBS_H

struct QtnKnobs {
  int k3_route;     // QTN_K3_ROUTE  -1 default | 0 never | 1 merged expansions | 2 all large | >=10 width threshold
  int k4_min_e;     // QTN_K4        fewest expansion bits routed to K4 (0 = K4 off)
  int k4_all;       // QTN_K4_ALL    -1 default (complex128 only) | 0 | 1: non-expansion items to K4
  int k5;           // QTN_K5        1: streaming items (a member carries every result bit) to K5 | 2: also
                    //               expansions (<= 4 missing bits) | 0 off
  int pdl;          // QTN_PDL       1: programmatic graph edges | 0 plain edges
  int k3_tcap;      // QTN_K3_TCAP   K3 tile-bit cap (0 = planner's choice)
  int k3_stage_kb;  // QTN_K3_STAGE_KB  K3 staging budget per block (KB)
  int k3_run;       // QTN_K3_RUN    K3 contiguous-run target (bytes)
  int k3_v1;        // QTN_K3_V1     1: K3 first-generation kernel
  int k3_ulim;      // QTN_K3_ULIM   K3 folded-table bits limit
  int k3_inv2;      // QTN_K3_INV2   0: no second invariant operand in K3
  int k6_min_w;     // QTN_K6        narrowest producer fused with its consumer by K6 (0 = K6 off)
  int k2_jitter;    // QTN_K2_JITTER 0 off | seed: K2 blocks stall a pseudo-random 0-4 us before each tile
                    //               (schedule perturbation for the race tests, tests/test_k2_schedule.py)
};

const QtnKnobs& qtn_knobs();

#endif  // QTN_KNOBS_H
