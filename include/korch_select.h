/*
 * korch_select.h — exact solver for the kernel orchestration problem (host side).
 *
 * This is the caller-side selection step of SURVEY.md §8(b): it is NOT part of
 * libkorch.so (the hot-path library never chooses an orchestration; the caller
 * passes its selection to korch_set_orchestration).  It lives in its own library,
 * libkorch_select.so, as the native replacement of the paper's PuLP BLP solve
 * ("solved to optimality ... within 1000 seconds").
 *
 * Problem (with reading A2 of DESIGN.md):
 *   minimise  sum_i c_i u_i                                   (Eq. 2)
 *   s.t.      some selected kernel outputs p_j, for p_j in T  (Eq. 3)
 *             every input p_j of a selected kernel K_k is the
 *             output of some selected kernel                  (Eq. 4)
 * Each candidate has ONE output (reading A4), so an optimal selection assigns
 * exactly one producing candidate to every tensor that must be materialised
 * (a second producer can be dropped: costs are positive).  The solver searches
 * those producer assignments exactly (A* over "pending tensor" sets, below).
 *
 * Tie-break (reading A8): among selections of minimal total cost it returns one
 * with the fewest kernels.
 */
#ifndef KORCH_SELECT_H_
#define KORCH_SELECT_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes (same values as korch.h). */
#define KORCH_SEL_OK              0
#define KORCH_SEL_E_ARG          -1  /* bad argument                                     */
#define KORCH_SEL_E_LIMIT        -5  /* state or time limit reached before proving optimality */
#define KORCH_SEL_E_INFEASIBLE   -6  /* some required tensor has no producer chain        */

/*
 * korch_select_exact — minimum-cost orchestration by A* search.
 *
 * Tensors are numbered 0..n_tensors-1 IN A TOPOLOGICAL ORDER of the primitive
 * graph (every input of a candidate has a smaller number than its output).
 * Tensors that are free (graph inputs, tensors materialised by an earlier
 * partition part) must simply not appear in any candidate's input list.
 *
 *   n_tensors     number of tensors (<= 512)
 *   n_cands       number of candidates M (only generable ones: cost finite, > 0)
 *   cand_output   [M] output tensor of candidate i
 *   cand_in_off   [M+1] CSR offsets into cand_in
 *   cand_in       [cand_in_off[M]] input tensors of candidate i (non-free only)
 *   cand_cost     [M] cost c_i (integer ns, 1 <= c_i < 2^40)
 *   n_required    |T|
 *   required      [n_required] tensors of T
 *   max_states    search-state limit (0 = 50,000,000)
 *   time_limit_s  wall-clock limit in seconds (<= 0: none)
 * Outputs (caller-owned):
 *   best_cost     total cost of the returned selection
 *   sel           [M] 0/1 flags of the selected candidates
 *   n_expanded    number of search states expanded (may be NULL)
 * Returns KORCH_SEL_OK when the selection is proven optimal; KORCH_SEL_E_LIMIT
 * when a limit was hit (sel/best_cost then hold nothing useful);
 * KORCH_SEL_E_INFEASIBLE when no feasible selection exists.  Thread-safe; no
 * global state.
 */
int32_t korch_select_exact(int32_t n_tensors, int32_t n_cands, const int32_t* cand_output,
                           const int32_t* cand_in_off, const int32_t* cand_in, const int64_t* cand_cost,
                           int32_t n_required, const int32_t* required, int64_t max_states,
                           double time_limit_s, int64_t* best_cost, int32_t* sel, int64_t* n_expanded);

#ifdef __cplusplus
}
#endif
#endif /* KORCH_SELECT_H_ */
