/* ORACLE — test infrastructure only (oracle/refc.py).
 *
 * Forced-include prelude (gcc -include) that lets the reference's own C
 * emission compile unchanged:
 *
 *   - `func main() {` is the entry the reference emits around the program's
 *     statements (src/gpuoffload/codegen.py:141-160); `func` becomes `void`
 *     and `main` is renamed on the command line (-Dmain=b2o_ref_main) so the
 *     shared object can be re-entered;
 *   - top-level declarations stay file-scope globals (codegen.py:143-146), so
 *     the runner reaches every program variable by name (dlsym);
 *   - opaque library calls and replaced blocks are emitted as `name(args);`
 *     (codegen.py:171-180); oracle/refc.py defines each such name as a
 *     function-like macro that reports the call site's ordinal (emission
 *     order, __COUNTER__) to b2o_ref_ext, and the checker applies the app
 *     spec's semantics for it (oracle/externals.py) to the globals in place.
 */
#ifndef B2O_REF_PRELUDE_H
#define B2O_REF_PRELUDE_H

#define func void

typedef void (*b2o_ref_ext_fn)(int site);
b2o_ref_ext_fn b2o_ref_ext = 0;

#endif
