/* oracle/bag.h -- TEST INFRASTRUCTURE ONLY (the parity checker, never the product).
 *
 * A "bag" is a named collection of typed arrays used to hand variable-size
 * oracle results (hierarchy artefacts, aggregation maps, coarse operators)
 * across the C boundary to the Python test harness without per-result
 * structs. Both oracle libraries (the C restatement and the wrapper around
 * the compiled reference) export the same bag accessors under their own
 * prefix; ORACLE_PREFIX selects it at compile time.
 */
#ifndef LAMG_ORACLE_BAG_H
#define LAMG_ORACLE_BAG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { BAG_I32 = 0, BAG_I64 = 1, BAG_F64 = 2 };

typedef struct bag bag;

bag* bag_new(void);
void bag_free(bag* b);
/* Copies len elements of the given type under `name` (replacing any prior entry). */
void bag_put(bag* b, const char* name, int type, const void* data, int64_t len);
void bag_put_i32(bag* b, const char* name, int32_t v);
void bag_put_i64(bag* b, const char* name, int64_t v);
void bag_put_f64(bag* b, const char* name, double v);
int bag_count(const bag* b);
const char* bag_name(const bag* b, int i);
int bag_type(const bag* b, const char* name);     /* -1 if absent */
int64_t bag_len(const bag* b, const char* name);  /* -1 if absent */
int bag_get(const bag* b, const char* name, void* dst); /* 0 ok, -1 absent */

#ifdef __cplusplus
}
#endif

#endif
