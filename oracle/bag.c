/* oracle/bag.c -- TEST INFRASTRUCTURE ONLY. See bag.h. */
#include "bag.h"

#include <stdlib.h>
#include <string.h>

typedef struct {
  char* name;
  int type;
  int64_t len;
  void* data;
} bag_entry;

struct bag {
  bag_entry* e;
  int n, cap;
};

static size_t elem_size(int type) { return type == BAG_I32 ? 4u : 8u; }

bag* bag_new(void) { return (bag*)calloc(1, sizeof(bag)); }

void bag_free(bag* b) {
  if (!b) return;
  for (int i = 0; i < b->n; ++i) {
    free(b->e[i].name);
    free(b->e[i].data);
  }
  free(b->e);
  free(b);
}

static bag_entry* find(const bag* b, const char* name) {
  for (int i = 0; i < b->n; ++i)
    if (strcmp(b->e[i].name, name) == 0) return &b->e[i];
  return NULL;
}

void bag_put(bag* b, const char* name, int type, const void* data, int64_t len) {
  bag_entry* e = find(b, name);
  if (!e) {
    if (b->n == b->cap) {
      b->cap = b->cap ? 2 * b->cap : 16;
      b->e = (bag_entry*)realloc(b->e, (size_t)b->cap * sizeof(bag_entry));
    }
    e = &b->e[b->n++];
    e->name = (char*)malloc(strlen(name) + 1);
    strcpy(e->name, name);
  } else {
    free(e->data);
  }
  size_t bytes = (size_t)len * elem_size(type);
  e->type = type;
  e->len = len;
  e->data = malloc(bytes ? bytes : 1);
  if (bytes) memcpy(e->data, data, bytes);
}

void bag_put_i32(bag* b, const char* name, int32_t v) { bag_put(b, name, BAG_I32, &v, 1); }
void bag_put_i64(bag* b, const char* name, int64_t v) { bag_put(b, name, BAG_I64, &v, 1); }
void bag_put_f64(bag* b, const char* name, double v) { bag_put(b, name, BAG_F64, &v, 1); }

int bag_count(const bag* b) { return b->n; }
const char* bag_name(const bag* b, int i) { return (i >= 0 && i < b->n) ? b->e[i].name : NULL; }

int bag_type(const bag* b, const char* name) {
  const bag_entry* e = find(b, name);
  return e ? e->type : -1;
}

int64_t bag_len(const bag* b, const char* name) {
  const bag_entry* e = find(b, name);
  return e ? e->len : -1;
}

int bag_get(const bag* b, const char* name, void* dst) {
  const bag_entry* e = find(b, name);
  if (!e) return -1;
  memcpy(dst, e->data, (size_t)e->len * elem_size(e->type));
  return 0;
}
