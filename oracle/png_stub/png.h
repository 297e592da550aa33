/* Minimal libpng stand-in so the reference io.cpp compiles without libpng
 * (absent from this image).  Written for the oracle build only; every
 * constructor returns NULL, so the reference's PNG reader/writer throws its
 * own io_error at run time.  PGM / SPK1 / raw / SPKR paths are unaffected. */
#ifndef SPK_ORACLE_PNG_STUB_H
#define SPK_ORACLE_PNG_STUB_H
#include <setjmp.h>
#include <stdio.h>

#define PNG_LIBPNG_VER_STRING "stub"
#define PNG_COLOR_TYPE_GRAY 0
#define PNG_INTERLACE_NONE 0
#define PNG_COMPRESSION_TYPE_DEFAULT 0
#define PNG_FILTER_TYPE_DEFAULT 0

typedef unsigned int png_uint_32;
typedef struct png_stub_s { jmp_buf jb; } *png_structp;
typedef void *png_infop;
typedef unsigned char *png_bytep;

static inline png_structp png_create_write_struct(const char*, void*, void*, void*) { return 0; }
static inline png_structp png_create_read_struct(const char*, void*, void*, void*) { return 0; }
static inline png_infop png_create_info_struct(png_structp) { return 0; }
static inline void png_destroy_write_struct(png_structp*, png_infop*) {}
static inline void png_destroy_read_struct(png_structp*, png_infop*, png_infop*) {}
static jmp_buf png_stub_jb;
#define png_jmpbuf(p) (png_stub_jb)
static inline void png_init_io(png_structp, FILE*) {}
static inline void png_set_IHDR(png_structp, png_infop, png_uint_32, png_uint_32, int, int, int, int, int) {}
static inline void png_write_info(png_structp, png_infop) {}
static inline void png_write_row(png_structp, const unsigned char*) {}
static inline void png_write_end(png_structp, png_infop) {}
static inline void png_read_info(png_structp, png_infop) {}
static inline void png_set_expand(png_structp) {}
static inline void png_set_strip_16(png_structp) {}
static inline void png_set_rgb_to_gray(png_structp, int, double, double) {}
static inline void png_set_strip_alpha(png_structp) {}
static inline void png_read_update_info(png_structp, png_infop) {}
static inline png_uint_32 png_get_image_width(png_structp, png_infop) { return 0; }
static inline png_uint_32 png_get_image_height(png_structp, png_infop) { return 0; }
static inline void png_read_row(png_structp, unsigned char*, unsigned char*) {}
#endif
