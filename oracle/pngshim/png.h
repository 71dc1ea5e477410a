/* Declarations of the libpng 1.6 entry points the reference's io_image.cpp
 * calls (core/src/io_image.cpp:92-171), so that file compiles unmodified into
 * the oracle and links against the libpng16 shared object shipped in this
 * image (Pillow's wheel: pillow.libs/libpng16-*.so.16.56.0; no png.h is
 * installed).  Prototypes and constants as in libpng 1.6's png.h.
 * TEST INFRASTRUCTURE ONLY. */
#pragma once
#include <setjmp.h>
#include <stddef.h>
#include <stdio.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PNG_LIBPNG_VER_STRING "1.6.56"

typedef unsigned char png_byte;
typedef unsigned int png_uint_32;
typedef struct png_struct_def png_struct;
typedef png_struct* png_structp;
typedef png_struct** png_structpp;
typedef struct png_info_def png_info;
typedef png_info* png_infop;
typedef png_info** png_infopp;
typedef png_byte* png_bytep;
typedef const png_byte* png_const_bytep;
typedef const char* png_const_charp;
typedef void* png_voidp;
typedef FILE* png_FILE_p;
typedef void (*png_error_ptr)(png_structp, png_const_charp);
typedef void (*png_longjmp_ptr)(jmp_buf, int);

#define PNG_COLOR_MASK_PALETTE 1
#define PNG_COLOR_MASK_COLOR 2
#define PNG_COLOR_MASK_ALPHA 4
#define PNG_COLOR_TYPE_GRAY 0
#define PNG_COLOR_TYPE_PALETTE (PNG_COLOR_MASK_COLOR | PNG_COLOR_MASK_PALETTE)
#define PNG_COLOR_TYPE_RGB (PNG_COLOR_MASK_COLOR)
#define PNG_COLOR_TYPE_RGB_ALPHA (PNG_COLOR_MASK_COLOR | PNG_COLOR_MASK_ALPHA)
#define PNG_COLOR_TYPE_GRAY_ALPHA (PNG_COLOR_MASK_ALPHA)
#define PNG_INTERLACE_NONE 0
#define PNG_COMPRESSION_TYPE_DEFAULT 0
#define PNG_FILTER_TYPE_DEFAULT 0

png_structp png_create_read_struct(png_const_charp user_png_ver, png_voidp error_ptr, png_error_ptr error_fn,
                                   png_error_ptr warn_fn);
png_structp png_create_write_struct(png_const_charp user_png_ver, png_voidp error_ptr, png_error_ptr error_fn,
                                    png_error_ptr warn_fn);
png_infop png_create_info_struct(const png_struct* png_ptr);
void png_destroy_read_struct(png_structpp png_ptr_ptr, png_infopp info_ptr_ptr, png_infopp end_info_ptr_ptr);
void png_destroy_write_struct(png_structpp png_ptr_ptr, png_infopp info_ptr_ptr);
jmp_buf* png_set_longjmp_fn(png_structp png_ptr, png_longjmp_ptr longjmp_fn, size_t jmp_buf_size);
#define png_jmpbuf(png_ptr) (*png_set_longjmp_fn((png_ptr), longjmp, (sizeof(jmp_buf))))
void png_init_io(png_structp png_ptr, png_FILE_p fp);
void png_set_IHDR(const png_struct* png_ptr, png_infop info_ptr, png_uint_32 width, png_uint_32 height, int bit_depth,
                  int color_type, int interlace_method, int compression_method, int filter_method);
void png_write_info(png_structp png_ptr, const png_info* info_ptr);
void png_write_row(png_structp png_ptr, png_const_bytep row);
void png_write_end(png_structp png_ptr, png_infop info_ptr);
int png_sig_cmp(png_const_bytep sig, size_t start, size_t num_to_check);
void png_set_sig_bytes(png_structp png_ptr, int num_bytes);
void png_read_info(png_structp png_ptr, png_infop info_ptr);
png_byte png_get_bit_depth(const png_struct* png_ptr, const png_info* info_ptr);
png_byte png_get_color_type(const png_struct* png_ptr, const png_info* info_ptr);
void png_set_palette_to_rgb(png_structp png_ptr);
void png_set_expand_gray_1_2_4_to_8(png_structp png_ptr);
void png_set_strip_alpha(png_structp png_ptr);
void png_read_update_info(png_structp png_ptr, png_infop info_ptr);
png_uint_32 png_get_image_width(const png_struct* png_ptr, const png_info* info_ptr);
png_uint_32 png_get_image_height(const png_struct* png_ptr, const png_info* info_ptr);
png_byte png_get_channels(const png_struct* png_ptr, const png_info* info_ptr);
void png_read_row(png_structp png_ptr, png_bytep row, png_bytep display_row);
void png_read_end(png_structp png_ptr, png_infop info_ptr);

#ifdef __cplusplus
}
#endif
