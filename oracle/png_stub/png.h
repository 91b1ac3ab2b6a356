/* TEST INFRASTRUCTURE — NOT PART OF THE PRODUCT.
 * Declarations-only stand-in for libpng's png.h (absent in this image), so
 * the reference's io.cpp compiles UNMODIFIED into oracle/_ref/libsvr_ref.so
 * and its save_checkpoint / load_checkpoint (io.cpp:229-359) can pin the
 * product's SVRX writer and reader. The PNG functions are defined in
 * oracle/png_stub.cpp to throw: no test decodes or encodes a PNG. */
#pragma once
#include <csetjmp>
#include <cstddef>
#include <cstdio>

typedef unsigned char png_byte;
typedef png_byte* png_bytep;
typedef png_byte** png_bytepp;
typedef struct png_struct_def png_struct;
typedef png_struct* png_structp;
typedef png_struct** png_structpp;
typedef struct png_info_def png_info;
typedef png_info* png_infop;
typedef png_info** png_infopp;
typedef unsigned int png_uint_32;
typedef size_t png_size_t;
typedef void* png_voidp;
typedef void (*png_error_ptr)(png_structp, const char*);
typedef FILE* png_FILE_p;

#define PNG_LIBPNG_VER_STRING "1.6.0-stub"
#define PNG_TRANSFORM_IDENTITY 0x0000
#define PNG_TRANSFORM_STRIP_16 0x0001
#define PNG_TRANSFORM_STRIP_ALPHA 0x0002
#define PNG_TRANSFORM_EXPAND 0x0010
#define PNG_TRANSFORM_GRAY_TO_RGB 0x2000
#define PNG_COLOR_TYPE_RGB 2
#define PNG_INTERLACE_NONE 0
#define PNG_COMPRESSION_TYPE_DEFAULT 0
#define PNG_FILTER_TYPE_DEFAULT 0

extern "C" {
png_structp png_create_read_struct(const char*, png_voidp, png_error_ptr, png_error_ptr);
png_structp png_create_write_struct(const char*, png_voidp, png_error_ptr, png_error_ptr);
png_infop png_create_info_struct(png_structp);
void png_destroy_read_struct(png_structpp, png_infopp, png_infopp);
void png_destroy_write_struct(png_structpp, png_infopp);
std::jmp_buf* png_stub_jmpbuf(png_structp);
void png_init_io(png_structp, png_FILE_p);
void png_read_png(png_structp, png_infop, int, png_voidp);
void png_write_png(png_structp, png_infop, int, png_voidp);
png_uint_32 png_get_image_width(png_structp, png_infop);
png_uint_32 png_get_image_height(png_structp, png_infop);
png_bytepp png_get_rows(png_structp, png_infop);
png_size_t png_get_rowbytes(png_structp, png_infop);
void png_set_IHDR(png_structp, png_infop, png_uint_32, png_uint_32, int, int, int, int, int);
void png_set_rows(png_structp, png_infop, png_bytepp);
}
#define png_jmpbuf(png) (*png_stub_jmpbuf(png))
