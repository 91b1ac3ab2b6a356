// TEST INFRASTRUCTURE — NOT PART OF THE PRODUCT.
// Definitions behind oracle/png_stub/png.h: libpng is absent, so creating a
// PNG reader or writer fails the way libpng reports an allocation failure
// (a null struct), which io.cpp turns into std::runtime_error("libpng init
// failed"). Nothing past png_create_* is ever reached.
#include "png_stub/png.h"

extern "C" {
png_structp png_create_read_struct(const char*, png_voidp, png_error_ptr, png_error_ptr) {
    return nullptr;
}
png_structp png_create_write_struct(const char*, png_voidp, png_error_ptr, png_error_ptr) {
    return nullptr;
}
png_infop png_create_info_struct(png_structp) { return nullptr; }
void png_destroy_read_struct(png_structpp, png_infopp, png_infopp) {}
void png_destroy_write_struct(png_structpp, png_infopp) {}
std::jmp_buf* png_stub_jmpbuf(png_structp) {
    static thread_local std::jmp_buf jb;
    return &jb;
}
void png_init_io(png_structp, png_FILE_p) {}
void png_read_png(png_structp, png_infop, int, png_voidp) {}
void png_write_png(png_structp, png_infop, int, png_voidp) {}
png_uint_32 png_get_image_width(png_structp, png_infop) { return 0; }
png_uint_32 png_get_image_height(png_structp, png_infop) { return 0; }
png_bytepp png_get_rows(png_structp, png_infop) { return nullptr; }
png_size_t png_get_rowbytes(png_structp, png_infop) { return 0; }
void png_set_IHDR(png_structp, png_infop, png_uint_32, png_uint_32, int, int, int, int, int) {}
void png_set_rows(png_structp, png_infop, png_bytepp) {}
}
