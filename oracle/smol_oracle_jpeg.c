/*
 * smol_oracle_jpeg.c -- plain, slow baseline-JPEG entropy decoder (oracle).
 *
 * TEST INFRASTRUCTURE ONLY (see smol_oracle.h): shares no code with the CUDA
 * path.  It follows ITU-T T.81 step by step, sequentially, one bit at a time:
 *   - marker syntax: Annex B (B.2.2 SOF0, B.2.3 SOS, B.2.4.1 DQT, B.2.4.2 DHT,
 *     B.2.4.4 DRI, B.1.1.5 byte stuffing), restart markers RST0..7;
 *   - Huffman code generation: Annex C, Figures C.1 (HUFFSIZE), C.2
 *     (HUFFCODE);
 *   - decoder tables: F.2.2.3, Figure F.15 (MINCODE, MAXCODE, VALPTR);
 *   - DECODE (Figure F.16), RECEIVE (F.17), NEXTBIT (F.18), EXTEND (F.12);
 *   - DC difference decoding F.2.2.1 with prediction (F.2.1.3.1: predictor
 *     reset to 0 at the start of the scan and of every restart interval);
 *   - AC decoding F.2.2.2, Figure F.13 (RRRR/SSSS, ZRL, EOB);
 *   - zig-zag to natural order: Figure A.6;
 *   - MCU order of an interleaved scan: A.2.3; non-interleaved: A.2.2.
 * The paper keeps this step on the host because it "requires substantial
 * branching" (§6.4); SURVEY §8(f) N4 moves it onto the GPU with
 * restart-interval parallelism, checked against this decoder.
 */
#include <stdint.h>
#include <string.h>

#include "smol_oracle.h"

/* Figure A.6: zig-zag index -> natural index (written out). */
static const int oracle_zz[64] = {
   0,  1,  8, 16,  9,  2,  3, 10, 17, 24, 32, 25, 18, 11,  4,  5,
  12, 19, 26, 33, 40, 48, 41, 34, 27, 20, 13,  6,  7, 14, 21, 28,
  35, 42, 49, 56, 57, 50, 43, 36, 29, 22, 15, 23, 30, 37, 44, 51,
  58, 59, 52, 45, 38, 31, 39, 46, 53, 60, 61, 54, 47, 55, 62, 63};

typedef struct {
  int present;
  uint8_t huffval[256];
  int32_t mincode[17], maxcode[17], valptr[17];
} oracle_htab;

static unsigned oracle_be16(const uint8_t* p) { return ((unsigned)p[0] << 8) | p[1]; }

/* Annex C, Figures C.1 and C.2, then F.2.2.3 Figure F.15. */
static int oracle_build_htab(const uint8_t* bits, const uint8_t* vals, int nvals, oracle_htab* t) {
  int huffsize[257], huffcode[257];
  int k = 0;
  for (int i = 1; i <= 16; ++i)                       /* C.1: Generate_size_table */
    for (int j = 1; j <= bits[i - 1]; ++j) {
      if (k >= 256) return 1;
      huffsize[k++] = i;
    }
  huffsize[k] = 0;
  const int lastk = k;
  if (lastk != nvals) return 1;
  int code = 0, si = huffsize[0];                     /* C.2: Generate_code_table */
  k = 0;
  while (huffsize[k]) {
    while (huffsize[k] == si) { huffcode[k++] = code++; }
    if (code > (1 << si)) return 1;                   /* not a prefix code */
    code <<= 1;
    ++si;
  }
  int j = 0;                                          /* F.15: decoder tables */
  for (int l = 1; l <= 16; ++l) {
    if (bits[l - 1] == 0) { t->maxcode[l] = -1; t->mincode[l] = 0; t->valptr[l] = 0; continue; }
    t->valptr[l] = j;
    t->mincode[l] = huffcode[j];
    j += bits[l - 1] - 1;
    t->maxcode[l] = huffcode[j];
    ++j;
  }
  memcpy(t->huffval, vals, (size_t)nvals);
  t->present = 1;
  return 0;
}

typedef struct {
  const uint8_t* d;
  int64_t pos, end;
  int cnt;                   /* bits left in b (F.18 CNT) */
  unsigned b;                /* current byte (F.18 B) */
  int marker;                /* a marker was met inside the entropy-coded data */
} oracle_bits;

/* F.18 NEXTBIT: next bit of the entropy-coded segment; a stuffed 0xFF00 is one
 * 0xFF byte; at a marker the decoder would stop -- here the remaining bits read
 * as 0 and the condition is flagged (a well-formed stream never needs them). */
static int oracle_nextbit(oracle_bits* s) {
  if (s->cnt == 0) {
    unsigned b = 0;
    if (s->pos >= s->end) s->marker = 1;        /* ran off the end of the data */
    if (s->pos < s->end && !s->marker) {
      b = s->d[s->pos++];
      if (b == 0xFF) {
        const unsigned b2 = s->pos < s->end ? s->d[s->pos] : 0xD9;
        if (b2 == 0x00) ++s->pos;
        else { s->marker = 1; --s->pos; b = 0; }
      }
    }
    s->b = b;
    s->cnt = 8;
  }
  --s->cnt;
  return (int)((s->b >> s->cnt) & 1u);
}

/* F.16 DECODE */
static int oracle_decode_sym(oracle_bits* s, const oracle_htab* t) {
  int i = 1;
  int32_t code = oracle_nextbit(s);
  while (i <= 16 && code > t->maxcode[i]) {
    ++i;
    if (i > 16) return -1;
    code = (code << 1) + oracle_nextbit(s);
  }
  if (i > 16) return -1;
  const int j = t->valptr[i] + code - t->mincode[i];
  return t->huffval[j & 255];
}

/* F.17 RECEIVE + F.12 EXTEND */
static int32_t oracle_receive_extend(oracle_bits* s, int ssss) {
  int32_t v = 0;
  for (int i = 0; i < ssss; ++i) v = (v << 1) + oracle_nextbit(s);
  if (ssss && v < (1 << (ssss - 1))) v += (-1 * (1 << ssss)) + 1;
  return v;
}

typedef struct {
  oracle_htab dc[4], ac[4];
  int32_t sos_td[3], sos_ta[3];
  int32_t comp_id[3];
  int64_t scan_start;        /* first byte of entropy-coded data */
} oracle_jpeg_state;

static int oracle_parse(const uint8_t* d, int64_t size, oracle_jpeg_info* info, oracle_jpeg_state* st) {
  memset(info, 0, sizeof(*info));
  memset(st, 0, sizeof(*st));
  if (size < 4 || d[0] != 0xFF || d[1] != 0xD8) return 1;            /* SOI */
  int64_t i = 2;
  int have_sof = 0;
  while (i + 4 <= size) {
    if (d[i] != 0xFF) return 2;
    const unsigned m = d[i + 1];
    if (m == 0xFF) { ++i; continue; }                                  /* fill bytes (B.1.1.2) */
    const unsigned len = oracle_be16(d + i + 2);
    if (len < 2 || i + 2 + len > size) return 3;
    const uint8_t* p = d + i + 4;
    const int64_t plen = (int64_t)len - 2;
    if (m == 0xDB) {                                                   /* DQT */
      int64_t o = 0;
      while (o < plen) {
        const int pq = p[o] >> 4, tq = p[o] & 15;
        if (pq != 0 || tq > 3 || o + 65 > plen) return 4;                /* 8-bit tables only */
        for (int k = 0; k < 64; ++k) info->qt[tq][oracle_zz[k]] = p[o + 1 + k];
        o += 65;
      }
    } else if (m == 0xC4) {                                            /* DHT */
      int64_t o = 0;
      while (o < plen) {
        if (o + 17 > plen) return 5;
        const int tc = p[o] >> 4, th = p[o] & 15;
        int nv = 0;
        for (int k = 0; k < 16; ++k) nv += p[o + 1 + k];
        if (tc > 1 || th > 3 || nv > 256 || o + 17 + nv > plen) return 5;
        if (oracle_build_htab(p + o + 1, p + o + 17, nv, tc ? &st->ac[th] : &st->dc[th])) return 5;
        o += 17 + nv;
      }
    } else if (m == 0xC0 || m == 0xC1) {                               /* SOF0 / SOF1 (Huffman, sequential) */
      if (plen < 6 || p[0] != 8) return 6;
      info->height = (int32_t)oracle_be16(p + 1);
      info->width = (int32_t)oracle_be16(p + 3);
      info->ncomp = p[5];
      if ((info->ncomp != 1 && info->ncomp != 3) || plen < 6 + 3 * info->ncomp) return 6;
      if (info->width <= 0 || info->height <= 0) return 6;
      for (int c = 0; c < info->ncomp; ++c) {
        st->comp_id[c] = p[6 + 3 * c];
        info->h[c] = p[7 + 3 * c] >> 4;
        info->v[c] = p[7 + 3 * c] & 15;
        info->tq[c] = p[8 + 3 * c];
        if (info->h[c] < 1 || info->h[c] > 4 || info->v[c] < 1 || info->v[c] > 4 || info->tq[c] > 3) return 6;
      }
      have_sof = 1;
    } else if ((m >= 0xC2 && m <= 0xCF && m != 0xC4 && m != 0xC8 && m != 0xCC)) {
      return 7;                                                        /* progressive / arithmetic / lossless */
    } else if (m == 0xDD) {                                            /* DRI */
      if (plen < 2) return 8;
      info->restart_interval = (int32_t)oracle_be16(p);
    } else if (m == 0xDA) {                                            /* SOS */
      if (!have_sof || plen < 1) return 9;
      const int ns = p[0];
      if (ns != info->ncomp || plen < 1 + 2 * ns + 3) return 9;        /* one interleaved scan of all components */
      for (int j = 0; j < ns; ++j) {
        if (p[1 + 2 * j] != st->comp_id[j]) return 9;
        st->sos_td[j] = p[2 + 2 * j] >> 4;
        st->sos_ta[j] = p[2 + 2 * j] & 15;
        if (st->sos_td[j] > 3 || st->sos_ta[j] > 3) return 9;
      }
      if (p[1 + 2 * ns] != 0 || p[2 + 2 * ns] != 63 || p[3 + 2 * ns] != 0) return 9;   /* baseline Ss, Se, Ah/Al */
      st->scan_start = i + 2 + len;
      break;
    }
    i += 2 + len;
  }
  if (!have_sof || !st->scan_start) return 10;
  int hmax = 1, vmax = 1;
  for (int c = 0; c < info->ncomp; ++c) {
    if (info->h[c] > hmax) hmax = info->h[c];
    if (info->v[c] > vmax) vmax = info->v[c];
  }
  if (info->ncomp == 1) {                         /* A.2.2: non-interleaved, data unit = MCU */
    const int cw = (info->width * info->h[0] + hmax - 1) / hmax, ch = (info->height * info->v[0] + vmax - 1) / vmax;
    info->blocks_w[0] = (cw + 7) / 8;
    info->blocks_h[0] = (ch + 7) / 8;
    info->mcus_x = info->blocks_w[0];
    info->mcus_y = info->blocks_h[0];
  } else {                                        /* A.2.3: interleaved MCUs of Hc x Vc blocks */
    info->mcus_x = (info->width + 8 * hmax - 1) / (8 * hmax);
    info->mcus_y = (info->height + 8 * vmax - 1) / (8 * vmax);
    for (int c = 0; c < info->ncomp; ++c) {
      info->blocks_w[c] = info->mcus_x * info->h[c];
      info->blocks_h[c] = info->mcus_y * info->v[c];
    }
  }
  for (int c = 0; c < info->ncomp; ++c)
    if (!st->dc[st->sos_td[c]].present || !st->ac[st->sos_ta[c]].present) return 11;
  return 0;
}

int oracle_jpeg_info_of(const uint8_t* data, int64_t size, oracle_jpeg_info* info) {
  oracle_jpeg_state st;
  if (!data || !info) return 1;
  return oracle_parse(data, size, info, &st);
}

/* Decode one block (F.2.2.1 + F.2.2.2) into natural order with absolute DC. */
static int oracle_decode_block(oracle_bits* s, const oracle_htab* dc, const oracle_htab* ac, int32_t* pred,
                               int16_t* blk) {
  int16_t zz[64];
  memset(zz, 0, sizeof(zz));
  const int t = oracle_decode_sym(s, dc);
  if (t < 0 || t > 15) return 1;
  const int32_t diff = oracle_receive_extend(s, t);
  *pred += diff;
  zz[0] = (int16_t)*pred;
  int k = 1;
  while (k <= 63) {                                   /* Figure F.13 */
    const int rs = oracle_decode_sym(s, ac);
    if (rs < 0) return 2;
    const int ssss = rs & 15, r = rs >> 4;
    if (ssss == 0) {
      if (r == 15) { k += 16; continue; }             /* ZRL */
      break;                                          /* EOB */
    }
    k += r;
    if (k > 63) return 3;
    zz[k] = (int16_t)oracle_receive_extend(s, ssss);
    ++k;
  }
  for (int i = 0; i < 64; ++i) blk[oracle_zz[i]] = zz[i];
  return 0;
}

int oracle_jpeg_decode(const uint8_t* data, int64_t size, int16_t* const planes[3]) {
  oracle_jpeg_info info;
  oracle_jpeg_state st;
  if (!data || !planes) return 1;
  int rc = oracle_parse(data, size, &info, &st);
  if (rc) return 100 + rc;
  oracle_bits s;
  memset(&s, 0, sizeof(s));
  s.d = data;
  s.pos = st.scan_start;
  s.end = size;
  int32_t pred[3] = {0, 0, 0};
  const int64_t nmcu = (int64_t)info.mcus_x * info.mcus_y;
  const int ri = info.restart_interval;
  for (int64_t m = 0; m < nmcu; ++m) {
    if (ri && m > 0 && m % ri == 0) {
      /* E.2.4 / F.2.1.3.1: restart interval ends -- discard the padding bits,
       * expect RST((m/ri - 1) mod 8), reset the DC predictors */
      s.cnt = 0;
      s.marker = 0;
      if (s.pos + 2 > s.end || s.d[s.pos] != 0xFF || s.d[s.pos + 1] != 0xD0 + ((m / ri - 1) & 7)) return 20;
      s.pos += 2;
      pred[0] = pred[1] = pred[2] = 0;
    }
    const int64_t my = m / info.mcus_x, mx = m % info.mcus_x;
    for (int c = 0; c < info.ncomp; ++c) {
      const int h = info.ncomp == 1 ? 1 : info.h[c], v = info.ncomp == 1 ? 1 : info.v[c];
      for (int y = 0; y < v; ++y)
        for (int x = 0; x < h; ++x) {
          const int64_t by = my * v + y, bx = mx * h + x;
          int16_t* blk = planes[c] + (by * info.blocks_w[c] + bx) * 64;
          if (oracle_decode_block(&s, &st.dc[st.sos_td[c]], &st.ac[st.sos_ta[c]], &pred[c], blk)) return 30;
        }
    }
  }
  return s.marker ? 40 : 0;      /* the scan ran into a marker before its last MCU */
}
