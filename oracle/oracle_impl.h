/*
 * CPU oracle kernels, instantiated once per value type (VT / SFX).
 *
 * TEST INFRASTRUCTURE ONLY: this is a plain-C restatement of the reference's
 * numba row kernels (pkg/src/maskmul/_kernels.py) used by tests/ and by
 * bench.py's cpu_baseline / --impl reference legs as the checker and the
 * CPU baseline.  The product path (paper_2111_09947_b200/) never calls it.
 *
 * Each function processes rows [lo, hi), writes only per-row output slots
 * and its own scratch, and returns the number of evaluated products, exactly
 * as the reference kernels do.  Line references are to _kernels.py.
 */

#define CAT2(a, b) a##b
#define CAT(a, b) CAT2(a, b)
#define FN(name) CAT(name, SFX)

/* msa_numeric: _kernels.py:30-87 */
static int64_t FN(msa_numeric)(int64_t lo, int64_t hi, const int64_t* a_ptr, const int64_t* a_idx,
                               const VT* a_val, const int64_t* b_ptr, const int64_t* b_idx,
                               const VT* b_val, const int64_t* m_ptr, const int64_t* m_idx,
                               int comp, int sr, int8_t* states, VT* values, int64_t* inserted,
                               const int64_t* out_off, int64_t* out_idx, VT* out_val,
                               int64_t* row_nnz) {
    int64_t evaluated = 0;
    for (int64_t i = lo; i < hi; i++) {
        int64_t ms = m_ptr[i], me = m_ptr[i + 1];
        if (comp) {
            for (int64_t t = ms; t < me; t++) states[m_idx[t]] = 0;
        } else {
            if (ms == me) { row_nnz[i] = 0; continue; }
            for (int64_t t = ms; t < me; t++) states[m_idx[t]] = 1;
        }
        int64_t nins = 0;
        for (int64_t t = a_ptr[i]; t < a_ptr[i + 1]; t++) {
            int64_t k = a_idx[t];
            VT av = sr == 0 ? a_val[t] : (VT)1;
            for (int64_t s = b_ptr[k]; s < b_ptr[k + 1]; s++) {
                int64_t j = b_idx[s];
                int8_t st = states[j];
                if (st == 0) continue;
                VT p = sr == 0 ? av * b_val[s] : (VT)1;
                evaluated++;
                if (st == 1) {
                    values[j] = p;
                    states[j] = 2;
                    if (comp) inserted[nins++] = j;
                } else {
                    values[j] += p;
                }
            }
        }
        int64_t w = out_off[i], n = 0;
        if (comp) {
            qsort(inserted, (size_t)nins, sizeof(int64_t), cmp_i64);   /* :69 */
            for (int64_t q = 0; q < nins; q++) {
                int64_t j = inserted[q];
                out_idx[w + n] = j;
                out_val[w + n] = values[j];
                n++;
                states[j] = 1;
            }
            for (int64_t t = ms; t < me; t++) states[m_idx[t]] = 1;
        } else {
            for (int64_t t = ms; t < me; t++) {
                int64_t j = m_idx[t];
                if (states[j] == 2) {
                    out_idx[w + n] = j;
                    out_val[w + n] = values[j];
                    n++;
                }
                states[j] = 0;
            }
        }
        row_nnz[i] = n;
    }
    return evaluated;
}

/* hash_numeric: _kernels.py:130-218 (open addressing, linear probing, sentinel = ncols) */
static int64_t FN(hash_numeric)(int64_t lo, int64_t hi, const int64_t* a_ptr, const int64_t* a_idx,
                                const VT* a_val, const int64_t* b_ptr, const int64_t* b_idx,
                                const VT* b_val, const int64_t* m_ptr, const int64_t* m_idx,
                                int comp, int sr, int64_t ncols, const int64_t* row_cap,
                                int64_t* hkeys, int8_t* hstates, VT* hvals, int64_t* inserted,
                                const int64_t* out_off, int64_t* out_idx, VT* out_val,
                                int64_t* row_nnz) {
    int64_t evaluated = 0;
    const int64_t empty = ncols;
    for (int64_t i = lo; i < hi; i++) {
        int64_t ms = m_ptr[i], me = m_ptr[i + 1];
        int64_t flops = 0;
        for (int64_t t = a_ptr[i]; t < a_ptr[i + 1]; t++) {
            int64_t k = a_idx[t];
            flops += b_ptr[k + 1] - b_ptr[k];
        }
        if ((!comp && ms == me) || flops == 0) { row_nnz[i] = 0; continue; }
        int64_t cap = row_cap[i], cap_mask = cap - 1;
        int shift = 64;
        for (int64_t c = cap; c > 1; c >>= 1) shift--;
        for (int64_t q = 0; q < cap; q++) hkeys[q] = empty;
        int8_t mark = comp ? 0 : 1;
        for (int64_t t = ms; t < me; t++) {
            int64_t j = m_idx[t];
            int64_t h = fib_hash(j, shift) & cap_mask;
            while (hkeys[h] != empty && hkeys[h] != j) h = (h + 1) & cap_mask;
            hkeys[h] = j;
            hstates[h] = mark;
        }
        int64_t nins = 0;
        for (int64_t t = a_ptr[i]; t < a_ptr[i + 1]; t++) {
            int64_t k = a_idx[t];
            VT av = sr == 0 ? a_val[t] : (VT)1;
            for (int64_t s = b_ptr[k]; s < b_ptr[k + 1]; s++) {
                int64_t j = b_idx[s];
                int64_t h = fib_hash(j, shift) & cap_mask;
                while (hkeys[h] != empty && hkeys[h] != j) h = (h + 1) & cap_mask;
                if (hkeys[h] == empty) {
                    if (!comp) continue;                       /* :173-174 */
                    hkeys[h] = j;                              /* :175-180 */
                    hvals[h] = sr == 0 ? av * b_val[s] : (VT)1;
                    evaluated++;
                    hstates[h] = 2;
                    inserted[nins++] = j;
                } else {
                    int8_t st = hstates[h];
                    if (st == 0) continue;
                    VT p = sr == 0 ? av * b_val[s] : (VT)1;
                    evaluated++;
                    if (st == 1) {
                        hvals[h] = p;
                        hstates[h] = 2;
                        if (comp) inserted[nins++] = j;
                    } else {
                        hvals[h] += p;
                    }
                }
            }
        }
        int64_t w = out_off[i], n = 0;
        if (comp) {
            qsort(inserted, (size_t)nins, sizeof(int64_t), cmp_i64);   /* :198 */
            for (int64_t q = 0; q < nins; q++) {
                int64_t j = inserted[q];
                int64_t h = fib_hash(j, shift) & cap_mask;
                while (hkeys[h] != j) h = (h + 1) & cap_mask;
                out_idx[w + n] = j;
                out_val[w + n] = hvals[h];
                n++;
            }
        } else {
            for (int64_t t = ms; t < me; t++) {
                int64_t j = m_idx[t];
                int64_t h = fib_hash(j, shift) & cap_mask;
                while (hkeys[h] != empty && hkeys[h] != j) h = (h + 1) & cap_mask;
                if (hkeys[h] == j && hstates[h] == 2) {
                    out_idx[w + n] = j;
                    out_val[w + n] = hvals[h];
                    n++;
                }
            }
        }
        row_nnz[i] = n;
    }
    return evaluated;
}

/* mca_numeric: _kernels.py:275-315 (slots by mask rank, merge scan of B_k vs M_i) */
static int64_t FN(mca_numeric)(int64_t lo, int64_t hi, const int64_t* a_ptr, const int64_t* a_idx,
                               const VT* a_val, const int64_t* b_ptr, const int64_t* b_idx,
                               const VT* b_val, const int64_t* m_ptr, const int64_t* m_idx, int sr,
                               int8_t* states, VT* values, const int64_t* out_off,
                               int64_t* out_idx, VT* out_val, int64_t* row_nnz) {
    int64_t evaluated = 0;
    for (int64_t i = lo; i < hi; i++) {
        int64_t ms = m_ptr[i], me = m_ptr[i + 1], nm = me - ms;
        if (nm == 0) { row_nnz[i] = 0; continue; }
        for (int64_t t = a_ptr[i]; t < a_ptr[i + 1]; t++) {
            int64_t k = a_idx[t];
            VT av = sr == 0 ? a_val[t] : (VT)1;
            int64_t pos = b_ptr[k], end = b_ptr[k + 1];
            for (int64_t rank = 0; rank < nm; rank++) {
                int64_t j = m_idx[ms + rank];
                while (pos < end && b_idx[pos] < j) pos++;
                if (pos >= end) break;
                if (b_idx[pos] == j) {
                    VT p = sr == 0 ? av * b_val[pos] : (VT)1;
                    evaluated++;
                    if (states[rank] == 1) { values[rank] = p; states[rank] = 2; }
                    else values[rank] += p;
                }
            }
        }
        int64_t w = out_off[i], n = 0;
        for (int64_t rank = 0; rank < nm; rank++) {
            if (states[rank] == 2) {
                out_idx[w + n] = m_idx[ms + rank];
                out_val[w + n] = values[rank];
                n++;
                states[rank] = 1;
            }
        }
        row_nnz[i] = n;
    }
    return evaluated;
}

/* heap_numeric: _kernels.py:431-475 (multiway merge of B-row iterators) */
static int64_t FN(heap_numeric)(int64_t lo, int64_t hi, const int64_t* a_ptr, const int64_t* a_idx,
                                const VT* a_val, const int64_t* b_ptr, const int64_t* b_idx,
                                const VT* b_val, const int64_t* m_ptr, const int64_t* m_idx,
                                int comp, int64_t ninspect, int sr, heap_t* hp,
                                const int64_t* out_off, int64_t* out_idx, VT* out_val,
                                int64_t* row_nnz) {
    int64_t evaluated = 0;
    int64_t ni = comp ? 0 : ninspect;
    for (int64_t i = lo; i < hi; i++) {
        int64_t mpos = m_ptr[i], mend = m_ptr[i + 1];
        if (!comp && mpos == mend) { row_nnz[i] = 0; continue; }
        int64_t hn = 0;
        for (int64_t t = a_ptr[i]; t < a_ptr[i + 1]; t++) {
            int64_t k = a_idx[t];
            hn = heap_insert(hp, hn, b_idx, b_ptr[k], b_ptr[k + 1], t, m_idx, mpos, mend, ni);
        }
        int64_t w = out_off[i], n = 0, prev = -1;
        while (hn > 0) {
            int64_t col, pos, end, apos;
            hn = heap_pop(hp, hn, &col, &pos, &end, &apos);
            while (mpos < mend && m_idx[mpos] < col) mpos++;
            int hit;
            if (comp) {
                hit = !(mpos < mend && m_idx[mpos] == col);
            } else {
                if (mpos >= mend) break;
                hit = m_idx[mpos] == col;
            }
            if (hit) {
                VT p = sr == 0 ? a_val[apos] * b_val[pos] : (VT)1;
                evaluated++;
                if (prev == col) {
                    out_val[w + n - 1] += p;
                } else {
                    out_idx[w + n] = col;
                    out_val[w + n] = p;
                    n++;
                    prev = col;
                }
            }
            hn = heap_insert(hp, hn, b_idx, pos + 1, end, apos, m_idx, mpos, mend, ni);
        }
        row_nnz[i] = n;
    }
    return evaluated;
}

/* inner_numeric: _kernels.py:519-554 (pull, B as CSC, ascending-k two-pointer merge) */
static int64_t FN(inner_numeric)(int64_t lo, int64_t hi, const int64_t* a_ptr, const int64_t* a_idx,
                                 const VT* a_val, const int64_t* bc_ptr, const int64_t* bc_row,
                                 const VT* bc_val, const int64_t* m_ptr, const int64_t* m_idx,
                                 int sr, const int64_t* out_off, int64_t* out_idx, VT* out_val,
                                 int64_t* row_nnz) {
    int64_t evaluated = 0;
    for (int64_t i = lo; i < hi; i++) {
        int64_t w = out_off[i], n = 0, ae = a_ptr[i + 1];
        for (int64_t t = m_ptr[i]; t < m_ptr[i + 1]; t++) {
            int64_t j = m_idx[t];
            int64_t ap = a_ptr[i], bp = bc_ptr[j], be = bc_ptr[j + 1];
            VT acc = (VT)1;
            int hit = 0;
            while (ap < ae && bp < be) {
                int64_t ak = a_idx[ap], bk = bc_row[bp];
                if (ak == bk) {
                    VT p = sr == 0 ? a_val[ap] * bc_val[bp] : (VT)1;
                    evaluated++;
                    acc = hit ? acc + p : p;
                    hit = 1;
                    ap++;
                    bp++;
                } else if (ak < bk) {
                    ap++;
                } else {
                    bp++;
                }
            }
            if (hit) {
                out_idx[w + n] = j;
                out_val[w + n] = acc;
                n++;
            }
        }
        row_nnz[i] = n;
    }
    return evaluated;
}

/* compact_rows: _kernels.py:586-594 */
static void FN(compact_rows)(int64_t nrows, const int64_t* bounds_off, const int64_t* row_nnz,
                             const int64_t* tmp_idx, const VT* tmp_val, const int64_t* out_ptr,
                             int64_t* out_idx, VT* out_val) {
    for (int64_t i = 0; i < nrows; i++) {
        int64_t w = out_ptr[i], r = bounds_off[i];
        for (int64_t t = 0; t < row_nnz[i]; t++) {
            out_idx[w + t] = tmp_idx[r + t];
            out_val[w + t] = tmp_val[r + t];
        }
    }
}

/* One row chunk of the numeric phase for any algorithm (multiply.py:269-311). */
static int64_t FN(numeric_chunk)(const or_problem_t* p, int64_t lo, int64_t hi, scratch_t* s,
                                 const int64_t* out_off, int64_t* out_idx, void* out_val_v,
                                 int64_t* row_nnz) {
    VT* out_val = (VT*)out_val_v;
    const VT* a_val = (const VT*)p->a_val;
    const VT* b_val = (const VT*)p->b_val;
    switch (p->algo) {
    case OR_MSA:
        return FN(msa_numeric)(lo, hi, p->a_ptr, p->a_idx, a_val, p->b_ptr, p->b_idx, b_val,
                               p->m_ptr, p->m_idx, p->comp, p->sr, s->states, (VT*)s->values,
                               s->inserted, out_off, out_idx, out_val, row_nnz);
    case OR_HASH:
        return FN(hash_numeric)(lo, hi, p->a_ptr, p->a_idx, a_val, p->b_ptr, p->b_idx, b_val,
                                p->m_ptr, p->m_idx, p->comp, p->sr, p->ncols, p->row_cap,
                                s->hkeys, s->states, (VT*)s->values, s->inserted, out_off,
                                out_idx, out_val, row_nnz);
    case OR_MCA:
        return FN(mca_numeric)(lo, hi, p->a_ptr, p->a_idx, a_val, p->b_ptr, p->b_idx, b_val,
                               p->m_ptr, p->m_idx, p->sr, s->states, (VT*)s->values, out_off,
                               out_idx, out_val, row_nnz);
    case OR_HEAP:
    case OR_HEAPDOT:
        return FN(heap_numeric)(lo, hi, p->a_ptr, p->a_idx, a_val, p->b_ptr, p->b_idx, b_val,
                                p->m_ptr, p->m_idx, p->comp, p->ninspect, p->sr, &s->heap,
                                out_off, out_idx, out_val, row_nnz);
    default:
        return FN(inner_numeric)(lo, hi, p->a_ptr, p->a_idx, a_val, p->b_ptr, p->b_idx, b_val,
                                 p->m_ptr, p->m_idx, p->sr, out_off, out_idx, out_val, row_nnz);
    }
}

#undef FN
