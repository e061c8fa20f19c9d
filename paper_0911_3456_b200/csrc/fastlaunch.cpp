// _fastlaunch -- the per-call host path of generated kernels, in C++.
//
// The reference marshals every call in Python: arity and dtype checks, n
// inference, one 8-byte widened slot per scalar (src/elementwise.py:316-366),
// then a ctypes call per worker range.  Here a Plan, built once per (kernel,
// device) from the same rules, does all of that plus the vector-path decision
// (16-byte alignment, no aliasing of written vectors), the grid policy and the
// cuLaunchKernel parameter pack in one C call, then launches through the
// C-ABI runtime (rtcg_launch).  Anything unusual -- a wrong type or dtype, a
// freed array, a short vector, a conversion error -- returns None so the
// Python binder re-runs the call and raises the reference's exception; the
// fast path never guesses.
#define PY_SSIZE_T_CLEAN
#include <Python.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <vector>

namespace {

using launch_fn = int (*)(void *function, unsigned grid, unsigned block, unsigned smem,
                          void *stream, void **params, unsigned flags);   // rtcg_launch_ex
launch_fn g_launch = nullptr;

PyObject *s_dtype, *s_size, *s_freed, *s_block, *s_address;

struct Param {
    bool vec;
    PyObject *dtype;  // borrowed from the plan's owner list
    long long itemsize;
    char kind;        // scalars: 'f', 'i', 'u'
    bool used, written;
};

struct Entry {
    void *fn = nullptr;
    long long per_thread = 1;  // elements per thread-step
    long long resident = 1;    // SMs x occupancy (CTAs)
    int waves = 0;
    unsigned smem = 0;
    long long min_parts = 0;   // partials a launch may store (dynamic chunks), beyond the grid
};

struct Plan {
    PyObject_HEAD
    std::vector<Param> *params;
    PyObject *owners;          // keeps dtype objects / array type alive
    PyTypeObject *array_type;
    Entry vec, gen;
    bool has_vec, has_gen;
    unsigned block;
    long long workers;         // 0 = policy
    int nextra;
};

void plan_dealloc(Plan *self) {
    delete self->params;
    Py_XDECREF(self->owners);
    Py_TYPE(self)->tp_free(reinterpret_cast<PyObject *>(self));
}

bool read_entry(PyObject *t, Entry &e) {
    // (function, per_thread, resident, waves, smem[, min_parts])
    unsigned long long fn;
    long long pt, res, min_parts = 0;
    int waves;
    unsigned smem;
    if (!PyArg_ParseTuple(t, "KLLiI|L", &fn, &pt, &res, &waves, &smem, &min_parts)) return false;
    e.min_parts = min_parts > 0 ? min_parts : 0;
    e.fn = reinterpret_cast<void *>(fn);
    e.per_thread = pt > 0 ? pt : 1;
    e.resident = res > 0 ? res : 1;
    e.waves = waves;
    e.smem = smem;
    return true;
}

// Plan(params, array_type, block, workers, gen_entry_or_None, vec_entry_or_None, nextra)
// params: sequence of (is_vector, dtype, itemsize, kind, used, written)
int plan_init(Plan *self, PyObject *args, PyObject *) {
    PyObject *params, *array_type, *gen, *vec;
    unsigned block;
    long long workers;
    int nextra;
    if (!PyArg_ParseTuple(args, "OOILOOi", &params, &array_type, &block, &workers, &gen, &vec,
                          &nextra))
        return -1;
    if (!PyType_Check(array_type)) {
        PyErr_SetString(PyExc_TypeError, "array_type must be a type");
        return -1;
    }
    PyObject *seq = PySequence_Fast(params, "params must be a sequence");
    if (!seq) return -1;
    self->params = new std::vector<Param>();
    self->owners = PyList_New(0);
    Py_INCREF(array_type);
    PyList_Append(self->owners, array_type);
    Py_DECREF(array_type);
    self->array_type = reinterpret_cast<PyTypeObject *>(array_type);
    const Py_ssize_t count = PySequence_Fast_GET_SIZE(seq);
    for (Py_ssize_t k = 0; k < count; ++k) {
        PyObject *item = PySequence_Fast_GET_ITEM(seq, k);
        int is_vec, used, written;
        PyObject *dtype;
        long long size;
        const char *kind;
        if (!PyArg_ParseTuple(item, "pOLspp", &is_vec, &dtype, &size, &kind, &used, &written)) {
            Py_DECREF(seq);
            return -1;
        }
        PyList_Append(self->owners, dtype);
        self->params->push_back({is_vec != 0, dtype, size, kind[0], used != 0, written != 0});
    }
    Py_DECREF(seq);
    self->block = block;
    self->workers = workers;
    self->nextra = nextra;
    self->has_gen = gen != Py_None;
    if (self->has_gen && !read_entry(gen, self->gen)) return -1;
    self->has_vec = vec != Py_None;
    if (self->has_vec && !read_entry(vec, self->vec)) return -1;
    return 0;
}

long long grid_of(const Plan *p, const Entry &e, long long n) {
    const long long chunk = static_cast<long long>(p->block) * e.per_thread;
    const long long useful = (n + chunk - 1) / chunk;
    long long grid;
    if (p->workers > 0) grid = p->workers;
    else if (e.waves == 0) grid = useful;
    else grid = std::min(e.resident * e.waves, useful);
    if (grid < 1) grid = 1;
    if (grid > 0x7fffffffLL) grid = 0x7fffffffLL;
    return grid;
}

bool attr_ll(PyObject *obj, PyObject *name, long long *out) {
    PyObject *v = PyObject_GetAttr(obj, name);
    if (!v) return false;
    *out = PyLong_AsLongLong(v);
    Py_DECREF(v);
    return !(*out == -1 && PyErr_Occurred());
}

struct VecUse {
    uint64_t local;
    long long size;
    bool written;
};

// plan.launch(args, n, base, stream, max_grid, extra[, flags]) -> grid (int), 0 when
// n == 0 (nothing launched), None = take the Python path, -status on a launch
// error.  `extra` holds the trailing uint64 parameters (reductions);
// `max_grid` >= 0 caps the grid (a reduction's partials capacity), -1 = none;
// `flags` are rtcg_launch_ex flags (RTCG_LAUNCH_OVERLAP_PREVIOUS).
PyObject *plan_launch(Plan *self, PyObject *const *argv, Py_ssize_t argc) {
    if (argc != 6 && argc != 7) {
        PyErr_SetString(PyExc_TypeError,
                        "launch(args, n, base, stream, max_grid, extra[, flags])");
        return nullptr;
    }
    unsigned flags = 0;
    if (argc == 7) {
        flags = static_cast<unsigned>(PyLong_AsUnsignedLong(argv[6]));
        if (PyErr_Occurred()) return nullptr;
    }
    PyObject *args = argv[0];
    if (!PyTuple_Check(args)) Py_RETURN_NONE;
    const auto &params = *self->params;
    const Py_ssize_t count = static_cast<Py_ssize_t>(params.size());
    if (PyTuple_GET_SIZE(args) != count) Py_RETURN_NONE;
    long long n = -1;
    if (argv[1] != Py_None) {
        n = PyLong_AsLongLong(argv[1]);
        if (n == -1 && PyErr_Occurred()) return nullptr;
        if (n < 0) Py_RETURN_NONE;
    }
    const long long base = PyLong_AsLongLong(argv[2]);
    if (base == -1 && PyErr_Occurred()) return nullptr;
    const unsigned long long stream = PyLong_AsUnsignedLongLong(argv[3]);
    if (PyErr_Occurred()) return nullptr;
    const long long max_grid = PyLong_AsLongLong(argv[4]);
    if (max_grid == -1 && PyErr_Occurred()) return nullptr;
    PyObject *extra = argv[5];

    const int total = static_cast<int>(count) + 2 + self->nextra;
    uint64_t vals[128];
    void *ptrs[128];
    if (total > 128) Py_RETURN_NONE;
    VecUse uses[64];
    int nuse = 0;
    uint64_t bits = 0;
    for (Py_ssize_t k = 0; k < count; ++k) {
        const Param &p = params[k];
        PyObject *a = PyTuple_GET_ITEM(args, k);
        if (p.vec) {
            if (Py_TYPE(a) != self->array_type) Py_RETURN_NONE;
            PyObject *dt = PyObject_GetAttr(a, s_dtype);
            if (!dt) return nullptr;
            const bool same = dt == p.dtype;
            Py_DECREF(dt);
            if (!same) Py_RETURN_NONE;
            long long size;
            if (!attr_ll(a, s_size, &size)) return nullptr;
            PyObject *freed = PyObject_GetAttr(a, s_freed);
            if (!freed) return nullptr;
            const bool dead = freed != Py_False;
            Py_DECREF(freed);
            if (dead) Py_RETURN_NONE;
            if (n < 0) n = size;
            else if (size < n) Py_RETURN_NONE;
            PyObject *blk = PyObject_GetAttr(a, s_block);
            if (!blk) return nullptr;
            long long local = 0;
            if (blk != Py_None) {
                const bool ok = attr_ll(blk, s_address, &local);
                Py_DECREF(blk);
                if (!ok) return nullptr;
            } else {
                Py_DECREF(blk);
            }
            const uint64_t addr0 = static_cast<uint64_t>(local) -
                                   static_cast<uint64_t>(base) * static_cast<uint64_t>(p.itemsize);
            vals[k] = addr0;
            if (p.used && nuse < 64) {
                bits |= addr0;
                uses[nuse++] = {static_cast<uint64_t>(local), p.itemsize, p.written};
            }
        } else {
            if (PyObject_TypeCheck(a, self->array_type)) Py_RETURN_NONE;
            if (p.kind == 'f') {
                const double d = PyFloat_AsDouble(a);
                if (d == -1.0 && PyErr_Occurred()) { PyErr_Clear(); Py_RETURN_NONE; }
                memcpy(&vals[k], &d, 8);
            } else {
                PyObject *i = PyNumber_Long(a);
                if (!i) { PyErr_Clear(); Py_RETURN_NONE; }
                vals[k] = PyLong_AsUnsignedLongLongMask(i);
                Py_DECREF(i);
                if (PyErr_Occurred()) { PyErr_Clear(); Py_RETURN_NONE; }
            }
        }
    }
    if (n < 0) Py_RETURN_NONE;            // no vector argument: Python raises
    if (n == 0) return PyLong_FromLong(0);
    // vector path: every used vector 16-byte aligned, no written vector
    // overlapping another used vector over the n elements
    bool vec_ok = self->has_vec && (bits & 15u) == 0;
    for (int a = 0; vec_ok && a < nuse; ++a) {
        if (!uses[a].written) continue;
        const uint64_t lo_a = uses[a].local, hi_a = lo_a + n * uses[a].size;
        for (int b = 0; b < nuse; ++b) {
            if (b == a) continue;
            const uint64_t lo_b = uses[b].local, hi_b = lo_b + n * uses[b].size;
            if (lo_a < hi_b && lo_b < hi_a) { vec_ok = false; break; }
        }
    }
    if (!vec_ok && !self->has_gen) Py_RETURN_NONE;   // general entry not built yet
    const Entry &e = vec_ok ? self->vec : self->gen;
    const long long grid = grid_of(self, e, n);
    if (max_grid >= 0 && std::max(grid, e.min_parts) > max_grid) Py_RETURN_NONE;
    vals[count] = static_cast<uint64_t>(base);
    vals[count + 1] = static_cast<uint64_t>(base + n);
    if (self->nextra) {
        if (!PyTuple_Check(extra) || PyTuple_GET_SIZE(extra) != self->nextra) Py_RETURN_NONE;
        for (int j = 0; j < self->nextra; ++j) {
            vals[count + 2 + j] = PyLong_AsUnsignedLongLongMask(PyTuple_GET_ITEM(extra, j));
            if (PyErr_Occurred()) return nullptr;
        }
    }
    for (int j = 0; j < total; ++j) ptrs[j] = &vals[j];
    if (!g_launch) {
        PyErr_SetString(PyExc_RuntimeError, "_fastlaunch: launcher not set");
        return nullptr;
    }
    const int status = g_launch(e.fn, static_cast<unsigned>(grid), self->block, e.smem,
                                reinterpret_cast<void *>(stream), ptrs, flags);
    if (status != 0) return PyLong_FromLong(-status);   // the caller raises the runtime error
    return PyLong_FromLongLong(grid);
}

PyMethodDef plan_methods[] = {
    {"launch", reinterpret_cast<PyCFunction>(reinterpret_cast<void (*)()>(plan_launch)),
     METH_FASTCALL, "launch(args, n, base, stream, max_grid, extra[, flags]) -> grid | None"},
    {nullptr, nullptr, 0, nullptr}};

PyTypeObject PlanType = {PyVarObject_HEAD_INIT(nullptr, 0)};

PyObject *set_launcher(PyObject *, PyObject *arg) {
    const unsigned long long p = PyLong_AsUnsignedLongLong(arg);
    if (PyErr_Occurred()) return nullptr;
    g_launch = reinterpret_cast<launch_fn>(p);
    Py_RETURN_NONE;
}

PyMethodDef module_methods[] = {
    {"set_launcher", set_launcher, METH_O, "address of rtcg_launch_ex in librtcg_b200.so"},
    {nullptr, nullptr, 0, nullptr}};

PyModuleDef module_def = {PyModuleDef_HEAD_INIT, "_fastlaunch",
                          "Native per-call marshalling and launch of generated kernels.", -1,
                          module_methods};

}  // namespace

PyMODINIT_FUNC PyInit__fastlaunch(void) {
    PlanType.tp_name = "_fastlaunch.Plan";
    PlanType.tp_basicsize = sizeof(Plan);
    PlanType.tp_flags = Py_TPFLAGS_DEFAULT;
    PlanType.tp_new = PyType_GenericNew;
    PlanType.tp_init = reinterpret_cast<initproc>(plan_init);
    PlanType.tp_dealloc = reinterpret_cast<destructor>(plan_dealloc);
    PlanType.tp_methods = plan_methods;
    if (PyType_Ready(&PlanType) < 0) return nullptr;
    s_dtype = PyUnicode_InternFromString("dtype");
    s_size = PyUnicode_InternFromString("size");
    s_freed = PyUnicode_InternFromString("_freed");
    s_block = PyUnicode_InternFromString("_block");
    s_address = PyUnicode_InternFromString("address");
    PyObject *m = PyModule_Create(&module_def);
    if (!m) return nullptr;
    Py_INCREF(&PlanType);
    if (PyModule_AddObject(m, "Plan", reinterpret_cast<PyObject *>(&PlanType)) < 0) {
        Py_DECREF(&PlanType);
        Py_DECREF(m);
        return nullptr;
    }
    return m;
}
