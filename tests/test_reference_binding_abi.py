"""The reference-side ctypes binding (integration/reference_binding.py) loads
libghostx.so and finds every entry point it declares -- no GPU needed."""

from integration import reference_binding as rb


def test_binding_loads_the_library_and_its_entry_points():
    L = rb.lib()
    for name in ("ghx_host_alloc", "ghx_host_free", "ghx_plan_build_fill_boundary", "ghx_plan_free",
                 "ghx_exec_create", "ghx_exec_free", "ghx_exec_run", "ghx_stream_sync", "ghx_interp",
                 "ghx_last_error"):
        assert getattr(L, name) is not None


def test_box_rows_pad_to_3d():
    class B:
        def __init__(self, lo, hi):
            self.lo, self.hi = lo, hi

    rows = rb._rows([B((1, 2), (5, 6))], grow=(1, 2, 0))
    assert rows.tolist() == [[0, 0, 0, 6, 8, 0]]
