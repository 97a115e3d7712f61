// Forwarding header: the declarations the reference keeps in hisa/audit.hpp live in hisa/api.hpp.
#pragma once
#include "hisa/api.hpp"
