// Forwarding header: the declarations the reference keeps in hisa/inputs.hpp live in hisa/api.hpp.
#pragma once
#include "hisa/api.hpp"
